// launch_tma.cuh -- host side of the TMA-staged back-projection (bp_tma.cuh):
// tensor maps over raw projection buffers, the per-call footprint-box bound,
// the per-projection scan, and the launcher. Internal part of
// libconebeam_b200.so: included by cbb_runtime.cu after launch.cuh.
#pragma once

namespace cbb {

// cuTensorMapEncodeTiled through the runtime's driver entry point (the
// library does not link libcuda).
using PfnTensorMapEncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                             const cuuint64_t*, const cuuint64_t*,
                                             const cuuint32_t*, const cuuint32_t*,
                                             CUtensorMapInterleave, CUtensorMapSwizzle,
                                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline PfnTensorMapEncodeTiled tensor_map_encoder() {
    static PfnTensorMapEncodeTiled fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        cudaGetLastError();
        return reinterpret_cast<PfnTensorMapEncodeTiled>(f);
    }();
    return fn;
}

// Raw projection buffer as a 3-D float tensor (x: W, y: rows, z: count),
// box PITCH x bh x 1, zero fill out of bounds.
inline CUtensorMap raw_tensor_map(const float* raw, int W, int rows, long long stride, int count,
                                  int pitch, int bh) {
    CUtensorMap map;
    const auto enc = tensor_map_encoder();
    if (!enc)
        fail(CBB_ERR_INTERNAL, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)rows, (cuuint64_t)count};
    const cuuint64_t strides[2] = {(cuuint64_t)W * 4, (cuuint64_t)stride * 4};
    const cuuint32_t box[3] = {(cuuint32_t)pitch, (cuuint32_t)bh, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(raw), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        fail(CBB_ERR_INTERNAL, "cuTensorMapEncodeTiled failed (CUresult %d)", (int)r);
    return map;
}

// Box widths the kernel is instantiated for (== 16 mod 32 floats: the rows
// iy and iy + 1 of a warp's taps fall on shifted bank halves).
constexpr int kPitches[] = {48, 80, 112, 144};
#ifndef CBB_TMA_SMEM_KB
#define CBB_TMA_SMEM_KB 60
#endif
constexpr int kTmaSmemBudget = CBB_TMA_SMEM_KB * 1024; // stages per block: 3 blocks/SM (+13.5 KB static)
constexpr int kTmaMinStages = 3;

struct TmaPlan {
    bool ok = false;
    int pitch = 0, bh = 0, stages = 0;
    int bw_need = 0, bh_need = 0; // sampled footprint bound (before rounding)
};

// Footprint bound of a 16 x 16 x 8 block tile over the slab, for these
// projections: exact (double) footprints of 5 x 5 x 5 sampled block positions
// (the slab's extreme blocks included), each spanning
// [floor(min ix), floor(max ix) + 2], plus 2 pixels for the device's
// approximate corner arithmetic. Blocks whose footprint exceeds the box at
// run time read their taps from global memory instead, so this bound only
// affects speed. Cached per (geometry, slab, detector, matrices).
inline TmaPlan plan_tma(const cbb_volume_geometry& g, int W, int H, int z_begin, int z_end,
                        const double* mats, int count) {
    TmaPlan plan;
    if (W % 4 != 0 || count < 1 || z_end <= z_begin)
        return plan;
    static std::mutex mu;
    static std::map<uint64_t, TmaPlan> cache;
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](const void* d, size_t n) {
        const unsigned char* b = static_cast<const unsigned char*>(d);
        for (size_t i = 0; i < n; ++i) {
            h ^= b[i];
            h *= 1099511628211ull;
        }
    };
    const int key_ints[5] = {g.edge_voxels, W, H, z_begin, z_end};
    mix(key_ints, sizeof key_ints);
    mix(&g.voxel_mm, 8);
    mix(&g.origin_mm, 8);
    mix(mats, sizeof(double) * 12 * (size_t)count);
    if (const char* e = std::getenv("CBB_TMA_BOX"))
        mix(e, std::strlen(e));
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(h);
        if (it != cache.end())
            return it->second;
    }
    const int L = g.edge_voxels;
    const int nbx = (L + kTBX - 1) / kTBX, nbz = (z_end - z_begin + kTR - 1) / kTR;
    auto pick = [](int n, int i) { return std::min(n - 1, (n - 1) * i / 4); };
    double bw = 0.0, bhh = 0.0;
    bool finite = true;
    for (int p = 0; p < count && finite; ++p) {
        const double* a = mats + 12 * (size_t)p;
        for (int sx = 0; sx < 5; ++sx)
            for (int sy = 0; sy < 5; ++sy)
                for (int sz = 0; sz < 5; ++sz) {
                    const int bx = pick(nbx, sx), by = pick(nbx, sy), bz = pick(nbz, sz);
                    const double x0 = g.origin_mm + std::min(bx * kTBX, L - 1) * g.voxel_mm;
                    const double x1 = g.origin_mm + std::min(bx * kTBX + kTBX - 1, L - 1) * g.voxel_mm;
                    const double y0 = g.origin_mm + std::min(by * kTBY, L - 1) * g.voxel_mm;
                    const double y1 = g.origin_mm + std::min(by * kTBY + kTBY - 1, L - 1) * g.voxel_mm;
                    const int za = z_begin + bz * kTR;
                    const double z0 = g.origin_mm + za * g.voxel_mm;
                    const double z1 = g.origin_mm + std::min(za + kTR - 1, z_end - 1) * g.voxel_mm;
                    double lx = 1e300, hx = -1e300, ly = 1e300, hy = -1e300;
                    for (int c = 0; c < 8; ++c) {
                        const double X = (c & 1) ? x1 : x0, Y = (c & 2) ? y1 : y0,
                                     Z = (c & 4) ? z1 : z0;
                        const double w = a[2] * X + a[5] * Y + a[8] * Z + a[11];
                        if (!(w > 0.0)) {
                            finite = false;
                            break;
                        }
                        const double ix = (a[0] * X + a[3] * Y + a[6] * Z + a[9]) / w;
                        const double iy = (a[1] * X + a[4] * Y + a[7] * Z + a[10]) / w;
                        lx = std::min(lx, ix);
                        hx = std::max(hx, ix);
                        ly = std::min(ly, iy);
                        hy = std::max(hy, iy);
                    }
                    if (!finite)
                        break;
                    // footprints entirely off the detector are culled (unless a
                    // warp holds -0.0 voxels: then the runtime check decides)
                    if (hx < -2.0 || lx > W || hy < -2.0 || ly > H)
                        continue;
                    // box starts are aligned down to 4 floats (TMA, 16 B)
                    const double ax = 4.0 * std::floor(std::floor(lx) / 4.0);
                    bw = std::max(bw, std::floor(hx) + 2.0 - ax + 1.0);
                    bhh = std::max(bhh, std::floor(hy) + 2.0 - std::floor(ly) + 1.0);
                }
    }
    if (const char* e = std::getenv("CBB_TMA_BOX")) { // tests: force a box, blocks overflow
        int fw = 0, fh = 0;
        if (std::sscanf(e, "%dx%d", &fw, &fh) == 2 && fw > 0 && fh > 0) {
            bw = fw - 2;
            bhh = fh - 2;
        }
    }
    if (finite && bw > 0.0) {
        plan.bw_need = (int)bw + 2;
        plan.bh_need = (int)bhh + 2;
        for (int pch : kPitches)
            if (pch >= plan.bw_need) {
                plan.pitch = pch;
                break;
            }
        plan.bh = (plan.bh_need + 1) & ~1;
        if (plan.pitch > 0)
            plan.stages = std::min(kTMaxStages, kTmaSmemBudget / (plan.pitch * plan.bh * 4));
        plan.ok = plan.pitch > 0 && plan.bh <= 256 && plan.stages >= kTmaMinStages;
    }
    std::lock_guard<std::mutex> lk(mu);
    if (cache.size() > 256)
        cache.clear();
    cache[h] = plan;
    return plan;
}

// CBB_BP_PATH=quad selects the packed-quad gather kernel everywhere (read on
// every call: tests switch it inside one process).
inline bool tma_path_enabled() {
    const char* e = std::getenv("CBB_BP_PATH");
    return !(e && std::string(e) == "quad");
}

// Scans `count` raw projections (rows x W floats each, `stride` floats apart)
// into flags (zeroed here) and err bit 2.
inline void launch_scan(const float* raw, int W, int rows, long long stride, int count,
                        unsigned* flags, int* err, cudaStream_t st) {
    if (count <= 0)
        return;
    CK(cudaMemsetAsync(flags, 0, sizeof(unsigned) * count, st));
    const long long n = (long long)W * rows;
    const int per = (int)std::min<long long>(64, std::max<long long>(1, n / (256 * 16)));
    for (int c0 = 0; c0 < count; c0 += 65535) {
        const int c = std::min(65535, count - c0);
        scan_projections<<<dim3(per, c), 256, 0, st>>>(raw + (long long)c0 * stride, n, stride,
                                                       flags + c0, err);
        CK(cudaGetLastError());
        ++g_launches;
    }
}

template <int MODE, int PITCH>
void launch_tma_kernel(const CUtensorMap& map, const TmaArgs& a, const TmaMats& m, int nz,
                       cudaStream_t st, bool cnt) {
    const size_t smem = (size_t)a.stages * PITCH * a.bh * 4;
    const dim3 grid((a.L + kTBX - 1) / kTBX, (a.L + kTBY - 1) / kTBY, (nz - a.gap + kTR - 1) / kTR);
    static bool attr[2][64] = {};
    int dev = 0;
    CK(cudaGetDevice(&dev));
    auto kern = cnt ? bp_tma_kernel<MODE, PITCH, true> : bp_tma_kernel<MODE, PITCH, false>;
    if (dev < 64 && !attr[cnt][dev]) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kTmaSmemBudget + 1024));
        attr[cnt][dev] = true;
    }
    kern<<<grid, kTThreads, smem, st>>>(map, a, m);
    CK(cudaGetLastError());
    ++g_launches;
}

template <int MODE>
void launch_tma_pitch(const CUtensorMap& map, const TmaArgs& a, const TmaMats& m, int nz,
                      cudaStream_t st, bool cnt, int pitch) {
    switch (pitch) {
    case 48: return launch_tma_kernel<MODE, 48>(map, a, m, nz, st, cnt);
    case 80: return launch_tma_kernel<MODE, 80>(map, a, m, nz, st, cnt);
    case 112: return launch_tma_kernel<MODE, 112>(map, a, m, nz, st, cnt);
    default: return launch_tma_kernel<MODE, 144>(map, a, m, nz, st, cnt);
    }
}

// Back-projects `count` raw projections (held rows [band.r0, band.r0 +
// band.rn) of each, `raw_stride` floats apart; raw points at row band.r0 of
// projection 0) into slab [z_begin, z_end), in launches of opt.batch.
// flags: the scan_projections flags of these projections. Returns the
// number of guarded launches. The caller checked plan.ok.
inline uint64_t launch_backproject_raw(float* vol_slab, const cbb_volume_geometry& g, int z_begin,
                                       int z_end, const float* raw, long long raw_stride, int W,
                                       int H, int band_r0, int band_rn, int count,
                                       const double* mats, const unsigned* flags,
                                       const TmaPlan& plan, const cbb_options& opt, int* err,
                                       cudaStream_t st, int gap_lo = 0, int gap_hi = 0,
                                       unsigned long long* counters = nullptr) {
    const int nz = z_end - z_begin;
    if (nz <= 0 || count <= 0)
        return 0;
    TmaArgs a{};
    a.vol = vol_slab;
    a.raw_stride = raw_stride;
    a.err = err;
    a.neg_zero2 = 0x8000000080000000ull;
    a.counters = counters;
    a.L = g.edge_voxels;
    a.z_begin = z_begin;
    a.z_end = z_end;
    a.O = (float)g.origin_mm;
    a.MM = (float)g.voxel_mm;
    a.Wf = (float)W;
    a.Hf = (float)H;
    a.W = W;
    a.H = H;
    a.raw_row0 = band_r0;
    a.raw_rows = band_rn;
    a.tz0 = 0;
    a.bh = plan.bh;
    a.stages = plan.stages;
    a.cull = opt.cull ? 1 : 0;
    a.gap_at = gap_hi > gap_lo ? gap_lo - z_begin : (1 << 30);
    a.gap = gap_hi > gap_lo ? gap_hi - gap_lo : 0;
    a.magic_off = 0u - 4u * (unsigned)kMagic;
    const float Of = (float)g.origin_mm, MMf = (float)g.voxel_mm;
    const double cxy = min_nonzero_coord(Of, MMf, 0, g.edge_voxels);
    const double cmin[3] = {cxy, cxy, min_nonzero_coord(Of, MMf, z_begin, z_end)};
    const bool force_guarded = std::getenv("CBB_FORCE_GUARDED") != nullptr && err;
    uint64_t guarded = 0;
    // launches of up to kTmaBatch projections (64-bit masks), whatever
    // opt.batch (the pipeline's upload batch) is: the per-block setup and the
    // slab's read-modify-write are amortised over more projections
    for (int first = 0; first < count; first += kTmaBatch) {
        const int n = std::min(kTmaBatch, count - first);
        TmaMats m;
        bool safe = !force_guarded;
        for (int p = 0; p < n; ++p) {
            const double* am = mats + 12 * (size_t)(first + p);
            store_matrix(m.a[p], am);
            safe = safe && projection_is_safe(am, g, z_begin, z_end, cmin);
        }
        if (!safe && !err)
            fail(CBB_ERR_INVALID,
                 "guarded batch requires an error flag (matrix near w == 0 over the volume)");
        a.count = n;
        a.raw = raw + (long long)first * raw_stride;
        a.flags = flags + first;
        if (safe) {
            const CUtensorMap map =
                raw_tensor_map(a.raw, W, band_rn, raw_stride, n, plan.pitch, plan.bh);
            if (opt.mode == CBB_MODE_EXACT)
                launch_tma_pitch<0>(map, a, m, nz, st, counters != nullptr, plan.pitch);
            else
                launch_tma_pitch<1>(map, a, m, nz, st, counters != nullptr, plan.pitch);
        } else {
            const dim3 grid((a.L + 31) / 32, (a.L + 7) / 8, (nz - a.gap + kGR - 1) / kGR);
            if (opt.mode == CBB_MODE_EXACT)
                bp_guarded_raw<0><<<grid, 256, 0, st>>>(a, m);
            else
                bp_guarded_raw<1><<<grid, 256, 0, st>>>(a, m);
            CK(cudaGetLastError());
            ++g_launches;
            ++guarded;
        }
    }
    return guarded;
}

} // namespace cbb
