// launch.cuh -- kernel launchers: packing (full or row band), the
// guard decision per batch, kernel-variant dispatch, row bands of a slab.
// Internal part of libconebeam_b200.so: included, in this order, by
// cbb_runtime.cu (one translation unit: runtime_common.cuh, launch.cuh,
// memory.cuh, pipeline.cuh).
#pragma once

namespace cbb {

// ---------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------

constexpr int kR = 8; // voxels per thread along z

// Detector rows a worker holds and packed cell rows it packs (see
// pack_quads). full(): the whole detector.
struct RowBand {
    int r0 = 0, rn = 0; // raw rows [r0, r0 + rn)
    int q0 = 0, qn = 0; // packed rows [q0, q0 + qn), packed row = py + kPad
    static RowBand full(int H) { return RowBand{0, H, 0, quad_rows(H)}; }
    bool is_full(int H) const { return r0 == 0 && rn == H && q0 == 0 && qn == quad_rows(H); }
};

// The detector rows the voxels of slab [z_begin, z_end) can touch for the
// given projections: the slab box's 8 corners projected (w > 0 over the box
// makes v/w extremal at corners), 2 cells of margin, and the rows -2 / H the
// clamped gathers fall back to when a footprint leaves the detector. The
// kernel computes padding voxels at real ones, so nothing outside is read.
// Full band when w <= 0 somewhere on the box or the rows are unbounded.
RowBand row_band_for(const cbb_volume_geometry& g, int W, int H, int z_begin, int z_end,
                     const double* mats, int count) {
    (void)W;
    const RowBand full = RowBand::full(H);
    const int L = g.edge_voxels;
    const double xs[2] = {g.origin_mm, g.origin_mm + (L - 1) * g.voxel_mm};
    const double zs[2] = {g.origin_mm + z_begin * g.voxel_mm,
                          g.origin_mm + (z_end - 1) * g.voxel_mm};
    double lo = 1e300, hi = -1e300;
    for (int p = 0; p < count; ++p) {
        const double* a = mats + 12 * (size_t)p;
        for (int c = 0; c < 8; ++c) {
            const double x = xs[c & 1], y = xs[(c >> 1) & 1], z = zs[c >> 2];
            const double v = a[1] * x + a[4] * y + a[7] * z + a[10];
            const double ww = a[2] * x + a[5] * y + a[8] * z + a[11];
            if (!(ww > 0.0))
                return full;
            lo = std::min(lo, v / ww);
            hi = std::max(hi, v / ww);
        }
    }
    if (!(lo > -1e7 && hi < 1e7))
        return full;
    const long long fl = (long long)std::floor(lo), fh = (long long)std::floor(hi);
    auto clampll = [](long long v, long long a, long long b) {
        return std::min(std::max(v, a), b);
    };
    const long long c0 = std::min(std::max(fl - 2, (long long)-kPad), clampll(fl - 2, -2, H));
    const long long c1 =
        std::max(std::min(fh + 2, (long long)H + kPad - 1), clampll(fh + 2, -2, H));
    RowBand b;
    b.q0 = (int)(c0 + kPad);
    b.qn = (int)(c1 - c0 + 1);
    b.r0 = (int)std::max(0LL, c0);
    b.rn = (int)std::max(0LL, std::min<long long>(H, c1 + 2) - b.r0);
    if (b.qn >= full.qn)
        return full;
    return b;
}

// Packs `count` projections whose raw rows [band.r0, band.r0 + band.rn) lie
// raw_stride floats apart (band.rn * W for a band buffer, W * H for a full one
// with raw pointing at row 0 -- then pass raw_row0 = 0, raw_rows = H).
void launch_pack_band(const float* raw, int raw_row0, int raw_rows, long long raw_stride, int W,
                      int H, int count, void* packed, const RowBand& band, cudaStream_t st,
                      int* err) {
    const int qp = quad_pitch_cells(W);
    dim3 grid((qp + 127) / 128, (band.qn + kPackRows - 1) / kPackRows, count);
    if (band.qn <= 0 || count <= 0)
        return;
    // zero every projection's metadata word (pack_quads only ever sets it)
    const size_t cells_bytes = (size_t)qp * band.qn * 16;
    CK(cudaMemset2DAsync(static_cast<char*>(packed) + cells_bytes, cells_bytes + kMetaBytes, 0,
                         kMetaBytes, count, st));
    pack_quads<<<grid, 128, 0, st>>>(raw, W, H, raw_row0, raw_rows, raw_stride,
                                     static_cast<float4*>(packed), qp, band.q0, band.qn, err);
    CK(cudaGetLastError());
    ++g_launches;
}

void launch_pack(const float* raw, int W, int H, int count, void* packed, cudaStream_t st,
                 int* err = nullptr) {
    launch_pack_band(raw, 0, H, (long long)W * H, W, H, count, packed, RowBand::full(H), st, err);
}

void launch_check_finite(const float* v, long long n, int* err, cudaStream_t st, int bit = 2) {
    if (n <= 0)
        return;
    const long long blocks = std::min<long long>(148 * 4, (n / 4 + 255) / 256 + 1);
    check_finite<<<(unsigned)blocks, 256, 0, st>>>(v, n, err, bit);
    CK(cudaGetLastError());
    ++g_launches;
}

template <int R, int MODE, bool GUARD, int MINB, int SW = 0, bool CNT = false,
          bool SOA = false, int TW = 8, int BY = kBlockY, bool BIGI = false>
void launch_bp_r(const BpArgs& a, const BpMats& mats, int nz, cudaStream_t st) {
    BpArgs args = a;
    args.nbx = (args.L + kBlockX - 1) / kBlockX;
    args.nby = (args.L + BY - 1) / BY;
    args.nbz = (nz - args.gap + R - 1) / R;
    dim3 block(kBlockX * BY);
    dim3 grid(args.nbx, args.nby, args.nbz);
    if (SW) {
        const long long ns = (long long)((args.nbx + kSX - 1) / kSX) *
                             ((args.nby + kSY - 1) / kSY) * ((args.nbz + kSZ - 1) / kSZ);
        grid = dim3((unsigned)(ns * kSX * kSY * kSZ), 1, 1);
    }
    bp_kernel<R, MODE, GUARD, MINB, SW, CNT, SOA, TW, BY, BIGI><<<grid, block, 0, st>>>(args, mats);
    CK(cudaGetLastError());
    ++g_launches;
}

// Kernel shape variant (tuning experiments; CBB_BP_VARIANT overrides):
// 0 = R 8 voxels/thread, 8x4-voxel warp tiles, 4-warp blocks at 6 blocks/SM,
// voxel-internal pairs (default, measured best on configs 2 and 3). The rest
// use 8-warp blocks at 3 blocks/SM: 1 = R 4, 4 blocks/SM; 2 = R 8, 2
// blocks/SM; 3 = R 4 with super-tile order; 4 = voxel-pair lanes (SOA); 5 =
// the default tile (the v9 shape); 6 / 7 / 8 = warp tiles of 16x2 / 4x8 /
// 32x1 voxels instead of 8x4 (783 / 784 / 774 vs 784 GUp/s exact on config 2).
// Measured and dropped (config 2, exact, vs 790 for variant 5 and 803 for
// the default): 4-warp blocks at 7 blocks/SM (72 registers) 761, at 8
// blocks/SM (64 registers, spills) 715; 16x2 tiles in 4-warp blocks 800;
// 2-warp blocks 770 (16x2 tiles) / 747 (32x1 tiles); 1-warp blocks 682-685;
// 4-warp blocks at 5 blocks/SM (96 registers) 784; R = 4 in 4-warp blocks 746.
// Gathers as ld.global.cg: 799 (no change); with L1::no_allocate: 724.
// z-products wz*(a6, a7), wz*a8 as FMUL2s from per-thread plane coordinates
// instead of broadcast LDS.64 from the block tables (fewer L1 wavefronts,
// more FMA-pipe work): 745 vs 806 exact, 825 vs 903 fast; config 3 811 vs 861.
int bp_variant() {
    const char* e = std::getenv("CBB_BP_VARIANT");
    return e ? std::atoi(e) : 0;
}

// bigi: the packed grid has >= 2^23 cells (detectors beyond ~2800 x 2800):
// integer cell indices, default shape only.
template <int MODE, bool GUARD>
void launch_bp_t(const BpArgs& args, const BpMats& mats, int nz, cudaStream_t st, bool bigi) {
    if constexpr (GUARD) { // (culling does not run here: nothing to count)
        if (bigi)
            return launch_bp_r<kR, MODE, true, 2, 0, false, false, 8, kBlockY, true>(args, mats,
                                                                                   nz, st);
        return launch_bp_r<kR, MODE, true, 2>(args, mats, nz, st);
    } else {
        if (bigi) {
            if (args.counters)
                return launch_bp_r<8, MODE, false, 6, 0, true, false, 8, 4, true>(args, mats, nz,
                                                                                 st);
            return launch_bp_r<8, MODE, false, 6, 0, false, false, 8, 4, true>(args, mats, nz, st);
        }
        if (args.counters) // statistics requested: the counting instantiation
            return launch_bp_r<8, MODE, false, 6, 0, true, false, 8, 4>(args, mats, nz, st);
        switch (bp_variant()) {
        case 1: return launch_bp_r<4, MODE, false, 4>(args, mats, nz, st);
        case 2: return launch_bp_r<8, MODE, false, 2>(args, mats, nz, st);
        case 3: return launch_bp_r<4, MODE, false, 4, 1>(args, mats, nz, st);
        case 4: return launch_bp_r<8, MODE, false, 3, 0, false, true>(args, mats, nz, st);
        case 5: return launch_bp_r<8, MODE, false, 3>(args, mats, nz, st);
        case 6: return launch_bp_r<8, MODE, false, 3, 0, false, false, 16>(args, mats, nz, st);
        case 7: return launch_bp_r<8, MODE, false, 3, 0, false, false, 4>(args, mats, nz, st);
        case 8: return launch_bp_r<8, MODE, false, 3, 0, false, false, 32>(args, mats, nz, st);
        default: // 8x4 warp tiles in 4-warp blocks, 6 blocks/SM: 803 (exact) / 898
                 // (fast) GUp/s on config 2 vs 790 / 879 with 8-warp blocks (variant 5)
            return launch_bp_r<8, MODE, false, 6, 0, false, false, 8, 4>(args, mats, nz, st);
        }
    }
}

// Launches ceil(count/batch) back-projection kernels over a slab. Returns the
// number of guarded launches.
uint64_t launch_backproject(float* vol_slab, const cbb_volume_geometry& g, int z_begin,
                            int z_end, const void* packed, int W, int H, int count,
                            const double* mats, const cbb_options& opt, int* err,
                            cudaStream_t st, int gap_lo = 0, int gap_hi = 0,
                            const RowBand* band = nullptr,
                            unsigned long long* counters = nullptr) {
    const int qp = quad_pitch_cells(W);
    const RowBand b = band ? *band : RowBand::full(H);
    // packed projections of qn rows each; cell row q0 is the buffer's first
    const long long proj_bytes = (long long)qp * b.qn * 16 + kMetaBytes;
    const long long band_shift = (long long)b.q0 * qp * 16;
    BpArgs args;
    args.vol = vol_slab;
    args.proj_bytes = proj_bytes;
    // args.packed is biased by -(kMagic*16 + band_shift): undo that, skip the cells
    args.meta_off = (long long)kMagic * 16 + band_shift + (long long)qp * b.qn * 16;
    args.L = g.edge_voxels;
    args.z_begin = z_begin;
    args.z_end = z_end;
    args.O = (float)g.origin_mm;
    args.MM = (float)g.voxel_mm;
    args.Wf = (float)W;
    args.Hf = (float)H;
    args.qpitchf = (float)qp;
    args.cell_bias = (float)(kPad * qp + kPad) + 8388608.0f;
    args.qpitch = qp;
    args.cell_base = kPad * qp + kPad + kMagic;
    const bool bigi = (double)qp * quad_rows(H) >= kFloatCells;
    args.err = err;
    args.counters = counters;
    args.neg_zero2 = 0x8000000080000000ull;
    args.cull = opt.cull ? 1 : 0;
    // optional skipped planes [gap_lo, gap_hi) (absolute z, gap_lo - z_begin
    // a multiple of 8 so that every z-block stays on one side of the gap)
    args.gap_at = gap_hi > gap_lo ? gap_lo - z_begin : (1 << 30);
    args.gap = gap_hi > gap_lo ? gap_hi - gap_lo : 0;
    uint64_t guarded_launches = 0;
    const int nz = z_end - z_begin;
    if (nz <= 0 || count <= 0)
        return 0;
    const float Of = (float)g.origin_mm, MMf = (float)g.voxel_mm;
    const double cxy = min_nonzero_coord(Of, MMf, 0, g.edge_voxels);
    const double cmin[3] = {cxy, cxy, min_nonzero_coord(Of, MMf, z_begin, z_end)};
    // CBB_FORCE_GUARDED (tests): run every batch through the guarded kernel
    const bool force_guarded = std::getenv("CBB_FORCE_GUARDED") != nullptr && err;
    const int per_launch = std::min(opt.batch, kMaxBatch);
    for (int first = 0; first < count; first += per_launch) {
        const int n = std::min(per_launch, count - first);
        BpMats m;
        bool safe = !force_guarded;
        for (int p = 0; p < n; ++p) {
            const double* a = mats + 12 * (size_t)(first + p);
            store_matrix(m.a[p], a);
            safe = safe && projection_is_safe(a, g, z_begin, z_end, cmin);
        }
        if (!safe && !err)
            fail(CBB_ERR_INVALID,
                 "guarded batch requires an error flag (matrix near w == 0 over the volume)");
        args.count = n;
        args.packed = static_cast<const char*>(packed) + (long long)first * proj_bytes -
                      (long long)kMagic * 16 - band_shift;
        if (opt.mode == CBB_MODE_EXACT) {
            if (safe)
                launch_bp_t<0, false>(args, m, nz, st, bigi);
            else
                launch_bp_t<0, true>(args, m, nz, st, bigi);
        } else {
            if (safe)
                launch_bp_t<1, false>(args, m, nz, st, bigi);
            else
                launch_bp_t<1, true>(args, m, nz, st, bigi);
        }
        guarded_launches += safe ? 0 : 1;
    }
    return guarded_launches;
}

} // namespace cbb
