// cbb_runtime.cu -- host runtime and C ABI of libconebeam_b200.so.
//
// Implements include/conebeam_b200.h: error model mirroring the reference C
// API (proj/src/capi.cpp:26-68), the guard decision per batch, launches of the
// sm_100a kernels in bp_kernels.cuh, and the staging pipeline:
//   host projections --(pinned, double-buffered cudaMemcpyAsync on a copy
//   stream)--> raw ring slot --(pack_quads on the compute stream)--> packed
//   ring slot --(bp_kernel, matrices as kernel parameters = constant bank)-->
//   register partial sums --> volume slab in HBM.
// Multi-GPU (one process): the volume is split into z-slabs, one per device;
// every device receives every projection batch; slabs are downloaded into the
// caller's volume at the end (no reduction: voxel ownership is disjoint).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include "../../include/conebeam_b200.h"
#include "bp_kernels.cuh"
#include "ramp_filter.cuh"
#include "metrics.cuh"
#include "texture_variant.cuh"

namespace cbb {

// ---------------------------------------------------------------------------
// Errors (reference: proj/include/conebeam/errors.hpp:10-44, capi.cpp:30-60)
// ---------------------------------------------------------------------------

struct Error : std::runtime_error {
    cbb_status status;
    Error(cbb_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

thread_local std::string g_last_error;
thread_local uint64_t g_launches = 0;

[[noreturn]] void fail(cbb_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    throw Error(s, buf);
}

void check_cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess)
        return;
    cudaGetLastError(); // clear sticky-free errors
    if (e == cudaErrorMemoryAllocation)
        fail(CBB_ERR_NOMEM, "%s: %s", what, cudaGetErrorString(e));
    fail(CBB_ERR_INTERNAL, "%s: %s", what, cudaGetErrorString(e));
}
#define CK(call) check_cuda((call), #call)

template <typename Fn>
cbb_status guarded(Fn&& fn) noexcept {
    try {
        fn();
        return CBB_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.status;
    } catch (const std::bad_alloc&) {
        g_last_error = "out of memory";
        return CBB_ERR_NOMEM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return CBB_ERR_INTERNAL;
    } catch (...) {
        g_last_error = "unknown error";
        return CBB_ERR_INTERNAL;
    }
}

// ---------------------------------------------------------------------------
// Validation (VolumeGeometry::validate, proj/src/geometry.cpp:17-24;
// ProjectionMatrix::validate :35-39)
// ---------------------------------------------------------------------------

void validate_geometry(const cbb_volume_geometry* g) {
    if (!g)
        fail(CBB_ERR_INVALID, "null volume geometry");
    if (g->edge_voxels < 1)
        fail(CBB_ERR_INVALID, "VolumeGeometry: field 'edge_voxels' must be >= 1");
    if (!(g->voxel_mm > 0.0) || !std::isfinite(g->voxel_mm))
        fail(CBB_ERR_INVALID, "VolumeGeometry: field 'voxel_mm' must be positive and finite");
    if (!std::isfinite(g->origin_mm))
        fail(CBB_ERR_INVALID, "VolumeGeometry: field 'origin_mm' must be finite");
    if (g->edge_voxels > 4096)
        fail(CBB_ERR_INVALID, "VolumeGeometry: edge_voxels > 4096 not supported");
}

void validate_detector(int32_t w, int32_t h) {
    if (w < 1 || h < 1)
        fail(CBB_ERR_INVALID, "ProjectionImage: dimensions must be >= 1");
    // packed cell indices are formed exactly in float: must stay below 2^23
    const double cells = (double)quad_pitch_cells(w) * quad_rows(h);
    if (cells >= 8388608.0 - 16)
        fail(CBB_ERR_INVALID, "detector %dx%d too large for the packed layout", w, h);
}

void validate_matrices(const double* mats, int32_t count) {
    for (int32_t p = 0; p < count; ++p)
        for (int i = 0; i < 12; ++i)
            if (!std::isfinite(mats[12 * (size_t)p + i]))
                fail(CBB_ERR_INVALID, "ProjectionMatrix: field 'a[%d]' must be finite", i);
}

cbb_options resolve_options(const cbb_options* o) {
    cbb_options r;
    cbb_options_defaults(&r);
    if (o)
        r = *o;
    if (r.batch < 1 || r.batch > kMaxBatch)
        fail(CBB_ERR_INVALID, "options: batch must be in [1, %d]", kMaxBatch);
    if (r.mode != CBB_MODE_EXACT && r.mode != CBB_MODE_FAST)
        fail(CBB_ERR_INVALID, "options: unknown mode %d", r.mode);
    if (r.num_gpus < 0)
        fail(CBB_ERR_INVALID, "options: num_gpus must be >= 0");
    if (r.slab_begin < 0 || r.slab_end < 0 || (r.slab_end != 0 && r.slab_end <= r.slab_begin))
        fail(CBB_ERR_INVALID, "options: bad slab [%d, %d)", r.slab_begin, r.slab_end);
    if (r.ramp_filter && !(r.filter_pixel_mm > 0.0 && std::isfinite(r.filter_pixel_mm)))
        fail(CBB_ERR_INVALID, "options: ramp filter needs a positive filter_pixel_mm");
    return r;
}

// ---------------------------------------------------------------------------
// Guard decision. A batch may run the unguarded kernel when, for every
// projection, w > 0 with margin at the 8 corners of the slab box and the
// projected corners satisfy |ix|,|iy| < 1e8. w is affine in the voxel
// coordinates, so positive corners imply w > 0 inside; u/w and v/w are
// linear-fractional with a positive denominator, hence monotone along every
// line and extremal at box vertices. The float kernel differs from the double
// evaluation by a few ulps, far inside both margins. Matrices containing a
// -0.0 coefficient are sent to the guarded kernel too (signed-zero corner
// cases of the IEEE division are then handled by the reference arithmetic).
// ---------------------------------------------------------------------------

// Smallest nonzero |O + i*MM| over i in [i0, i1), evaluated in float exactly
// as the kernel does (0 when every coordinate is exactly zero).
double min_nonzero_coord(float O, float MM, int i0, int i1) {
    double m = 0.0;
    for (int i = i0; i < i1; ++i) {
        volatile float t = (float)i * MM;
        volatile float c = O + t;
        const double ac = std::fabs((double)c);
        if (ac != 0.0 && (m == 0.0 || ac < m))
            m = ac;
    }
    return m;
}

// Every nonzero partial sum of ((t1 + t2) + t3) + t4 is a multiple of the
// smallest ulp among its nonzero float terms, so nonzero |u| >= 2^(e - 23)
// with e the exponent of the smallest nonzero term. Requires |u| >= 2^-63.
bool coordinate_sum_bounded(const float* af, const int idx[4], const double cmin[3]) {
    double tmin = 0.0;
    for (int k = 0; k < 4; ++k) {
        const double ak = std::fabs((double)af[idx[k]]);
        if (ak == 0.0)
            continue;
        double t = k < 3 ? ak * cmin[k] * 0.5 : ak; // 0.5: product rounding
        if (k < 3 && cmin[k] == 0.0)
            continue;
        if (tmin == 0.0 || t < tmin)
            tmin = t;
    }
    return tmin == 0.0 || tmin >= 0x1p-40;
}

bool projection_is_safe(const double* a, const cbb_volume_geometry& g, int z_begin, int z_end,
                        const double cmin[3]) {
    float af[12];
    for (int i = 0; i < 12; ++i) {
        af[i] = (float)a[i];
        if (af[i] == 0.0f && std::signbit(af[i]))
            return false;
    }
    static const int urow[4] = {0, 3, 6, 9}, vrow[4] = {1, 4, 7, 10};
    if (!coordinate_sum_bounded(af, urow, cmin) || !coordinate_sum_bounded(af, vrow, cmin))
        return false;
    const int L = g.edge_voxels;
    const double lo = g.origin_mm;
    const double hi = g.origin_mm + (L - 1) * g.voxel_mm;
    const double zlo = g.origin_mm + z_begin * g.voxel_mm;
    const double zhi = g.origin_mm + (z_end - 1) * g.voxel_mm;
    for (int c = 0; c < 8; ++c) {
        const double wx = (c & 1) ? hi : lo;
        const double wy = (c & 2) ? hi : lo;
        const double wz = (c & 4) ? zhi : zlo;
        const double u = wx * a[0] + wy * a[3] + wz * a[6] + a[9];
        const double v = wx * a[1] + wy * a[4] + wz * a[7] + a[10];
        const double w = wx * a[2] + wy * a[5] + wz * a[8] + a[11];
        const double scale = std::fabs(wx * a[2]) + std::fabs(wy * a[5]) +
                             std::fabs(wz * a[8]) + std::fabs(a[11]);
        if (!(w > 1e-4 * scale) || !(w >= 0x1p-7) || !(w <= 0x1p7))
            return false;
        if (!(std::fabs(u / w) < 1e8) || !(std::fabs(v / w) < 1e8))
            return false;
    }
    return true;
}

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
    dim3 grid((qp + 127) / 128, band.qn, count);
    if (band.qn <= 0 || count <= 0)
        return;
    pack_quads<<<grid, 128, 0, st>>>(raw, W, H, raw_row0, raw_rows, raw_stride,
                                     static_cast<float4*>(packed), qp, band.q0, band.qn, err);
    CK(cudaGetLastError());
    ++g_launches;
}

void launch_pack(const float* raw, int W, int H, int count, void* packed, cudaStream_t st,
                 int* err = nullptr) {
    launch_pack_band(raw, 0, H, (long long)W * H, W, H, count, packed, RowBand::full(H), st, err);
}

void launch_check_finite(const float* v, long long n, int* err, cudaStream_t st) {
    if (n <= 0)
        return;
    const long long blocks = std::min<long long>(148 * 4, (n / 4 + 255) / 256 + 1);
    check_finite<<<(unsigned)blocks, 256, 0, st>>>(v, n, err);
    CK(cudaGetLastError());
    ++g_launches;
}

template <int R, int MODE, bool GUARD, int MINB, int SW = 0, bool CNT = false>
void launch_bp_r(const BpArgs& a, const BpMats& mats, int nz, cudaStream_t st) {
    BpArgs args = a;
    args.nbx = (args.L + kBlockX - 1) / kBlockX;
    args.nby = (args.L + kBlockY - 1) / kBlockY;
    args.nbz = (nz - args.gap + R - 1) / R;
    dim3 block(kBlockX * kBlockY);
    dim3 grid(args.nbx, args.nby, args.nbz);
    if (SW) {
        const long long ns = (long long)((args.nbx + kSX - 1) / kSX) *
                             ((args.nby + kSY - 1) / kSY) * ((args.nbz + kSZ - 1) / kSZ);
        grid = dim3((unsigned)(ns * kSX * kSY * kSZ), 1, 1);
    }
    bp_kernel<R, MODE, GUARD, MINB, SW, CNT><<<grid, block, 0, st>>>(args, mats);
    CK(cudaGetLastError());
    ++g_launches;
}

// Kernel shape variant (tuning experiments; CBB_BP_VARIANT overrides):
// 0 = R 8 voxels/thread, 3 blocks/SM (default, measured best on config 2);
// 1 = R 4, 4 blocks/SM; 2 = R 8, 2 blocks/SM; 3 = R 4 with super-tile order.
int bp_variant() {
    const char* e = std::getenv("CBB_BP_VARIANT");
    return e ? std::atoi(e) : 0;
}

template <int MODE, bool GUARD>
void launch_bp_t(const BpArgs& args, const BpMats& mats, int nz, cudaStream_t st) {
    if (GUARD) // (culling does not run in the guarded kernel: nothing to count)
        return launch_bp_r<kR, MODE, GUARD, 2>(args, mats, nz, st);
    if (args.counters) // statistics requested: the counting instantiation
        return launch_bp_r<8, MODE, GUARD, 3, 0, true>(args, mats, nz, st);
    switch (bp_variant()) {
    case 1: return launch_bp_r<4, MODE, GUARD, 4>(args, mats, nz, st);
    case 2: return launch_bp_r<8, MODE, GUARD, 2>(args, mats, nz, st);
    case 3: return launch_bp_r<4, MODE, GUARD, 4, 1>(args, mats, nz, st);
    default: return launch_bp_r<8, MODE, GUARD, 3>(args, mats, nz, st);
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
    const long long proj_bytes = (long long)qp * b.qn * 16;
    const long long band_shift = (long long)b.q0 * qp * 16;
    BpArgs args;
    args.vol = vol_slab;
    args.proj_bytes = proj_bytes;
    args.L = g.edge_voxels;
    args.z_begin = z_begin;
    args.z_end = z_end;
    args.O = (float)g.origin_mm;
    args.MM = (float)g.voxel_mm;
    args.Wf = (float)W;
    args.Hf = (float)H;
    args.qpitchf = (float)qp;
    args.cell_bias = (float)(kPad * qp + kPad) + 8388608.0f;
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
    for (int first = 0; first < count; first += opt.batch) {
        const int n = std::min(opt.batch, count - first);
        BpMats m;
        bool safe = true;
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
                launch_bp_t<0, false>(args, m, nz, st);
            else
                launch_bp_t<0, true>(args, m, nz, st);
        } else {
            if (safe)
                launch_bp_t<1, false>(args, m, nz, st);
            else
                launch_bp_t<1, true>(args, m, nz, st);
        }
        guarded_launches += safe ? 0 : 1;
    }
    return guarded_launches;
}

// ---------------------------------------------------------------------------
// Device buffer cache: repeated reconstructions (per-projection calls,
// benchmark loops) reuse device buffers instead of paying cudaMalloc/cudaFree
// (~ms for GB-sized slabs) per call. Blocks are reused when the cached block
// is at least the request and at most twice its size.
// ---------------------------------------------------------------------------

class DevicePool {
  public:
    static DevicePool& get() {
        static DevicePool p;
        return p;
    }

    // A cached block for the request, or nullptr (never allocates).
    void* take_cached(int device, size_t bytes) {
        bytes = std::max<size_t>(bytes, 256);
        std::lock_guard<std::mutex> lk(mu_);
        auto& fl = free_[device];
        auto it = fl.lower_bound(bytes);
        if (it != fl.end() && it->first <= 2 * bytes) {
            void* p = it->second;
            sizes_[p] = it->first;
            fl.erase(it);
            return p;
        }
        return nullptr;
    }

    void* alloc(int device, size_t bytes) {
        bytes = std::max<size_t>(bytes, 256);
        if (void* c = take_cached(device, bytes))
            return c;
        void* p = nullptr;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            trim(device);
            e = cudaMalloc(&p, bytes);
        }
        check_cuda(e, "cudaMalloc");
        std::lock_guard<std::mutex> lk(mu_);
        sizes_[p] = bytes;
        return p;
    }

    void release(int device, void* p) {
        if (!p)
            return;
        std::lock_guard<std::mutex> lk(mu_);
        auto it = sizes_.find(p);
        if (it == sizes_.end())
            return;
        free_[device].emplace(it->second, p);
        sizes_.erase(it);
    }

    void trim(int device) {
        std::lock_guard<std::mutex> lk(mu_);
        for (auto& kv : free_[device])
            cudaFree(kv.second);
        free_[device].clear();
    }
    void trim_all() {
        std::vector<int> devs;
        {
            std::lock_guard<std::mutex> lk(mu_);
            for (auto& kv : free_)
                devs.push_back(kv.first);
        }
        for (int d : devs) {
            int cur = 0;
            cudaGetDevice(&cur);
            cudaSetDevice(d);
            trim(d);
            cudaSetDevice(cur);
        }
    }

  private:
    std::mutex mu_;
    std::map<int, std::multimap<size_t, void*>> free_;
    std::map<void*, size_t> sizes_;
};

// Pinned host staging cache: cudaHostAlloc pins pages at ~4 GB/s (measured:
// 2 GiB in 565 ms), which for two 153 MB staging slots would cost ~80 ms per
// cbb_reconstruct call; blocks are kept for the next call (at most 6, reused
// when at least the request and at most twice its size).
class HostPool {
  public:
    static HostPool& get() {
        static HostPool* p = new HostPool; // never destroyed: no CUDA calls at exit
        return *p;
    }
    float* alloc(size_t bytes) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            auto it = free_.lower_bound(bytes);
            if (it != free_.end() && it->first <= 2 * bytes) {
                void* p = it->second;
                sizes_[p] = it->first;
                free_.erase(it);
                return static_cast<float*>(p);
            }
        }
        void* p = nullptr;
        CK(cudaHostAlloc(&p, bytes, cudaHostAllocPortable));
        std::lock_guard<std::mutex> lk(mu_);
        sizes_[p] = bytes;
        return static_cast<float*>(p);
    }
    void release(void* p) {
        if (!p)
            return;
        std::lock_guard<std::mutex> lk(mu_);
        auto it = sizes_.find(p);
        if (it == sizes_.end())
            return;
        free_.emplace(it->second, p);
        sizes_.erase(it);
        while (free_.size() > 6) { // drop the smallest
            cudaFreeHost(free_.begin()->second);
            free_.erase(free_.begin());
        }
    }
    void trim() {
        std::lock_guard<std::mutex> lk(mu_);
        for (auto& kv : free_)
            cudaFreeHost(kv.second);
        free_.clear();
    }

  private:
    std::mutex mu_;
    std::multimap<size_t, void*> free_;
    std::map<void*, size_t> sizes_;
};

// ---------------------------------------------------------------------------
// Per-device worker: slab volume, raw/packed double buffers, streams, events.
// ---------------------------------------------------------------------------

struct Worker {
    int device = 0;
    int z_begin = 0, z_end = 0;
    float* d_vol = nullptr;
    float* d_raw[2] = {nullptr, nullptr};
    void* d_packed[2] = {nullptr, nullptr};
    int* d_err = nullptr;
    cudaStream_t copy = nullptr, compute = nullptr;
    cudaEvent_t h2d_done[2] = {}, raw_free[2] = {};
    cudaEvent_t k_beg = nullptr, k_end = nullptr, c_beg = nullptr, c_end = nullptr;
    double kernel_s = 0.0, h2d_s = 0.0, d2h_s = 0.0;
    uint64_t guarded = 0;
    bool started = false;
    bool k_end_set = false; // k_end already recorded (resident tail)
    // resident mode: every packed projection stays on the device; the head
    // planes [z_begin, tail_lo) + [tail_hi, z_end) are updated while the
    // batches stream in, the tail [tail_lo, tail_hi) afterwards while the
    // head is copied back
    void* d_packed_all = nullptr;
    int tail_lo = 0, tail_hi = 0;
    cudaEvent_t head_done = nullptr, tail_done = nullptr;
    // detector rows this worker holds / packs (RowBand::full unless set_bands)
    RowBand band;
    size_t pk_bytes = 0;               // packed bytes per projection (band rows)
    cudaEvent_t src_ready[2] = {};     // as root: raw slot filtered, peers may copy
    cudaEvent_t xfer_ev[2] = {};       // ChunkedXfer chunk events (copy stream)
    unsigned long long* d_counters = nullptr; // kCounterSlots culled-update counters
    bool count_culled = false;

    ~Worker() {
        if (!copy)
            return;
        cudaSetDevice(device);
        cudaStreamSynchronize(copy);
        cudaStreamSynchronize(compute);
        auto& pool = DevicePool::get();
        pool.release(device, d_vol);
        for (int i = 0; i < 2; ++i) {
            pool.release(device, d_raw[i]);
            pool.release(device, d_packed[i]);
            cudaEventDestroy(h2d_done[i]);
            cudaEventDestroy(raw_free[i]);
            cudaEventDestroy(src_ready[i]);
            cudaEventDestroy(xfer_ev[i]);
        }
        pool.release(device, d_err);
        pool.release(device, d_counters);
        pool.release(device, d_packed_all);
        if (head_done)
            cudaEventDestroy(head_done);
        if (tail_done)
            cudaEventDestroy(tail_done);
        cudaEventDestroy(k_beg);
        cudaEventDestroy(k_end);
        cudaEventDestroy(c_beg);
        cudaEventDestroy(c_end);
        cudaStreamDestroy(copy);
        cudaStreamDestroy(compute);
    }
};

// Host copy into pinned staging, split over a few threads for large blocks
// (a single thread moves ~5-10 GB/s, below the PCIe H2D rate).
void parallel_memcpy(void* dst, const void* src, size_t bytes) {
    const size_t kChunk = size_t(8) << 20;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t nt = std::min<size_t>(std::min<size_t>(hw, 8), (bytes + kChunk - 1) / kChunk);
    if (nt <= 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    std::vector<std::thread> pool;
    const size_t per = (bytes + nt - 1) / nt;
    for (size_t t = 0; t < nt; ++t) {
        const size_t off = t * per;
        if (off >= bytes)
            break;
        const size_t len = std::min(per, bytes - off);
        pool.emplace_back([=] {
            std::memcpy(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, len);
        });
    }
    for (auto& th : pool)
        th.join();
}

bool is_pinned(const void* p) {
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return attr.type == cudaMemoryTypeHost;
}

// Host <-> device copies of large blocks for pageable host memory: a plain
// cudaMemcpyAsync from/to pageable memory is synchronous and staged by the
// driver at a fraction of the link rate. Here 64 MB chunks go through two
// pinned buffers, the host copies (parallel_memcpy) overlapping the DMA of
// the neighbouring chunk. Pinned memory is copied directly (asynchronously).
// ev: two events of the stream's device.
struct ChunkedXfer {
    static constexpr size_t kChunk = size_t(64) << 20;
    float* buf[2] = {nullptr, nullptr};
    ~ChunkedXfer() {
        for (auto b : buf)
            HostPool::get().release(b);
    }
    void ensure() {
        for (auto& b : buf)
            if (!b)
                b = HostPool::get().alloc(kChunk);
    }
    // returns after the last chunk left the pageable source
    void upload(void* dst, const void* src, size_t bytes, cudaStream_t st, cudaEvent_t ev[2]) {
        if (bytes == 0)
            return;
        if (is_pinned(src)) {
            CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
            return;
        }
        ensure();
        int k = 0;
        for (size_t off = 0; off < bytes; off += kChunk, k ^= 1) {
            const size_t len = std::min(kChunk, bytes - off);
            CK(cudaEventSynchronize(ev[k])); // buf[k]'s previous DMA finished
            parallel_memcpy(buf[k], static_cast<const char*>(src) + off, len);
            CK(cudaMemcpyAsync(static_cast<char*>(dst) + off, buf[k], len,
                               cudaMemcpyHostToDevice, st));
            CK(cudaEventRecord(ev[k], st));
        }
    }
    // pageable dst: blocks until all bytes arrived; pinned dst: asynchronous
    void download(void* dst, const void* src, size_t bytes, cudaStream_t st, cudaEvent_t ev[2]) {
        if (bytes == 0)
            return;
        if (is_pinned(dst)) {
            CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
            return;
        }
        ensure();
        const size_t nchunks = (bytes + kChunk - 1) / kChunk;
        auto issue = [&](size_t c) {
            const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
            CK(cudaMemcpyAsync(buf[c & 1], static_cast<const char*>(src) + off, len,
                               cudaMemcpyDeviceToHost, st));
            CK(cudaEventRecord(ev[c & 1], st));
        };
        issue(0);
        for (size_t c = 0; c < nchunks; ++c) {
            if (c + 1 < nchunks)
                issue(c + 1);
            CK(cudaEventSynchronize(ev[c & 1]));
            const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
            parallel_memcpy(static_cast<char*>(dst) + off, buf[c & 1], len);
        }
    }
};

double elapsed_s(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.0f;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms * 1e-3;
}

struct Pipeline {
    cbb_volume_geometry g{};
    int W = 0, H = 0;
    cbb_options opt{};
    std::vector<std::unique_ptr<Worker>> workers;
    float* h_stage[2] = {nullptr, nullptr}; // pinned staging (batch x H x W)
    ChunkedXfer xfer;                       // volume up/download for pageable buffers
    int stage_fill = 0;                     // projections staged in the current slot
    int slot = 0;                           // current staging / ring slot
    std::vector<double> stage_mats;         // matrices of the staged batch
    uint64_t submitted = 0;
    uint64_t nbatch = 0;   // batches issued (root = nbatch mod workers)
    size_t raw_bytes_per_proj = 0;
    size_t packed_bytes_per_proj = 0;
    bool resident = false;         // see Worker::d_packed_all
    int resident_count = 0;
    std::vector<double> all_mats;  // resident mode: every matrix, for the tail pass
    const double* est_mats = nullptr; // matrices for choose_tails (else the first batch)
    int est_n = 0;

    // Resident mode for a stack of known size: when every packed projection
    // fits in device memory (with 2 GB to spare), keep them all so a dense
    // tail of each slab (choose_tails) can be back-projected after the stream
    // ends while the rest is already copied to the host (hides most of the
    // D2H).
    void enable_resident(int count) {
        if (std::getenv("CBB_NO_RESIDENT"))
            return;
        for (auto& w : workers)
            if (w->z_end - w->z_begin < 16)
                return;
        std::vector<void*> blocks;
        for (auto& w : workers) {
            const size_t need = w->pk_bytes * (size_t)count;
            CK(cudaSetDevice(w->device));
            void* p = DevicePool::get().take_cached(w->device, need);
            if (!p) {
                size_t free_b = 0, total_b = 0;
                CK(cudaMemGetInfo(&free_b, &total_b));
                if (free_b >= need + (size_t(2) << 30))
                    p = DevicePool::get().alloc(w->device, need);
                else if (std::getenv("CBB_TRACE"))
                    std::fprintf(stderr, "cbb: resident off, need %zu free %zu\n", need, free_b);
            }
            if (!p) {
                for (size_t i = 0; i < blocks.size(); ++i)
                    DevicePool::get().release(workers[i]->device, blocks[i]);
                return;
            }
            blocks.push_back(p);
        }
        for (size_t i = 0; i < workers.size(); ++i) {
            auto& w = workers[i];
            CK(cudaSetDevice(w->device));
            w->d_packed_all = blocks[i];
            if (!w->head_done) {
                CK(cudaEventCreate(&w->head_done));
                CK(cudaEventCreateWithFlags(&w->tail_done, cudaEventDisableTiming));
            }
        }
        resident = true;
        resident_count = count;
        all_mats.assign(12 * (size_t)count, 0.0);
    }

    // Picks each worker's tail: the contiguous run of 8-plane groups with the
    // fewest planes that holds ~kTailFrac of the slab's estimated work. Work
    // per group = fraction of sampled (x, y, projection) positions that land
    // on the detector (the rest is culled warp by warp) + a fixed overhead,
    // sampled on a 16 x 16 grid at the group's centre plane for up to 8 of
    // the given projections. A dense tail keeps its D2H short while its
    // compute hides the head's D2H.
    void choose_tails(const double* mats, int n) {
        double frac = 0.12;
        if (const char* e = std::getenv("CBB_TAIL_FRAC"))
            frac = std::atof(e);
        const int L = g.edge_voxels, S = 16, NP = std::min(n, 8);
        for (auto& w : workers) {
            std::vector<double> gw;
            std::vector<int> gz;
            for (int z = w->z_begin; z < w->z_end; z += 8) {
                const int pz = std::min(8, w->z_end - z);
                const double zc = g.origin_mm + (z + (pz - 1) * 0.5) * g.voxel_mm;
                int on = 0;
                for (int k = 0; k < NP; ++k) {
                    const double* a = mats + 12 * (size_t)((long long)k * n / NP);
                    for (int j = 0; j < S; ++j)
                        for (int i = 0; i < S; ++i) {
                            const double x = g.origin_mm + (L - 1) * (i / (S - 1.0)) * g.voxel_mm;
                            const double y = g.origin_mm + (L - 1) * (j / (S - 1.0)) * g.voxel_mm;
                            const double u = a[0] * x + a[3] * y + a[6] * zc + a[9];
                            const double v = a[1] * x + a[4] * y + a[7] * zc + a[10];
                            const double ww = a[2] * x + a[5] * y + a[8] * zc + a[11];
                            const double ix = u / ww, iy = v / ww;
                            on += ix > -2 && ix < W && iy > -2 && iy < H;
                        }
                }
                gw.push_back(pz * ((double)on / (NP * S * S) + 0.05));
                gz.push_back(z);
            }
            gz.push_back(w->z_end);
            const int G = (int)gw.size();
            double total = 0.0;
            for (double x : gw)
                total += x;
            int best_i = G - 1, best_j = G, best_planes = 1 << 30;
            for (int i = 0; i < G; ++i) {
                double s = 0.0;
                for (int j = i; j < G; ++j) {
                    s += gw[j];
                    if (s >= frac * total) {
                        const int planes = gz[j + 1] - gz[i];
                        if (planes < best_planes && !(i == 0 && j == G - 1)) {
                            best_planes = planes;
                            best_i = i;
                            best_j = j + 1;
                        }
                        break;
                    }
                }
            }
            w->tail_lo = gz[best_i];
            w->tail_hi = gz[best_j];
            if (std::getenv("CBB_TRACE"))
                std::fprintf(stderr, "cbb: device %d slab [%d, %d) tail [%d, %d)\n", w->device,
                             w->z_begin, w->z_end, w->tail_lo, w->tail_hi);
        }
    }

    ~Pipeline() {
        workers.clear();
        for (int i = 0; i < 2; ++i)
            HostPool::get().release(h_stage[i]);
    }

    void init(const cbb_volume_geometry& geom, int width, int height, const cbb_options& o,
              const float* initial_volume) {
        g = geom;
        W = width;
        H = height;
        opt = o;
        int ndev = 0;
        CK(cudaGetDeviceCount(&ndev));
        if (ndev < 1)
            fail(CBB_ERR_INTERNAL, "no CUDA device available");
        if (opt.slab_end > g.edge_voxels)
            fail(CBB_ERR_INVALID, "options: slab_end %d beyond L = %d", opt.slab_end,
                 g.edge_voxels);
        const int s0 = opt.slab_end ? opt.slab_begin : 0;
        const int s1 = opt.slab_end ? opt.slab_end : g.edge_voxels;
        int ng = opt.num_gpus > 0 ? opt.num_gpus : ndev;
        ng = std::min(ng, s1 - s0);
        if (!opt.device_ids && ng > ndev)
            fail(CBB_ERR_INVALID, "options: num_gpus %d exceeds %d visible devices", ng, ndev);
        raw_bytes_per_proj = (size_t)W * H * sizeof(float);
        packed_bytes_per_proj = (size_t)quad_pitch_cells(W) * quad_rows(H) * 16;
        const int L = g.edge_voxels;
        const size_t plane = (size_t)L * L;
        for (int i = 0; i < ng; ++i) {
            auto w = std::make_unique<Worker>();
            w->device = opt.device_ids ? opt.device_ids[i] : i;
            if (w->device < 0 || w->device >= ndev)
                fail(CBB_ERR_INVALID, "options: device id %d not visible", w->device);
            w->z_begin = s0 + (int)((long long)(s1 - s0) * i / ng);
            w->z_end = s0 + (int)((long long)(s1 - s0) * (i + 1) / ng);
            CK(cudaSetDevice(w->device));
            CK(cudaStreamCreateWithFlags(&w->copy, cudaStreamNonBlocking));
            CK(cudaStreamCreateWithFlags(&w->compute, cudaStreamNonBlocking));
            for (int s = 0; s < 2; ++s) {
                CK(cudaEventCreateWithFlags(&w->h2d_done[s], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&w->raw_free[s], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&w->src_ready[s], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&w->xfer_ev[s], cudaEventDisableTiming));
                w->d_raw[s] = static_cast<float*>(
                    DevicePool::get().alloc(w->device, raw_bytes_per_proj * opt.batch));
                w->d_packed[s] = DevicePool::get().alloc(w->device, packed_bytes_per_proj * opt.batch);
            }
            w->band = RowBand::full(H);
            w->pk_bytes = packed_bytes_per_proj;
            CK(cudaEventCreate(&w->k_beg));
            CK(cudaEventCreate(&w->k_end));
            CK(cudaEventCreate(&w->c_beg));
            CK(cudaEventCreate(&w->c_end));
            const size_t slab = plane * (w->z_end - w->z_begin);
            w->d_vol = static_cast<float*>(
                DevicePool::get().alloc(w->device, std::max<size_t>(slab, 1) * sizeof(float)));
            w->d_err = static_cast<int*>(DevicePool::get().alloc(w->device, sizeof(int)));
            CK(cudaMemsetAsync(w->d_err, 0, sizeof(int), w->compute));
            const size_t cbytes = sizeof(unsigned long long) * kCounterSlots;
            w->d_counters = static_cast<unsigned long long*>(
                DevicePool::get().alloc(w->device, cbytes));
            CK(cudaMemsetAsync(w->d_counters, 0, cbytes, w->compute));
            w->count_culled = opt.count_culled != 0;
            CK(cudaEventRecord(w->c_beg, w->copy));
            if (initial_volume && !opt.volume_is_zero)
                xfer.upload(w->d_vol, initial_volume + plane * w->z_begin, slab * sizeof(float),
                            w->copy, w->xfer_ev);
            else
                CK(cudaMemsetAsync(w->d_vol, 0, slab * sizeof(float), w->copy));
            CK(cudaEventRecord(w->c_end, w->copy));
            CK(cudaStreamWaitEvent(w->compute, w->c_end, 0));
            workers.push_back(std::move(w));
        }
        stage_mats.assign(12 * (size_t)opt.batch, 0.0);
        // band copies go straight over NVLink where the devices allow it
        for (auto& a : workers)
            for (auto& b : workers) {
                int can = 0;
                if (a->device == b->device ||
                    cudaDeviceCanAccessPeer(&can, b->device, a->device) != cudaSuccess || !can)
                    continue;
                CK(cudaSetDevice(b->device));
                const cudaError_t e = cudaDeviceEnablePeerAccess(a->device, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled)
                    cudaGetLastError();
                else
                    CK(e);
            }
        for (auto& w : workers) {
            CK(cudaSetDevice(w->device));
            CK(cudaEventSynchronize(w->c_end));
            w->h2d_s += elapsed_s(w->c_beg, w->c_end);
        }
    }

    // Issues one batch of n projections from host memory src (pinned or not)
    // to every worker. The caller guarantees src stays valid until the
    // corresponding h2d_done events complete (wait_slot).
    void issue(const float* src, const double* mats, int n) {
        const size_t bytes = raw_bytes_per_proj * n;
        if (resident && submitted == 0) {
            const auto t0 = std::chrono::steady_clock::now();
            choose_tails(est_mats ? est_mats : mats, est_mats ? est_n : n);
            if (std::getenv("CBB_TRACE"))
                std::fprintf(stderr, "cbb: choose_tails %.2f ms\n",
                             std::chrono::duration<double, std::milli>(
                                 std::chrono::steady_clock::now() - t0).count());
        }
        // Batch k is uploaded once, by the root worker k mod G, and each
        // other worker copies its row band from the root's raw slot (peer
        // copy over NVLink; a plain device copy when both are one device).
        const int G = (int)workers.size();
        Worker& root = *workers[nbatch % G];
        // raw[slot] of worker w may still be read by its own pack of batch
        // k-2 and, if w was that batch's root, by the other workers' band copies
        for (auto& w : workers) {
            CK(cudaSetDevice(w->device));
            CK(cudaStreamWaitEvent(w->copy, w->raw_free[slot], 0));
            for (auto& o : workers)
                if (o != w)
                    CK(cudaStreamWaitEvent(w->copy, o->h2d_done[slot], 0));
        }
        CK(cudaSetDevice(root.device));
        CK(cudaMemcpyAsync(root.d_raw[slot], src, bytes, cudaMemcpyHostToDevice, root.copy));
        CK(cudaEventRecord(root.h2d_done[slot], root.copy));
        CK(cudaStreamWaitEvent(root.compute, root.h2d_done[slot], 0));
        start_timing(root);
        // the root sees the whole batch: it checks the pixels its band skips
        if (!root.band.is_full(H))
            launch_check_finite(root.d_raw[slot], (long long)n * W * H, root.d_err, root.compute);
        cudaEvent_t ready = root.h2d_done[slot];
        if (opt.ramp_filter) {
            ramp_filter_device(root.d_raw[slot], root.d_raw[slot], W, H, n, opt.filter_pixel_mm,
                               root.compute);
            CK(cudaEventRecord(root.src_ready[slot], root.compute));
            ready = root.src_ready[slot];
        }
        for (auto& w : workers) {
            if (w.get() == &root)
                continue;
            CK(cudaSetDevice(w->device));
            CK(cudaStreamWaitEvent(w->copy, ready, 0));
            copy_band(root, *w, slot, n);
            CK(cudaEventRecord(w->h2d_done[slot], w->copy));
            CK(cudaStreamWaitEvent(w->compute, w->h2d_done[slot], 0));
            start_timing(*w);
        }
        for (auto& w : workers) {
            CK(cudaSetDevice(w->device));
            void* packed = resident ? static_cast<char*>(w->d_packed_all) + w->pk_bytes * submitted
                                    : w->d_packed[slot];
            if (w.get() == &root)
                launch_pack_band(w->d_raw[slot], 0, H, (long long)W * H, W, H, n, packed, w->band,
                                 w->compute, w->d_err);
            else
                launch_pack_band(w->d_raw[slot], w->band.r0, w->band.rn,
                                 (long long)w->band.rn * W, W, H, n, packed, w->band, w->compute,
                                 w->d_err);
            CK(cudaEventRecord(w->raw_free[slot], w->compute));
            // resident: the head, i.e. the slab minus the tail planes
            w->guarded += launch_backproject(w->d_vol, g, w->z_begin, w->z_end, packed, W, H, n,
                                             mats, opt, w->d_err, w->compute,
                                             resident ? w->tail_lo : 0, resident ? w->tail_hi : 0,
                                             &w->band, w->count_culled ? w->d_counters : nullptr);
        }
        ++nbatch;
        if (resident)
            std::memcpy(all_mats.data() + 12 * submitted, mats, 12 * sizeof(double) * n);
        submitted += n;
        slot ^= 1;
    }

    void start_timing(Worker& w) {
        if (!w.started) {
            CK(cudaEventRecord(w.k_beg, w.compute));
            w.started = true;
        }
    }

    // Rows [band.r0, band.r0 + band.rn) of the batch's n projections, from the
    // root's full raw slot to w's band slot (projection stride rn * W), one
    // strided peer copy on w's copy stream.
    void copy_band(const Worker& root, Worker& w, int s, int n) {
        const RowBand& b = w.band;
        if (b.rn <= 0)
            return;
        cudaMemcpy3DPeerParms p = {};
        const size_t row_bytes = (size_t)b.rn * W * sizeof(float);
        p.srcPtr = make_cudaPitchedPtr(root.d_raw[s] + (size_t)b.r0 * W, raw_bytes_per_proj,
                                       row_bytes, n);
        p.srcDevice = root.device;
        p.dstPtr = make_cudaPitchedPtr(w.d_raw[s], row_bytes, row_bytes, n);
        p.dstDevice = w.device;
        p.extent = make_cudaExtent(row_bytes, n, 1);
        CK(cudaMemcpy3DPeerAsync(&p, w.copy));
    }

    RowBand band_for(const Worker& w, const double* mats, int count) const {
        if (std::getenv("CBB_NO_BANDS"))
            return RowBand::full(H);
        return row_band_for(g, W, H, w.z_begin, w.z_end, mats, count);
    }

    // Sets every worker's row band for a stack whose matrices are all known.
    void set_bands(const double* mats, int count) {
        for (auto& w : workers) {
            w->band = band_for(*w, mats, count);
            w->pk_bytes = (size_t)quad_pitch_cells(W) * w->band.qn * 16;
            if (std::getenv("CBB_TRACE"))
                std::fprintf(stderr, "cbb: device %d slab [%d, %d) rows [%d, %d) cells %d of %d\n",
                             w->device, w->z_begin, w->z_end, w->band.r0,
                             w->band.r0 + w->band.rn, w->band.qn, quad_rows(H));
        }
    }

    // Host-side proof that every batch of the tail pass runs unguarded (no
    // possible w == 0 error), so the head may be copied out before the tail
    // is computed.
    bool tail_is_safe(const Worker& w) const {
        const float Of = (float)g.origin_mm, MMf = (float)g.voxel_mm;
        const double cxy = min_nonzero_coord(Of, MMf, 0, g.edge_voxels);
        const double cmin[3] = {cxy, cxy, min_nonzero_coord(Of, MMf, w.tail_lo, w.tail_hi)};
        for (int p = 0; p < resident_count; ++p)
            if (!projection_is_safe(all_mats.data() + 12 * (size_t)p, g, w.tail_lo, w.tail_hi,
                                    cmin))
                return false;
        return true;
    }

    // Blocks until no device still reads the staging slot s.
    void wait_slot(int s) {
        for (auto& w : workers) {
            CK(cudaSetDevice(w->device));
            CK(cudaEventSynchronize(w->h2d_done[s]));
        }
    }

    // Pinned staging for pageable sources, allocated on first use only.
    void ensure_staging() {
        for (int s = 0; s < 2; ++s)
            if (!h_stage[s])
                h_stage[s] = HostPool::get().alloc(raw_bytes_per_proj * opt.batch);
    }

    void stage_one(const float* img, const double* m) {
        ensure_staging();
        if (stage_fill == 0)
            wait_slot(slot);
        std::memcpy(h_stage[slot] + (size_t)stage_fill * W * H, img, raw_bytes_per_proj);
        std::memcpy(stage_mats.data() + 12 * (size_t)stage_fill, m, 12 * sizeof(double));
        if (++stage_fill == opt.batch)
            flush();
    }

    void flush() {
        if (stage_fill == 0)
            return;
        issue(h_stage[slot], stage_mats.data(), stage_fill);
        stage_fill = 0;
    }

    // Size of the batch starting at projection `first` of a stream: 4, 4, 8,
    // 16, ... up to opt.batch, so the first back-projection starts after a
    // small upload instead of a full batch (pipeline fill). Batch boundaries
    // do not change any result: each voxel still accumulates the projections
    // one by one in stack order.
    int batch_at(int first, int count) const {
        return std::min({opt.batch, std::max(4, first), count - first});
    }

    // Whole-stack submission straight from the caller's buffer: pinned
    // buffers are copied asynchronously in place, pageable ones are staged
    // through the pinned double buffer.
    // First submission of a stack whose matrices are all known: row bands,
    // resident mode, tail estimate.
    void begin_stack(const double* mats, int count) {
        if (submitted != 0)
            return;
        const auto t0 = std::chrono::steady_clock::now();
        set_bands(mats, count);
        enable_resident(count);
        if (std::getenv("CBB_TRACE"))
            std::fprintf(stderr, "cbb: enable_resident %.2f ms\n",
                         std::chrono::duration<double, std::milli>(
                             std::chrono::steady_clock::now() - t0).count());
        est_mats = mats;
        est_n = count;
    }

    void submit_stack(const float* imgs, const double* mats, int count) {
        begin_stack(mats, count);
        cudaPointerAttributes attr;
        bool pinned = false;
        if (cudaPointerGetAttributes(&attr, imgs) == cudaSuccess)
            pinned = attr.type == cudaMemoryTypeHost;
        else
            cudaGetLastError();
        for (int first = 0, n = 0; first < count; first += n) {
            n = batch_at(first, count);
            const float* src = imgs + (size_t)first * W * H;
            if (pinned) {
                issue(src, mats + 12 * (size_t)first, n);
            } else {
                ensure_staging();
                wait_slot(slot);
                parallel_memcpy(h_stage[slot], src, raw_bytes_per_proj * n);
                issue(h_stage[slot], mats + 12 * (size_t)first, n);
            }
        }
    }

    // Projections in separate host buffers (the reference's ProjectionStack):
    // each batch is gathered into a pinned staging slot by a few threads
    // (whole projections per thread) while the devices process the previous
    // batch.
    void submit_images(const float* const* imgs, const double* mats, int count) {
        begin_stack(mats, count);
        ensure_staging();
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        for (int first = 0, n = 0; first < count; first += n) {
            n = batch_at(first, count);
            wait_slot(slot);
            float* dst = h_stage[slot];
            const int nt = (int)std::min<unsigned>(std::min(8u, hw), (unsigned)n);
            std::vector<std::thread> pool;
            for (int t = 0; t < nt; ++t)
                pool.emplace_back([&, t] {
                    for (int j = t; j < n; j += nt)
                        std::memcpy(dst + (size_t)j * W * H, imgs[first + j], raw_bytes_per_proj);
                });
            for (auto& th : pool)
                th.join();
            issue(dst, mats + 12 * (size_t)first, n);
        }
    }

    // Streams the projection records of an open CBPS file (proj/src/dataset.cpp:
    // 155-212 layout: per record 12 little-endian f64 then W*H f32) straight
    // into the pinned staging slots: record i's image goes to its place in
    // the batch, its matrix to a small host array. Reads of batch k+1 run on
    // the host while the devices process batch k; each batch is read by a
    // few threads with pread.
    void submit_file(int fd, int count, uint64_t header_bytes, uint64_t rec_bytes) {
        if (submitted == 0)
            enable_resident(count);
        ensure_staging();
        std::vector<double> mats(12 * (size_t)opt.batch);
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const int nt = (int)std::min<unsigned>(8, hw);
        // the records are copied out of a read-only mapping of the file
        // (page-cache pages mapped, no per-call kernel copy); pread when the
        // file cannot be mapped
        const uint64_t file_bytes = header_bytes + rec_bytes * (uint64_t)count;
        const char* map = nullptr;
        if (!std::getenv("CBB_FILE_PREAD")) {
            void* m = ::mmap(nullptr, file_bytes, PROT_READ, MAP_SHARED, fd, 0);
            if (m != MAP_FAILED) {
                map = static_cast<const char*>(m);
                ::madvise(m, file_bytes, MADV_SEQUENTIAL);
            }
        }
        struct Unmap {
            const char* p;
            uint64_t n;
            ~Unmap() {
                if (p)
                    ::munmap(const_cast<char*>(p), n);
            }
        } unmap{map, file_bytes};
        double t_wait = 0, t_read = 0, t_issue = 0;
        auto now = [] { return std::chrono::steady_clock::now(); };
        auto ms_since = [](std::chrono::steady_clock::time_point t) {
            return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t)
                .count();
        };
        for (int first = 0, n = 0; first < count; first += n) {
            n = batch_at(first, count);
            auto t0 = now();
            wait_slot(slot);
            t_wait += ms_since(t0);
            t0 = now();
            float* dst = h_stage[slot];
            std::vector<std::thread> pool;
            std::vector<int> bad(nt, 0);
            for (int t = 0; t < nt; ++t)
                pool.emplace_back([&, t] {
                    for (int j = t; j < n; j += nt) {
                        const uint64_t off = header_bytes + rec_bytes * (uint64_t)(first + j);
                        if (map) {
                            std::memcpy(mats.data() + 12 * (size_t)j, map + off, 96);
                            std::memcpy(dst + (size_t)j * W * H, map + off + 96, rec_bytes - 96);
                        } else if (!pread_all(fd, mats.data() + 12 * (size_t)j, 96, off) ||
                                   !pread_all(fd, dst + (size_t)j * W * H, rec_bytes - 96,
                                              off + 96)) {
                            bad[t] = 1;
                        }
                    }
                });
            for (auto& th : pool)
                th.join();
            for (int b : bad)
                if (b)
                    fail(CBB_ERR_TRUNCATED, "file ends inside projection intensities");
            validate_matrices(mats.data(), n);
            t_read += ms_since(t0);
            t0 = now();
            issue(dst, mats.data(), n);
            t_issue += ms_since(t0);
        }
        if (std::getenv("CBB_TRACE"))
            std::fprintf(stderr, "cbb: file stream: wait %.1f ms, read %.1f ms, issue %.1f ms\n",
                         t_wait, t_read, t_issue);
    }

    static bool pread_all(int fd, void* buf, uint64_t bytes, uint64_t off) {
        char* p = static_cast<char*>(buf);
        while (bytes) {
            const ssize_t r = ::pread(fd, p, bytes, (off_t)off);
            if (r <= 0)
                return false;
            p += r;
            off += (uint64_t)r;
            bytes -= (uint64_t)r;
        }
        return true;
    }

    // Waits for all work, checks the w == 0 flag, downloads slabs into vol_out.
    // Synchronizes every worker's compute stream and raises the first error
    // the kernels flagged (nothing has been written to the host yet).
    void check_errors(bool close_timing) {
        int err_any = 0;
        for (auto& w : workers) {
            CK(cudaSetDevice(w->device));
            if (close_timing && w->started && !w->k_end_set)
                CK(cudaEventRecord(w->k_end, w->compute));
            w->k_end_set = false;
            CK(cudaStreamSynchronize(w->compute));
            if (close_timing && w->started) {
                w->kernel_s += elapsed_s(w->k_beg, w->k_end);
                w->started = false;
            }
            int e = 0;
            CK(cudaMemcpy(&e, w->d_err, sizeof(int), cudaMemcpyDeviceToHost));
            err_any |= e;
        }
        if (err_any & 2) // ProjectionImage::validate (proj/src/dataset.cpp:123-129)
            fail(CBB_ERR_INVALID, "ProjectionImage contains non-finite values");
        if (err_any & 1)
            fail(CBB_ERR_GEOMETRY, "backprojection hit a voxel with w == 0");
    }

    // Waits for all work, checks the error flags, downloads slabs into vol_out.
    void finish(float* vol_out) {
        flush();
        const size_t plane = (size_t)g.edge_voxels * g.edge_voxels;
        if (resident) {
            finish_resident(vol_out);
            return;
        }
        check_errors(true);
        for (auto& w : workers) {
            CK(cudaSetDevice(w->device));
            const size_t slab = plane * (w->z_end - w->z_begin);
            CK(cudaEventRecord(w->c_beg, w->copy));
            xfer.download(vol_out + plane * w->z_begin, w->d_vol, slab * sizeof(float), w->copy,
                          w->xfer_ev);
            CK(cudaEventRecord(w->c_end, w->copy));
        }
        for (auto& w : workers) {
            CK(cudaSetDevice(w->device));
            CK(cudaEventSynchronize(w->c_end));
            w->d2h_s += elapsed_s(w->c_beg, w->c_end);
        }
    }

    // Resident mode: the head planes are complete once the stream has been
    // consumed; the tail planes are back-projected from the resident packed
    // projections while the head is copied to the host (copy stream). The
    // head is released early only when no tail batch can raise an error
    // (tail_is_safe, no guarded head batch); otherwise everything is checked
    // before any byte reaches vol_out.
    void finish_resident(float* vol_out) {
        const size_t plane = (size_t)g.edge_voxels * g.edge_voxels;
        check_errors(false);
        bool overlap = true;
        for (auto& w : workers)
            overlap = overlap && w->guarded == 0 && tail_is_safe(*w);
        const bool trace = std::getenv("CBB_TRACE") != nullptr;
        cudaEvent_t t_tail = nullptr;
        auto d2h = [&](Worker& w, int z0, int z1) {
            if (z1 > z0)
                xfer.download(vol_out + plane * z0, w.d_vol + plane * (z0 - w.z_begin),
                              plane * (z1 - z0) * sizeof(float), w.copy, w.xfer_ev);
        };
        for (auto& w : workers) {
            CK(cudaSetDevice(w->device));
            if (trace && w == workers.front()) {
                CK(cudaEventCreate(&t_tail));
                CK(cudaEventRecord(t_tail, w->compute));
            }
            w->guarded += launch_backproject(
                w->d_vol + plane * (w->tail_lo - w->z_begin), g, w->tail_lo, w->tail_hi,
                w->d_packed_all, W, H, resident_count, all_mats.data(), opt, w->d_err,
                w->compute, 0, 0, &w->band, w->count_culled ? w->d_counters : nullptr);
            CK(cudaEventRecord(w->tail_done, w->compute));
            if (w->started) { // kernel time ends with the tail, not the downloads
                CK(cudaEventRecord(w->k_end, w->compute));
                w->k_end_set = true;
            }
        }
        if (overlap) {
            // the tail runs on the compute streams (launched above) while the
            // head is copied out; then the tail (no error can arise in it:
            // tail_is_safe). Downloads into pageable memory block this
            // thread chunk by chunk, the tail kernels keep running.
            for (auto& w : workers) {
                CK(cudaSetDevice(w->device));
                CK(cudaEventRecord(w->c_beg, w->copy));
                d2h(*w, w->z_begin, w->tail_lo);
                d2h(*w, w->tail_hi, w->z_end);
                CK(cudaEventRecord(w->head_done, w->copy));
            }
            for (auto& w : workers) {
                CK(cudaSetDevice(w->device));
                CK(cudaStreamWaitEvent(w->copy, w->tail_done, 0));
                d2h(*w, w->tail_lo, w->tail_hi);
                CK(cudaEventRecord(w->c_end, w->copy));
            }
        }
        // closes the kernel timing; with overlap this only re-checks flags
        // that cannot be set (pack errors were checked above)
        check_errors(true);
        for (auto& w : workers) {
            CK(cudaSetDevice(w->device));
            if (!overlap) {
                CK(cudaEventRecord(w->c_beg, w->copy));
                d2h(*w, w->z_begin, w->z_end);
                CK(cudaEventRecord(w->c_end, w->copy));
            }
        }
        for (auto& w : workers) {
            CK(cudaSetDevice(w->device));
            CK(cudaEventSynchronize(w->c_end));
            w->d2h_s += elapsed_s(w->c_beg, w->c_end);
        }
        if (t_tail) {
            auto& w = *workers.front();
            std::fprintf(stderr,
                         "cbb: resident, overlap %d, tail [%d, %d): k_beg->tail %.2f ms, "
                         "head d2h %.2f ms, k_beg->k_end %.2f ms, k_beg->c_end %.2f ms\n",
                         (int)overlap, w.tail_lo, w.tail_hi, elapsed_s(w.k_beg, t_tail) * 1e3,
                         overlap ? elapsed_s(w.c_beg, w.head_done) * 1e3 : 0.0,
                         elapsed_s(w.k_beg, w.k_end) * 1e3, elapsed_s(w.k_beg, w.c_end) * 1e3);
            cudaEventDestroy(t_tail);
        }
        resident = false;
    }

    void fill_stats(cbb_run_stats* st, double total) {
        if (!st)
            return;
        std::memset(st, 0, sizeof *st);
        uint64_t culled = 0;
        for (auto& w : workers) {
            std::vector<unsigned long long> c(kCounterSlots);
            CK(cudaSetDevice(w->device));
            CK(cudaMemcpy(c.data(), w->d_counters, sizeof(unsigned long long) * c.size(),
                          cudaMemcpyDeviceToHost));
            for (auto x : c)
                culled += x;
        }
        st->culled_updates = culled;
        st->total_seconds = total;
        st->num_gpus = (int32_t)workers.size();
        uint64_t planes = 0;
        for (const auto& w : workers)
            planes += (uint64_t)(w->z_end - w->z_begin);
        st->voxel_updates = (uint64_t)g.edge_voxels * g.edge_voxels * planes * submitted;
        for (size_t i = 0; i < workers.size(); ++i) {
            const auto& w = *workers[i];
            st->h2d_seconds = std::max(st->h2d_seconds, w.h2d_s);
            st->kernel_seconds = std::max(st->kernel_seconds, w.kernel_s);
            st->d2h_seconds = std::max(st->d2h_seconds, w.d2h_s);
            st->guarded_batches += w.guarded;
            if (i < 8)
                st->per_gpu_kernel_seconds[i] = w.kernel_s;
        }
        st->culled_fraction = !opt.count_culled ? -1.0
                              : st->voxel_updates
                                  ? (double)st->culled_updates / (double)st->voxel_updates
                                  : 0.0;
    }
};

} // namespace cbb

using namespace cbb;

struct cbb_session_s {
    Pipeline pipe;
    std::chrono::steady_clock::time_point t0;
};

extern "C" {

const char* cbb_status_name(cbb_status status) {
    switch (status) {
    case CBB_OK: return "ok";
    case CBB_ERR_INVALID: return "invalid argument";
    case CBB_ERR_IO: return "i/o error";
    case CBB_ERR_FORMAT: return "format error";
    case CBB_ERR_TRUNCATED: return "truncated file";
    case CBB_ERR_GEOMETRY: return "geometry error";
    case CBB_ERR_NOMEM: return "out of memory";
    case CBB_ERR_INTERNAL: return "internal error";
    }
    return "unknown status";
}

const char* cbb_last_error(void) { return g_last_error.c_str(); }

const char* cbb_version(void) { return "conebeam_b200 0.1 (sm_100a)"; }

int32_t cbb_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

uint64_t cbb_launch_count(void) { return g_launches; }

void cbb_options_defaults(cbb_options* o) {
    if (!o)
        return;
    o->num_gpus = 0;
    o->device_ids = nullptr;
    o->batch = 32;
    o->mode = CBB_MODE_EXACT;
    o->cull = 1;
    o->volume_is_zero = 0;
    o->slab_begin = 0;
    o->slab_end = 0;
    o->ramp_filter = 0;
    o->filter_pixel_mm = 0.0;
    o->count_culled = 0;
}

cbb_status cbb_packed_layout(int32_t width, int32_t height, int32_t* qpitch, int32_t* qrows,
                             int64_t* bytes) {
    return guarded([&] {
        validate_detector(width, height);
        if (qpitch)
            *qpitch = quad_pitch_cells(width);
        if (qrows)
            *qrows = quad_rows(height);
        if (bytes)
            *bytes = (int64_t)quad_pitch_cells(width) * quad_rows(height) * 16;
    });
}

cbb_status cbb_compare_volumes_device(const float* test, const float* ref, int64_t n,
                                      double denom_floor, cbb_volume_diff* out, void* stream) {
    return guarded([&] {
        if (!test || !ref || !out || n < 1)
            fail(CBB_ERR_INVALID, "cbb_compare_volumes_device: null or empty argument");
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        int dev = 0;
        CK(cudaGetDevice(&dev));
        auto* part = static_cast<MetricPartial*>(
            DevicePool::get().alloc(dev, sizeof(MetricPartial) * kMetricBlocks));
        metrics_partial<<<kMetricBlocks, kMetricThreads, 0, st>>>(test, ref, n, denom_floor, part);
        ++g_launches;
        std::vector<MetricPartial> h(kMetricBlocks);
        const cudaError_t e1 = cudaGetLastError();
        const cudaError_t e2 = cudaMemcpyAsync(h.data(), part, sizeof(MetricPartial) * kMetricBlocks,
                                               cudaMemcpyDeviceToHost, st);
        const cudaError_t e3 = cudaStreamSynchronize(st);
        DevicePool::get().release(dev, part);
        CK(e1);
        CK(e2);
        CK(e3);
        double ssd = 0, ssr = 0, mabs = 0, mrel = 0, rmin = DBL_MAX, rmax = -DBL_MAX;
        uint64_t nd = 0;
        for (const auto& p : h) { // fixed order: deterministic
            ssd += p.sum_sq_diff;
            ssr += p.sum_sq_ref;
            mabs = std::max(mabs, p.max_abs);
            mrel = std::max(mrel, p.max_rel);
            rmin = std::min(rmin, p.ref_min);
            rmax = std::max(rmax, p.ref_max);
            nd += p.bit_diff;
        }
        out->mse = ssd / (double)n;
        out->psnr_db = out->mse == 0.0 ? INFINITY : 10.0 * std::log10(rmax * rmax / out->mse);
        out->max_relative_error = mrel;
        out->rel_l2 = ssr > 0.0 ? std::sqrt(ssd / ssr) : (ssd > 0.0 ? INFINITY : 0.0);
        out->max_abs = mabs;
        out->ref_min = rmin;
        out->ref_max = rmax;
        out->max_abs_over_range = rmax > rmin ? mabs / (rmax - rmin) : (mabs > 0 ? INFINITY : 0.0);
        out->bitwise_different = nd;
    });
}

namespace {
std::mutex g_tex_mu;
std::map<int, std::tuple<cudaArray_t, int, int, int>> g_tex_arrays; // device -> array, W, H, layers
} // namespace

cbb_status cbb_release_cached_memory(void) {
    return guarded([&] {
        DevicePool::get().trim_all();
        HostPool::get().trim();
        std::lock_guard<std::mutex> lk(g_tex_mu);
        for (auto& kv : g_tex_arrays) {
            int cur = 0;
            cudaGetDevice(&cur);
            cudaSetDevice(kv.first);
            cudaDeviceSynchronize();
            cudaFreeArray(std::get<0>(kv.second));
            cudaSetDevice(cur);
        }
        g_tex_arrays.clear();
    });
}

cbb_status cbb_backproject_texture_device(float* vol_slab, const cbb_volume_geometry* geometry,
                                          int32_t z_begin, int32_t z_end, const float* raw,
                                          int32_t width, int32_t height, int32_t count,
                                          const double* mats, void* stream) {
    return guarded([&] {
        validate_geometry(geometry);
        if (!vol_slab || !raw || !mats)
            fail(CBB_ERR_INVALID, "cbb_backproject_texture_device: null argument");
        if (width < 1 || height < 1 || count < 1)
            fail(CBB_ERR_INVALID, "cbb_backproject_texture_device: empty input");
        if (z_begin < 0 || z_end > geometry->edge_voxels || z_begin >= z_end)
            fail(CBB_ERR_INVALID, "cbb_backproject_texture_device: bad slab");
        validate_matrices(mats, count);
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        const int L = geometry->edge_voxels;
        constexpr int kLayers = 2048; // layered-texture depth limit
        int dev = 0;
        CK(cudaGetDevice(&dev));
        // one layered array per device, kept between calls (allocating and
        // freeing GB-sized arrays costs tens of ms)
        auto& arrays = g_tex_arrays;
        std::lock_guard<std::mutex> lk(g_tex_mu);
        for (int chunk0 = 0; chunk0 < count; chunk0 += kLayers) {
            const int nc = std::min(kLayers, count - chunk0);
            cudaChannelFormatDesc fd = cudaCreateChannelDesc<float>();
            auto it = arrays.find(dev);
            if (it != arrays.end() && (std::get<1>(it->second) != width ||
                                       std::get<2>(it->second) != height ||
                                       std::get<3>(it->second) < nc)) {
                CK(cudaStreamSynchronize(st));
                cudaFreeArray(std::get<0>(it->second));
                arrays.erase(it);
                it = arrays.end();
            }
            if (it == arrays.end()) {
                cudaArray_t a = nullptr;
                CK(cudaMalloc3DArray(&a, &fd, make_cudaExtent(width, height, nc),
                                     cudaArrayLayered));
                it = arrays.emplace(dev, std::make_tuple(a, width, height, nc)).first;
            }
            cudaArray_t arr = std::get<0>(it->second);
            cudaMemcpy3DParms cp = {};
            cp.srcPtr = make_cudaPitchedPtr(const_cast<float*>(raw) + (size_t)chunk0 * width * height,
                                            (size_t)width * sizeof(float), width, height);
            cp.dstArray = arr;
            cp.extent = make_cudaExtent(width, height, nc);
            cp.kind = cudaMemcpyDeviceToDevice;
            cudaError_t e = cudaMemcpy3DAsync(&cp, st);
            cudaResourceDesc rd = {};
            rd.resType = cudaResourceTypeArray;
            rd.res.array.array = arr;
            cudaTextureDesc td = {};
            td.addressMode[0] = td.addressMode[1] = cudaAddressModeBorder;
            td.filterMode = cudaFilterModeLinear;
            td.readMode = cudaReadModeElementType;
            td.normalizedCoords = 0;
            cudaTextureObject_t tex = 0;
            if (e == cudaSuccess)
                e = cudaCreateTextureObject(&tex, &rd, &td, nullptr);
            for (int first = 0; e == cudaSuccess && first < nc; first += kMaxBatch) {
                const int n = std::min(kMaxBatch, nc - first);
                BpMats m;
                for (int p = 0; p < n; ++p)
                    store_matrix(m.a[p], mats + 12 * (size_t)(chunk0 + first + p));
                constexpr int R = 8;
                dim3 grid((L + kBlockX - 1) / kBlockX, (L + kBlockY - 1) / kBlockY,
                          (z_end - z_begin + R - 1) / R);
                bp_texture_kernel<R><<<grid, 256, 0, st>>>(
                    vol_slab, L, z_begin, z_end, (float)geometry->origin_mm,
                    (float)geometry->voxel_mm, tex, first, n, m);
                ++g_launches;
                e = cudaGetLastError();
            }
            // the texture object is released (and the array reused) once the
            // chunk has run
            const cudaError_t es = cudaStreamSynchronize(st);
            if (tex)
                cudaDestroyTextureObject(tex);
            CK(e);
            CK(es);
        }
    });
}

cbb_status cbb_ramp_filter_device(const float* raw, float* out, int32_t width, int32_t height,
                                  int32_t count, double pixel_mm, void* stream) {
    return guarded([&] {
        if (!raw || !out || count < 0)
            fail(CBB_ERR_INVALID, "cbb_ramp_filter_device: null argument");
        if (width < 1 || height < 1)
            fail(CBB_ERR_INVALID, "ProjectionImage: dimensions must be >= 1");
        if (!(pixel_mm > 0.0) || !std::isfinite(pixel_mm))
            fail(CBB_ERR_INVALID, "cbb_ramp_filter_device: pixel_mm must be positive");
        if (count == 0)
            return;
        ramp_filter_device(raw, out, width, height, count, pixel_mm,
                           static_cast<cudaStream_t>(stream));
    });
}

cbb_status cbb_pack_device(const float* raw, int32_t width, int32_t height, int32_t count,
                           void* packed, void* stream) {
    return guarded([&] {
        if (!raw || !packed || count < 0)
            fail(CBB_ERR_INVALID, "cbb_pack_device: null argument");
        validate_detector(width, height);
        if (count > 65535)
            fail(CBB_ERR_INVALID, "cbb_pack_device: count > 65535 per call");
        if (count == 0)
            return;
        launch_pack(raw, width, height, count, packed, static_cast<cudaStream_t>(stream));
    });
}

cbb_status cbb_backproject_device(float* vol_slab, const cbb_volume_geometry* geometry,
                                  int32_t z_begin, int32_t z_end, const void* packed,
                                  int32_t width, int32_t height, int32_t count,
                                  const double* mats, const cbb_options* options,
                                  int32_t* err_flag, void* stream) {
    return guarded([&] {
        validate_geometry(geometry);
        validate_detector(width, height);
        if (!vol_slab || !packed || !mats)
            fail(CBB_ERR_INVALID, "cbb_backproject_device: null argument");
        if (z_begin < 0 || z_end > geometry->edge_voxels || z_begin > z_end)
            fail(CBB_ERR_INVALID, "cbb_backproject_device: bad slab [%d, %d)", z_begin, z_end);
        validate_matrices(mats, count);
        const cbb_options opt = resolve_options(options);
        launch_backproject(vol_slab, *geometry, z_begin, z_end, packed, width, height, count,
                           mats, opt, err_flag, static_cast<cudaStream_t>(stream));
    });
}

namespace {
RowBand band_from_c(const cbb_row_band* b, int H) {
    if (!b)
        return RowBand::full(H);
    RowBand r;
    r.r0 = b->raw_row0;
    r.rn = b->raw_rows;
    r.q0 = b->cell_row0;
    r.qn = b->cell_rows;
    if (r.r0 < 0 || r.rn < 0 || r.r0 + r.rn > H || r.q0 < 0 || r.qn < 1 ||
        r.q0 + r.qn > quad_rows(H))
        fail(CBB_ERR_INVALID, "row band [%d, +%d) rows / [%d, +%d) cells outside the detector",
             r.r0, r.rn, r.q0, r.qn);
    return r;
}
} // namespace

cbb_status cbb_row_band_for_slab(const cbb_volume_geometry* geometry, int32_t width,
                                 int32_t height, int32_t z_begin, int32_t z_end,
                                 const double* mats, int32_t count, cbb_row_band* band) {
    return guarded([&] {
        validate_geometry(geometry);
        validate_detector(width, height);
        if (!mats || !band || count < 1)
            fail(CBB_ERR_INVALID, "cbb_row_band_for_slab: null argument or count < 1");
        if (z_begin < 0 || z_end > geometry->edge_voxels || z_begin >= z_end)
            fail(CBB_ERR_INVALID, "cbb_row_band_for_slab: bad slab [%d, %d)", z_begin, z_end);
        validate_matrices(mats, count);
        const RowBand b = row_band_for(*geometry, width, height, z_begin, z_end, mats, count);
        band->raw_row0 = b.r0;
        band->raw_rows = b.rn;
        band->cell_row0 = b.q0;
        band->cell_rows = b.qn;
    });
}

cbb_status cbb_pack_device_band(const float* raw, int64_t raw_stride, int32_t width,
                                int32_t height, int32_t count, const cbb_row_band* band,
                                void* packed, int32_t* err_flag, void* stream) {
    return guarded([&] {
        validate_detector(width, height);
        if (!raw || !packed || !band || count < 0)
            fail(CBB_ERR_INVALID, "cbb_pack_device_band: null argument");
        if (count > 65535)
            fail(CBB_ERR_INVALID, "cbb_pack_device_band: count > 65535 per call");
        const RowBand b = band_from_c(band, height);
        if (raw_stride < (int64_t)b.rn * width)
            fail(CBB_ERR_INVALID, "cbb_pack_device_band: raw_stride below the band size");
        if (count == 0)
            return;
        launch_pack_band(raw, b.r0, b.rn, raw_stride, width, height, count, packed, b,
                         static_cast<cudaStream_t>(stream), err_flag);
    });
}

cbb_status cbb_backproject_device_band(float* vol_slab, const cbb_volume_geometry* geometry,
                                       int32_t z_begin, int32_t z_end, const void* packed,
                                       int32_t width, int32_t height, int32_t count,
                                       const double* mats, const cbb_row_band* band,
                                       const cbb_options* options, int32_t* err_flag,
                                       void* stream) {
    return guarded([&] {
        validate_geometry(geometry);
        validate_detector(width, height);
        if (!vol_slab || !packed || !mats)
            fail(CBB_ERR_INVALID, "cbb_backproject_device_band: null argument");
        if (z_begin < 0 || z_end > geometry->edge_voxels || z_begin > z_end)
            fail(CBB_ERR_INVALID, "cbb_backproject_device_band: bad slab [%d, %d)", z_begin,
                 z_end);
        validate_matrices(mats, count);
        const RowBand b = band_from_c(band, height);
        if (band && z_end > z_begin && count > 0) {
            const RowBand need =
                row_band_for(*geometry, width, height, z_begin, z_end, mats, count);
            if (need.q0 < b.q0 || need.q0 + need.qn > b.q0 + b.qn ||
                (need.rn > 0 && (need.r0 < b.r0 || need.r0 + need.rn > b.r0 + b.rn)))
                fail(CBB_ERR_INVALID,
                     "cbb_backproject_device_band: band cells [%d, %d) do not cover the "
                     "slab's footprint [%d, %d)",
                     b.q0, b.q0 + b.qn, need.q0, need.q0 + need.qn);
        }
        const cbb_options opt = resolve_options(options);
        launch_backproject(vol_slab, *geometry, z_begin, z_end, packed, width, height, count,
                           mats, opt, err_flag, static_cast<cudaStream_t>(stream), 0, 0, &b);
    });
}

cbb_status cbb_check_finite_device(const float* values, int64_t n, int32_t* err_flag,
                                   void* stream) {
    return guarded([&] {
        if (!values || !err_flag || n < 0)
            fail(CBB_ERR_INVALID, "cbb_check_finite_device: null argument");
        launch_check_finite(values, n, err_flag, static_cast<cudaStream_t>(stream));
    });
}

cbb_status cbb_reconstruct(float* vol, const cbb_volume_geometry* geometry, const float* imgs,
                           int32_t width, int32_t height, int32_t count, const double* mats,
                           const cbb_options* options, cbb_run_stats* stats) {
    return guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();
        if (!vol || !imgs || !mats)
            fail(CBB_ERR_INVALID, "cbb_reconstruct: null argument");
        validate_geometry(geometry);
        validate_detector(width, height);
        if (count < 1)
            fail(CBB_ERR_INVALID, "ProjectionStack: at least one projection required");
        validate_matrices(mats, count);
        const cbb_options opt = resolve_options(options);
        const bool trace = std::getenv("CBB_TRACE") != nullptr;
        auto ms = [&] {
            return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                .count();
        };
        double t_init = 0, t_sub = 0, t_fin = 0;
        {
            Pipeline pipe;
            pipe.init(*geometry, width, height, opt, vol);
            t_init = ms();
            pipe.submit_stack(imgs, mats, count);
            t_sub = ms();
            // finish() checks the error flags before any download, so on a
            // geometry error vol is left unchanged; only the slab planes are written
            pipe.finish(vol);
            t_fin = ms();
            pipe.fill_stats(stats, 0.0);
        }
        const double total =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (stats)
            stats->total_seconds = total;
        if (trace)
            std::fprintf(stderr, "cbb: host init %.2f submit %.2f finish %.2f teardown %.2f ms\n",
                         t_init, t_sub, t_fin, total * 1e3);
    });
}

cbb_status cbb_reconstruct_images(float* vol, const cbb_volume_geometry* geometry,
                                  const float* const* imgs, int32_t width, int32_t height,
                                  int32_t count, const double* mats,
                                  const cbb_options* options, cbb_run_stats* stats) {
    return guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();
        if (!vol || !imgs || !mats)
            fail(CBB_ERR_INVALID, "cbb_reconstruct_images: null argument");
        validate_geometry(geometry);
        validate_detector(width, height);
        if (count < 1)
            fail(CBB_ERR_INVALID, "ProjectionStack: at least one projection required");
        for (int32_t i = 0; i < count; ++i)
            if (!imgs[i])
                fail(CBB_ERR_INVALID, "cbb_reconstruct_images: image %d is null", i);
        validate_matrices(mats, count);
        const cbb_options opt = resolve_options(options);
        {
            Pipeline pipe;
            pipe.init(*geometry, width, height, opt, vol);
            pipe.submit_images(imgs, mats, count);
            pipe.finish(vol);
            pipe.fill_stats(stats, 0.0);
        }
        if (stats)
            stats->total_seconds =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

// CBPS header (proj/include/conebeam/dataset.hpp:62-72, proj/src/dataset.cpp:
// 181-212): "CBPS", u16 version 1, u16 reserved, u32 W, u32 H, u32 count,
// f64 voxel_mm, f64 origin_mm, u32 L; then count records of 96 + 4*W*H bytes.
struct StackFile {
    int fd = -1;
    cbb_stack_file_info info{};
    uint64_t header_bytes = 40, rec_bytes = 0;
    ~StackFile() {
        if (fd >= 0)
            ::close(fd);
    }
};

void open_stack_file(const char* path, StackFile& f) {
    static_assert(sizeof(double) == 8 && sizeof(float) == 4, "IEEE sizes");
    const uint16_t probe = 1;
    if (*reinterpret_cast<const uint8_t*>(&probe) != 1)
        fail(CBB_ERR_INTERNAL, "big-endian hosts are not supported by the streaming reader");
    f.fd = ::open(path, O_RDONLY);
    if (f.fd < 0)
        fail(CBB_ERR_IO, "cannot open '%s' for reading", path);
    unsigned char h[40];
    if (!Pipeline::pread_all(f.fd, h, 4, 0))
        fail(CBB_ERR_TRUNCATED, "file ends inside magic");
    if (std::memcmp(h, "CBPS", 4) != 0)
        fail(CBB_ERR_FORMAT, "not a stack file (magic mismatch)");
    if (!Pipeline::pread_all(f.fd, h + 4, 4, 4))
        fail(CBB_ERR_TRUNCATED, "file ends inside version");
    uint16_t version;
    std::memcpy(&version, h + 4, 2);
    if (version != 1)
        fail(CBB_ERR_FORMAT, "stack file version %u not supported (expected 1)", version);
    if (!Pipeline::pread_all(f.fd, h + 8, 32, 8))
        fail(CBB_ERR_TRUNCATED, "file ends inside header");
    uint32_t W, H, N, L;
    std::memcpy(&W, h + 8, 4);
    std::memcpy(&H, h + 12, 4);
    std::memcpy(&N, h + 16, 4);
    std::memcpy(&f.info.voxel_mm, h + 20, 8);
    std::memcpy(&f.info.origin_mm, h + 28, 8);
    std::memcpy(&L, h + 36, 4);
    if (W < 1 || H < 1 || N < 1)
        fail(CBB_ERR_FORMAT, "stack header has zero width, height, or count");
    if (W > (1u << 20) || H > (1u << 20) || N > (1u << 30) || L > (1u << 30))
        fail(CBB_ERR_FORMAT, "stack header sizes out of range");
    f.info.width = (int32_t)W;
    f.info.height = (int32_t)H;
    f.info.count = (int32_t)N;
    f.info.edge_voxels = (int32_t)L;
    const cbb_volume_geometry g{f.info.edge_voxels, f.info.voxel_mm, f.info.origin_mm};
    validate_geometry(&g);
    f.rec_bytes = 96 + 4ull * W * H;
    struct stat st;
    if (::fstat(f.fd, &st) != 0)
        fail(CBB_ERR_IO, "cannot stat '%s'", path);
    const uint64_t want = f.header_bytes + f.rec_bytes * N;
    if ((uint64_t)st.st_size < want)
        fail(CBB_ERR_TRUNCATED, "file ends inside projection intensities");
    if ((uint64_t)st.st_size > want)
        fail(CBB_ERR_FORMAT, "stack file has trailing bytes after payload");
}

cbb_status cbb_backproject(float* vol, const cbb_volume_geometry* geometry, const float* img,
                           int32_t width, int32_t height, const double* matrix12) {
    cbb_options o;
    cbb_options_defaults(&o);
    o.num_gpus = 1;
    o.batch = 1;
    return cbb_reconstruct(vol, geometry, img, width, height, 1, matrix12, &o, nullptr);
}

cbb_status cbb_stack_file_query(const char* path, cbb_stack_file_info* out) {
    return guarded([&] {
        if (!path || !out)
            fail(CBB_ERR_INVALID, "cbb_stack_file_query: null argument");
        StackFile f;
        open_stack_file(path, f);
        *out = f.info;
    });
}

cbb_status cbb_reconstruct_file(float* vol, const char* path, const cbb_options* options,
                                cbb_run_stats* stats) {
    return guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();
        if (!vol || !path)
            fail(CBB_ERR_INVALID, "cbb_reconstruct_file: null argument");
        StackFile f;
        open_stack_file(path, f);
        validate_detector(f.info.width, f.info.height);
        const cbb_options opt = resolve_options(options);
        const cbb_volume_geometry g{f.info.edge_voxels, f.info.voxel_mm, f.info.origin_mm};
        Pipeline pipe;
        pipe.init(g, f.info.width, f.info.height, opt, vol);
        pipe.submit_file(f.fd, f.info.count, f.header_bytes, f.rec_bytes);
        pipe.finish(vol);
        const double total =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        pipe.fill_stats(stats, total);
    });
}

cbb_status cbb_session_create(const cbb_volume_geometry* geometry, int32_t width,
                              int32_t height, const float* initial_volume,
                              const cbb_options* options, cbb_session** out) {
    return guarded([&] {
        if (!out)
            fail(CBB_ERR_INVALID, "cbb_session_create: null argument");
        validate_geometry(geometry);
        validate_detector(width, height);
        const cbb_options opt = resolve_options(options);
        auto s = std::make_unique<cbb_session_s>();
        s->t0 = std::chrono::steady_clock::now();
        s->pipe.init(*geometry, width, height, opt, initial_volume);
        *out = s.release();
    });
}

cbb_status cbb_session_backproject(cbb_session* s, const float* img, const double* m) {
    return guarded([&] {
        if (!s || !img || !m)
            fail(CBB_ERR_INVALID, "cbb_session_backproject: null argument");
        validate_matrices(m, 1);
        s->pipe.stage_one(img, m);
    });
}

cbb_status cbb_session_finish(cbb_session* s, float* vol_out, cbb_run_stats* stats) {
    return guarded([&] {
        if (!s || !vol_out)
            fail(CBB_ERR_INVALID, "cbb_session_finish: null argument");
        s->pipe.finish(vol_out);
        const double total =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - s->t0).count();
        s->pipe.fill_stats(stats, total);
    });
}

void cbb_session_free(cbb_session* s) { delete s; }

} // extern "C"
