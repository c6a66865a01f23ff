// runtime_common.cuh -- error model, input validation and the host-side
// range proofs that let a batch run the unguarded kernel.
// Internal part of libconebeam_b200.so: included, in this order, by
// cbb_runtime.cu (one translation unit: runtime_common.cuh, launch.cuh,
// memory.cuh, pipeline.cuh).
#pragma once

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

// NVTX range for the lifetime of the object (host phases in nsys / ncu
// timelines: call, batch issue, finish); no cost without a profiler.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

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
    // packed cell indices (kMagic-biased int32, see cell_index) must stay
    // below 2^31: detectors up to ~29800 x 29800
    const double cells = (double)quad_pitch_cells(w) * quad_rows(h);
    if (cells >= kMaxCells)
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
    if (r.batch < 1 || r.batch > kMaxOptBatch)
        fail(CBB_ERR_INVALID, "options: batch must be in [1, %d]", kMaxOptBatch);
    if (r.mode != CBB_MODE_EXACT && r.mode != CBB_MODE_FAST)
        fail(CBB_ERR_INVALID, "options: unknown mode %d", r.mode);
    if (r.num_gpus < 0)
        fail(CBB_ERR_INVALID, "options: num_gpus must be >= 0");
    // device_ids has no length of its own: num_gpus gives it
    if (r.device_ids && r.num_gpus == 0)
        fail(CBB_ERR_INVALID, "options: device_ids needs num_gpus > 0 (its length)");
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
        // [2^-20, 2^20]: the range the kernel's FCHK-free divisions are proven
        // for (bp_kernels.cuh, kBigBits); calibrated mm-scaled matrices with
        // w ~ 500-1500 stay on the fast kernels
        if (!(w > 1e-4 * scale) || !(w >= 0x1p-20) || !(w <= 0x1p20))
            return false;
        if (!(std::fabs(u / w) < 1e8) || !(std::fabs(v / w) < 1e8))
            return false;
    }
    return true;
}

} // namespace cbb
