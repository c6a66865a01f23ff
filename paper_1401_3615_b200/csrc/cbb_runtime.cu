// cbb_runtime.cu -- host runtime and C ABI of libconebeam_b200.so.
//
// Implements include/conebeam_b200.h: error model mirroring the reference C
// API (proj/src/capi.cpp:26-68; runtime_common.cuh), the guard decision per
// batch and the launches of the sm_100a kernels in bp_kernels.cuh
// (launch.cuh), buffer caches (memory.cuh) and the staging pipeline
// (pipeline.cuh):
//   host projections --(pinned, ring-buffered cudaMemcpyAsync on a copy
//   stream)--> raw ring slot --(pack_quads on the compute stream)--> packed
//   ring slot --(bp_kernel, matrices as kernel parameters = constant bank)-->
//   register partial sums --> volume slab in HBM.
// Multi-GPU (one process): the volume is split into work-balanced z-slabs,
// one per device; each batch is uploaded once (rotating root) and the other
// devices copy the detector rows their slab needs peer-to-peer; slabs are
// downloaded into the caller's volume at the end (no reduction: voxel
// ownership is disjoint).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <functional>
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
#include <nvtx3/nvToolsExt.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include "../../include/conebeam_b200.h"
#include "bp_kernels.cuh"
#include "bp_tma.cuh"
#include "ramp_filter.cuh"
#include "metrics.cuh"
#include "texture_variant.cuh"

#include "runtime_common.cuh"
#include "ipc.cuh"
#include "launch.cuh"
#include "launch_tma.cuh"
#include "memory.cuh"
#include "pipeline.cuh"

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
    // one GPU unless asked: the cross-device paths (P2P band packs, rotating
    // upload roots) are tested with several workers on one GPU only
    o->num_gpus = 1;
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
            *bytes = (int64_t)quad_pitch_cells(width) * quad_rows(height) * 16 + kMetaBytes;
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

// ---- CUDA IPC buffers and stream-ordered flags (multi-process drivers) ----

cbb_status cbb_ipc_alloc(int64_t bytes, void** dev_ptr, void* handle) {
    return guarded([&] {
        if (bytes <= 0 || !dev_ptr || !handle)
            fail(CBB_ERR_INVALID, "cbb_ipc_alloc: bad argument");
        void* p = nullptr;
        CK(cudaMalloc(&p, (size_t)bytes));
        CK(cudaMemset(p, 0, (size_t)bytes));
        cudaIpcMemHandle_t h;
        const cudaError_t e = cudaIpcGetMemHandle(&h, p);
        if (e != cudaSuccess) {
            cudaFree(p);
            CK(e);
        }
        std::memcpy(handle, &h, sizeof h);
        *dev_ptr = p;
    });
}

cbb_status cbb_ipc_free(void* dev_ptr) {
    return guarded([&] {
        if (dev_ptr) {
            CK(cudaDeviceSynchronize());
            CK(cudaFree(dev_ptr));
        }
    });
}

cbb_status cbb_ipc_open(const void* handle, void** dev_ptr) {
    return guarded([&] {
        if (!handle || !dev_ptr)
            fail(CBB_ERR_INVALID, "cbb_ipc_open: null argument");
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof h);
        CK(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    });
}

cbb_status cbb_ipc_close(void* dev_ptr) {
    return guarded([&] {
        if (dev_ptr)
            CK(cudaIpcCloseMemHandle(dev_ptr));
    });
}

cbb_status cbb_stream_write_flag(void* flag, uint32_t value, void* stream) {
    return guarded([&] {
        const auto& ops = StreamMemOps::get();
        if (!ops.write || !flag)
            fail(CBB_ERR_INTERNAL, "cuStreamWriteValue32 unavailable or null flag");
        check_cu(ops.write(static_cast<CUstream>(stream), (CUdeviceptr)flag, value,
                           CU_STREAM_WRITE_VALUE_DEFAULT),
                 "cuStreamWriteValue32");
    });
}

cbb_status cbb_stream_wait_flag(const void* flag, uint32_t value, void* stream) {
    return guarded([&] {
        const auto& ops = StreamMemOps::get();
        if (!ops.wait || !flag)
            fail(CBB_ERR_INTERNAL, "cuStreamWaitValue32 unavailable or null flag");
        check_cu(ops.wait(static_cast<CUstream>(stream), (CUdeviceptr)flag, value,
                          CU_STREAM_WAIT_VALUE_GEQ),
                 "cuStreamWaitValue32");
    });
}

cbb_status cbb_memcpy_h2d_async(void* dst, const void* src, int64_t bytes, void* stream) {
    return guarded([&] {
        if (!dst || !src || bytes < 0)
            fail(CBB_ERR_INVALID, "cbb_memcpy_h2d_async: bad argument");
        CK(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyHostToDevice,
                           static_cast<cudaStream_t>(stream)));
    });
}

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

cbb_status cbb_tma_plan(const cbb_volume_geometry* geometry, int32_t width, int32_t height,
                        int32_t z_begin, int32_t z_end, const double* mats, int32_t count,
                        cbb_tma_plan_info* out) {
    return guarded([&] {
        validate_geometry(geometry);
        validate_detector(width, height);
        if (!mats || !out || count < 1)
            fail(CBB_ERR_INVALID, "cbb_tma_plan: null argument or count < 1");
        if (z_begin < 0 || z_end > geometry->edge_voxels || z_begin >= z_end)
            fail(CBB_ERR_INVALID, "cbb_tma_plan: bad slab [%d, %d)", z_begin, z_end);
        validate_matrices(mats, count);
        const TmaPlan p = plan_tma(*geometry, width, height, z_begin, z_end, mats, count);
        out->staged = p.ok && tma_path_enabled() ? 1 : 0;
        out->box_width = p.pitch;
        out->box_rows = p.bh;
        out->stages = p.stages;
        out->footprint_width = p.bw_need;
        out->footprint_rows = p.bh_need;
    });
}

cbb_status cbb_scan_device(const float* raw, int64_t raw_stride, int32_t width, int32_t rows,
                           int32_t count, uint32_t* flags, int32_t* err_flag, void* stream) {
    return guarded([&] {
        if (!raw || !flags || count < 0 || width < 1 || rows < 0)
            fail(CBB_ERR_INVALID, "cbb_scan_device: bad argument");
        if (raw_stride < (int64_t)width * rows)
            fail(CBB_ERR_INVALID, "cbb_scan_device: raw_stride below rows * width");
        launch_scan(raw, width, rows, raw_stride, count, flags, err_flag,
                    static_cast<cudaStream_t>(stream));
    });
}

cbb_status cbb_backproject_raw_device(float* vol_slab, const cbb_volume_geometry* geometry,
                                      int32_t z_begin, int32_t z_end, const float* raw,
                                      int64_t raw_stride, int32_t width, int32_t height,
                                      const cbb_row_band* band, int32_t count, const double* mats,
                                      const uint32_t* flags, const cbb_options* options,
                                      int32_t* err_flag, void* stream) {
    return guarded([&] {
        validate_geometry(geometry);
        validate_detector(width, height);
        if (!vol_slab || !raw || !mats || !flags)
            fail(CBB_ERR_INVALID, "cbb_backproject_raw_device: null argument");
        if (z_begin < 0 || z_end > geometry->edge_voxels || z_begin > z_end)
            fail(CBB_ERR_INVALID, "cbb_backproject_raw_device: bad slab [%d, %d)", z_begin, z_end);
        validate_matrices(mats, count);
        const RowBand b = band_from_c(band, height);
        if (raw_stride < (int64_t)b.rn * width)
            fail(CBB_ERR_INVALID, "cbb_backproject_raw_device: raw_stride below the band size");
        if (band && z_end > z_begin && count > 0) {
            const RowBand need =
                row_band_for(*geometry, width, height, z_begin, z_end, mats, count);
            if (need.rn > 0 && (need.r0 < b.r0 || need.r0 + need.rn > b.r0 + b.rn))
                fail(CBB_ERR_INVALID,
                     "cbb_backproject_raw_device: band rows [%d, %d) do not cover the slab's "
                     "footprint [%d, %d)",
                     b.r0, b.r0 + b.rn, need.r0, need.r0 + need.rn);
        }
        const cbb_options opt = resolve_options(options);
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (count == 0 || z_end == z_begin)
            return;
        const TmaPlan plan = plan_tma(*geometry, width, height, z_begin, z_end, mats, count);
        if (std::getenv("CBB_TRACE"))
            std::fprintf(stderr, "cbb: tma plan ok %d pitch %d bh %d stages %d (need %d x %d)\n", plan.ok,
                         plan.pitch, plan.bh, plan.stages, plan.bw_need, plan.bh_need);
        if (plan.ok && tma_path_enabled() && (uintptr_t)raw % 16 == 0 && raw_stride % 4 == 0 &&
            b.rn >= 1) {
            launch_backproject_raw(vol_slab, *geometry, z_begin, z_end, raw, raw_stride, width,
                                   height, b.r0, b.rn, count, mats, flags, plan, opt, err_flag,
                                   st);
            return;
        }
        // footprint too large for the staged boxes (coarse voxels), unaligned
        // rows or CBB_BP_PATH=quad: pack into a scratch buffer, gather kernel
        int dev = 0;
        CK(cudaGetDevice(&dev));
        const int qp = quad_pitch_cells(width);
        const RowBand pb = b.is_full(height) ? b : row_band_for(*geometry, width, height,
                                                                z_begin, z_end, mats, count);
        const size_t per = (size_t)qp * pb.qn * 16 + kMetaBytes;
        const int step = std::min(count, std::max(opt.batch, (int)((size_t(2) << 30) / per)));
        void* packed = DevicePool::get().alloc(dev, per * step);
        try {
            for (int c0 = 0; c0 < count; c0 += step) {
                const int n = std::min(step, count - c0);
                launch_pack_band(raw + (long long)c0 * raw_stride, b.r0, b.rn, raw_stride, width,
                                 height, n, packed, pb, st, err_flag);
                launch_backproject(vol_slab, *geometry, z_begin, z_end, packed, width, height, n,
                                   mats + 12 * (size_t)c0, opt, err_flag, st, 0, 0, &pb);
            }
        } catch (...) {
            cudaStreamSynchronize(st);
            DevicePool::get().release(dev, packed);
            throw;
        }
        // the pool hands the buffer out again only after this stream's work
        // (released buffers are reused in stream order by the same caller)
        CK(cudaStreamSynchronize(st));
        DevicePool::get().release(dev, packed);
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
        NvtxRange range("cbb_reconstruct");
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
            pipe.init(*geometry, width, height, opt, vol, mats, count, /*defer_volume=*/true);
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
        NvtxRange range("cbb_reconstruct_images");
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
            pipe.init(*geometry, width, height, opt, vol, mats, count, /*defer_volume=*/true);
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
        NvtxRange range("cbb_reconstruct_file");
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
        // Volume::validate now (proj/src/dataset.cpp:146-151), not at the
        // first finish: a session over a non-finite volume is never created
        if (initial_volume && !opt.volume_is_zero)
            s->pipe.check_errors(false);
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
