/*
 * conebeam_b200.h -- C ABI of the B200-native FDK back-projection library
 * (libconebeam_b200.so, built from paper_1401_3615_b200/csrc/).
 *
 * This is the drop-in boundary for the reference's hot path: voxel-driven
 * back-projection of filtered cone-beam projections into a float32 volume
 * (reference: proj/src/kernel_ref.cpp:5-38, proj/src/kernel_opt.cpp:658-716,
 * exposed there through proj/include/conebeam/capi.h:104-107).
 *
 * Conventions kept from the reference C API (proj/include/conebeam/capi.h):
 *  - every function returns a cbb_status whose numeric values are identical
 *    to cb_status (capi.h:20-29); the message of the last failure on the
 *    calling thread is available from cbb_last_error() (capi.cpp:26-28);
 *  - objects live behind opaque handles released with the matching *_free;
 *  - stats out-parameters are nullable.
 *
 * Data layouts are the reference's (proj/include/conebeam/dataset.hpp:15-60,
 * geometry.hpp:47-65): projections are row-major float32, index iy*W+ix;
 * volumes are float32, index (z*L+y)*L+x; each projection matrix is 12
 * doubles, column-major 3x4 (u = wx*a0 + wy*a3 + wz*a6 + a9, ...), cast to
 * float inside the kernel exactly as the reference does (kernel_ref.cpp:11-13).
 *
 * Semantics: reconstructions ACCUMULATE into the given volume (vol +=), in
 * projection order, like reconstruct_reference. In exact mode (the default)
 * the result is bitwise identical to reconstruct_reference; on any error the
 * host volume is left unchanged (the reference leaves it partially updated).
 *
 * No torch types appear here; device entry points take plain device
 * pointers and a cudaStream_t passed as void*.
 */
#ifndef CONEBEAM_B200_H
#define CONEBEAM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same values as cb_status (proj/include/conebeam/capi.h:20-29). */
typedef enum cbb_status {
    CBB_OK = 0,
    CBB_ERR_INVALID = 1,   /* bad arguments or configuration */
    CBB_ERR_IO = 2,        /* open/read/write failure */
    CBB_ERR_FORMAT = 3,    /* bad magic, version, or trailing bytes */
    CBB_ERR_TRUNCATED = 4, /* payload shorter than the header promises */
    CBB_ERR_GEOMETRY = 5,  /* degenerate geometry: a voxel with w == 0 */
    CBB_ERR_NOMEM = 6,     /* host or device allocation failed */
    CBB_ERR_INTERNAL = 7   /* CUDA / NCCL failure, no device, ... */
} cbb_status;

/* Replaces cb_status_name / cb_last_error (capi.h:31-32, capi.cpp:93-108). */
const char* cbb_status_name(cbb_status status);
const char* cbb_last_error(void);

/* Library/device introspection. */
const char* cbb_version(void);
int32_t cbb_device_count(void);

/* Volume descriptor (VolumeGeometry, proj/include/conebeam/geometry.hpp:15-34). */
typedef struct cbb_volume_geometry {
    int32_t edge_voxels; /* L */
    double voxel_mm;
    double origin_mm;    /* world coordinate of voxel index 0 */
} cbb_volume_geometry;

/* Kernel arithmetic variants. */
enum {
    CBB_MODE_EXACT = 0, /* bitwise equal to reconstruct_reference (default) */
    CBB_MODE_FAST = 1   /* weight 1/w^2 as r*r with one reciprocal; relL2 ~1e-7 */
};

/* Options (the B200 counterpart of cb_opt_options, capi.h:84-91). */
typedef struct cbb_options {
    int32_t num_gpus;          /* default 1; 0 = all visible devices (whole-stack calls) */
    const int32_t* device_ids; /* nullable: devices 0..num_gpus-1; else num_gpus ids
                                  (num_gpus must then be > 0: it is the array length) */
    int32_t batch;             /* projections per pipeline batch (upload + launch), 1..64
                                  (default 32); the gather kernel launches at most 32 at a time,
                                  the TMA-staged kernel up to 64 */
    int32_t mode;              /* CBB_MODE_EXACT / CBB_MODE_FAST */
    int32_t cull;              /* skip voxel tiles whose footprint misses the detector */
    int32_t volume_is_zero;    /* caller promises the input volume is all +0: skip its upload */
    int32_t slab_begin;        /* z-planes [slab_begin, slab_end) of the volume to update; */
    int32_t slab_end;          /* 0, 0 = all planes (one process per GPU drives one slab) */
    int32_t ramp_filter;       /* 1: projections are raw line integrals; apply the FDK row-wise
                                  Shepp-Logan ramp filter on the GPU before back-projecting */
    double filter_pixel_mm;    /* detector pixel pitch tau of the ramp filter (mm) */
    int32_t count_culled;      /* 1: count the updates warp culling skips (run stats
                                  culled_updates / culled_fraction; ~9 % slower kernels) */
} cbb_options;

void cbb_options_defaults(cbb_options* options);

/* Per-call statistics (cb_run_stats, capi.h:93-102, extended per phase). */
typedef struct cbb_run_stats {
    double total_seconds;      /* wall time of the call */
    double h2d_seconds;        /* max over GPUs, device-timed */
    double kernel_seconds;     /* max over GPUs, device-timed (pack + back-projection) */
    double d2h_seconds;        /* max over GPUs, device-timed */
    uint64_t voxel_updates;    /* full basis: L^3 * projections */
    uint64_t guarded_batches;  /* batches that needed the guarded kernel */
    int32_t num_gpus;
    double per_gpu_kernel_seconds[8];
    /* (voxel, projection) updates skipped because warp culling proved them
     * exactly zero (footprint off the detector); computed = voxel_updates -
     * culled_updates. Counted only with cbb_options.count_culled (else 0 and
     * culled_fraction = -1). */
    uint64_t culled_updates;
    double culled_fraction;    /* culled_updates / voxel_updates, or -1 if not counted */
} cbb_run_stats;

/* ---- host-pointer entry points (the drop-in) ------------------------------ */

/* One projection into the whole volume: backproject_reference
 * (proj/src/kernel_ref.cpp:5-30, kernel_ref.hpp:77). Synchronous. The volume
 * is uploaded, updated and downloaded on every call; prefer cbb_reconstruct
 * or a session for stacks. */
cbb_status cbb_backproject(float* vol, const cbb_volume_geometry* geometry,
                           const float* img, int32_t width, int32_t height,
                           const double* matrix12);

/* All projections in order: reconstruct_reference / cb_reconstruct_optimized
 * (proj/src/kernel_ref.cpp:32-38, capi.h:104-107). imgs holds count*height*width
 * floats, mats count*12 doubles. The input volume is validated like
 * Volume::validate (proj/src/dataset.cpp:146-151): a non-finite voxel gives
 * CBB_ERR_INVALID and the volume is left unchanged (skipped when
 * options->volume_is_zero promises zeros). On one GPU the input volume is
 * uploaded in z-chunks alongside the first batches rather than before them
 * (the call still reads it, and writes the result, only while it runs).
 * Multi-GPU: work-balanced z-slabs,
 * one per device, all driven from the calling thread; each batch is uploaded
 * once and the other devices read their row bands over peer memory (P2P
 * loads inside the pack kernel, not an NCCL broadcast -- NCCL is used by the
 * one-process-per-GPU driver, paper_1401_3615_b200/distributed.py). */
cbb_status cbb_reconstruct(float* vol, const cbb_volume_geometry* geometry,
                           const float* imgs, int32_t width, int32_t height,
                           int32_t count, const double* mats,
                           const cbb_options* options /* nullable */,
                           cbb_run_stats* stats /* nullable */);

/* cbb_reconstruct for projections held in separate buffers, as the
 * reference's ProjectionStack holds them (one std::vector<float> per
 * ProjectionImage, proj/include/conebeam/dataset.hpp:15-60): imgs[i] points
 * to height*width floats of projection i. Batches are gathered into pinned
 * staging by several host threads while the GPU works on the previous batch,
 * so no contiguous copy of the stack is needed. */
cbb_status cbb_reconstruct_images(float* vol, const cbb_volume_geometry* geometry,
                                  const float* const* imgs, int32_t width, int32_t height,
                                  int32_t count, const double* mats,
                                  const cbb_options* options /* nullable */,
                                  cbb_run_stats* stats /* nullable */);

/* ---- streaming from a CBPS stack file ------------------------------------ */

/* Header of a CBPS stack file (proj/include/conebeam/dataset.hpp:62-72) --
 * the counterpart of cb_stack_read + cb_stack_get_info (capi.h:57-73) without
 * loading the projections. Same error statuses as read_stack
 * (proj/src/dataset.cpp:181-212): IO, FORMAT (magic, version, trailing bytes),
 * TRUNCATED. */
typedef struct cbb_stack_file_info {
    int32_t edge_voxels;
    double voxel_mm;
    double origin_mm;
    int32_t count;
    int32_t width;
    int32_t height;
} cbb_stack_file_info;

cbb_status cbb_stack_file_query(const char* path, cbb_stack_file_info* out);

/* Reconstructs a CBPS file into vol (L^3 floats, accumulated like
 * cbb_reconstruct), streaming the projection records from disk into pinned
 * double buffers overlapped with the device work: HOST memory use is
 * independent of the projection count. DEVICE memory is not: when the whole
 * packed stack fits in HBM with 2 GB to spare, every packed projection is kept
 * resident (count x cbb_packed_layout bytes per device, ~61 GB for 1440 x
 * 1536^2) so the last planes can be finished from HBM while the head of the
 * volume downloads; the buffer stays in the library's cache until
 * cbb_release_cached_memory (set CBB_NO_RESIDENT=1 to stream only).
 * Non-finite pixels or voxels -> CBB_ERR_INVALID. */
cbb_status cbb_reconstruct_file(float* vol, const char* path, const cbb_options* options,
                                cbb_run_stats* stats);

/* ---- streaming session (RabbitCT-style per-projection module) ------------ */

typedef struct cbb_session_s cbb_session;

/* initial_volume (L^3 floats, nullable = zeros) is copied and validated at
 * creation (non-finite voxel -> CBB_ERR_INVALID, no session is created). */
cbb_status cbb_session_create(const cbb_volume_geometry* geometry, int32_t width,
                              int32_t height, const float* initial_volume,
                              const cbb_options* options, cbb_session** out);
/* Enqueues one projection (copied before return); launches when a batch fills. */
cbb_status cbb_session_backproject(cbb_session* s, const float* img, const double* matrix12);
/* Flushes and writes the accumulated volume (L^3 floats) to vol_out. The
 * session stays usable and keeps accumulating afterwards. */
cbb_status cbb_session_finish(cbb_session* s, float* vol_out, cbb_run_stats* stats);
void cbb_session_free(cbb_session* s);

/* ---- device-resident entry points (plain device pointers) ---------------- */

/* Layout of the packed projection buffer the back-projection kernel gathers
 * from: per projection, quad_rows x quad_pitch float4 cells; cell (px,py)
 * holds the four bilinear taps of detector position (px,py) with zeros
 * outside the detector (zero-pad semantics of bilinear_sample_guarded). */
cbb_status cbb_packed_layout(int32_t width, int32_t height, int32_t* quad_pitch,
                             int32_t* quad_rows, int64_t* bytes_per_projection);

/* raw: count x height x width floats (device). packed: count packed
 * projections (device, cbb_packed_layout bytes each). Enqueued on stream. */
cbb_status cbb_pack_device(const float* raw, int32_t width, int32_t height, int32_t count,
                           void* packed, void* stream);

/* Back-projects count packed projections into a z-slab [z_begin, z_end) of
 * the volume held on the device at vol_slab (voxel (0,0,z_begin) first,
 * z-major). mats: count*12 doubles on the HOST (they travel as kernel
 * parameters, i.e. constant memory). err_flag: device int (nullable) set to 1
 * when a voxel hits w == 0; the caller must check it (cbb_reconstruct does).
 * Enqueued on stream; returns after launch. */
cbb_status cbb_backproject_device(float* vol_slab, const cbb_volume_geometry* geometry,
                                  int32_t z_begin, int32_t z_end, const void* packed,
                                  int32_t width, int32_t height, int32_t count,
                                  const double* mats, const cbb_options* options,
                                  int32_t* err_flag, void* stream);

/* Row bands (multi-GPU z-slabs): the detector rows a slab's voxels can touch
 * over a set of projections. A worker then holds only those raw rows and
 * packs only the matching cell rows (cell row = detector row + pad, see
 * cbb_packed_layout); at 8 slabs of a 512^3 volume each needs about a third of
 * the detector. Full detector (raw 0..H, cells 0..quad_rows) when w <= 0
 * somewhere on the slab or the rows are unbounded. */
typedef struct cbb_row_band {
    int32_t raw_row0;  /* detector rows held: [raw_row0, raw_row0 + raw_rows) */
    int32_t raw_rows;
    int32_t cell_row0; /* packed cell rows: [cell_row0, cell_row0 + cell_rows) */
    int32_t cell_rows;
} cbb_row_band;

cbb_status cbb_row_band_for_slab(const cbb_volume_geometry* geometry, int32_t width,
                                 int32_t height, int32_t z_begin, int32_t z_end,
                                 const double* mats, int32_t count, cbb_row_band* band);

/* Packs count projections, band cell rows only (band->cell_rows * quad_pitch
 * float4 cells each). raw points at detector row band->raw_row0 of projection
 * 0; consecutive projections are raw_stride floats apart (width*height for a
 * full raw buffer offset by raw_row0*width, raw_rows*width for a band
 * buffer). Pixels outside the held rows read as 0. err_flag (device int,
 * nullable): bit 2 set on a non-finite pixel among the packed ones. */
cbb_status cbb_pack_device_band(const float* raw, int64_t raw_stride, int32_t width,
                                int32_t height, int32_t count, const cbb_row_band* band,
                                void* packed, int32_t* err_flag, void* stream);

/* cbb_backproject_device on band-packed projections. band must cover the
 * footprint of [z_begin, z_end) for these matrices (checked on the host:
 * CBB_ERR_INVALID otherwise); NULL = full detector. */
cbb_status cbb_backproject_device_band(float* vol_slab, const cbb_volume_geometry* geometry,
                                       int32_t z_begin, int32_t z_end, const void* packed,
                                       int32_t width, int32_t height, int32_t count,
                                       const double* mats, const cbb_row_band* band,
                                       const cbb_options* options, int32_t* err_flag,
                                       void* stream);

/* ---- TMA-staged back-projection from raw projections (no packing) ---------
 * cbb_scan_device: per projection of `count` (rows x width floats each,
 * raw_stride floats apart), flags[p] = 1 when a pixel has |value| >= 2^86
 * (the exact mode's fast division needs the flag) and bit 2
 * of *err_flag on a non-finite pixel (ProjectionImage::validate). flags: count
 * uint32 on the device. Enqueued on stream.
 * cbb_backproject_raw_device: cbb_backproject_device on RAW projections:
 * raw points at row band->raw_row0 (0 when band is NULL) of projection 0,
 * raw_stride floats between projections; flags from cbb_scan_device. Each
 * block's detector footprint is staged in shared memory by TMA. Same bits as
 * the packed path. Falls back to packing internally when the footprint boxes
 * do not fit (coarse voxels) or rows are not 16-byte aligned. */
/* The staging plan cbb_backproject_raw_device and cbb_reconstruct (one GPU,
 * whole stack known) use for a slab: staged = 1 when the TMA kernel runs
 * (box_width x box_rows floats per block and projection, `stages` deep),
 * 0 when the footprint boxes exceed the shared-memory budget (coarse voxels),
 * rows are not 16-byte aligned (width % 4 != 0) or CBB_BP_PATH=quad: then the
 * packed-quad kernel runs. Host-only (no GPU needed). */
typedef struct cbb_tma_plan_info {
    int32_t staged;
    int32_t box_width, box_rows, stages;
    int32_t footprint_width, footprint_rows; /* sampled bound incl. margins */
} cbb_tma_plan_info;
cbb_status cbb_tma_plan(const cbb_volume_geometry* geometry, int32_t width, int32_t height,
                        int32_t z_begin, int32_t z_end, const double* mats, int32_t count,
                        cbb_tma_plan_info* out);
cbb_status cbb_scan_device(const float* raw, int64_t raw_stride, int32_t width, int32_t rows,
                           int32_t count, uint32_t* flags, int32_t* err_flag, void* stream);
cbb_status cbb_backproject_raw_device(float* vol_slab, const cbb_volume_geometry* geometry,
                                      int32_t z_begin, int32_t z_end, const float* raw,
                                      int64_t raw_stride, int32_t width, int32_t height,
                                      const cbb_row_band* band, int32_t count, const double* mats,
                                      const uint32_t* flags, const cbb_options* options,
                                      int32_t* err_flag, void* stream);

/* ProjectionImage::validate on the device (proj/src/dataset.cpp:123-129):
 * sets bit 2 of *err_flag if any of the n floats is not finite. For the
 * uploading rank of a row-band pipeline, whose own band skips rows. */
cbb_status cbb_check_finite_device(const float* values, int64_t n, int32_t* err_flag,
                                   void* stream);

/* FDK filtering step (upstream of the back-projection; the reference consumes
 * pre-filtered data): row-wise Shepp-Logan ramp filter
 * h[n] = -2/(pi^2 tau (4n^2-1)) as a linear convolution (zero-padded float64
 * FFT, length >= 2W), rounded to float32. raw/out: count*height*width floats
 * on the device (may alias). Enqueued on stream. */
cbb_status cbb_ramp_filter_device(const float* raw, float* out, int32_t width, int32_t height,
                                  int32_t count, double pixel_mm, void* stream);

/* Side variant (north_star: "reported separately, only as a side number"):
 * hardware-texture bilinear back-projection of raw (unpacked) projections,
 * FMA coordinates and an approximate reciprocal. It does NOT match the
 * reference (8-bit texture weights, floor addressing); see DESIGN.md for its
 * measured deviation. Synchronous per batch of 32. */
cbb_status cbb_backproject_texture_device(float* vol_slab, const cbb_volume_geometry* geometry,
                                          int32_t z_begin, int32_t z_end, const float* raw,
                                          int32_t width, int32_t height, int32_t count,
                                          const double* mats, void* stream);

/* Volume comparison on the device: quality_metrics (proj/src/bench.cpp:65-82),
 * max_relative_error (:92-102) and the north_star parity figures. */
typedef struct cbb_volume_diff {
    double mse;                /* mean (t - r)^2 */
    double psnr_db;            /* 10 log10(max_ref^2 / mse); +inf when mse == 0 */
    double max_relative_error; /* max |t - r| / (|r| + denom_floor) */
    double rel_l2;             /* ||t - r||_2 / ||r||_2 */
    double max_abs;            /* max |t - r| */
    double ref_min, ref_max;
    double max_abs_over_range; /* max_abs / (ref_max - ref_min) */
    uint64_t bitwise_different;
} cbb_volume_diff;

/* test, ref: n floats each on the device. Synchronous on stream. */
cbb_status cbb_compare_volumes_device(const float* test, const float* ref, int64_t n,
                                      double denom_floor, cbb_volume_diff* out, void* stream);

/* ---- multi-process plumbing (one process per GPU) ------------------------
 * Device buffers another process can map (CUDA IPC; handle = 64 bytes), and
 * stream-ordered 32-bit flags (cuStreamWriteValue32 / cuStreamWaitValue32),
 * so a rank's pack kernel can read the uploading rank's projection slot over
 * NVLink once that rank has flagged it ready -- the broadcast and the layout
 * transform become one kernel. cbb_stream_wait_flag blocks the stream until
 * (int32_t)(*flag - value) >= 0. */
cbb_status cbb_ipc_alloc(int64_t bytes, void** dev_ptr, void* handle /* 64 bytes */);
cbb_status cbb_ipc_free(void* dev_ptr);
cbb_status cbb_ipc_open(const void* handle, void** dev_ptr);
cbb_status cbb_ipc_close(void* dev_ptr);
cbb_status cbb_stream_write_flag(void* flag, uint32_t value, void* stream);
cbb_status cbb_stream_wait_flag(const void* flag, uint32_t value, void* stream);
cbb_status cbb_memcpy_h2d_async(void* dst, const void* src, int64_t bytes, void* stream);

/* Frees the library's cached device buffers, pinned host staging and texture
 * arrays (kept between calls to avoid allocation costs), like
 * torch.cuda.empty_cache. Call when no other cbb_* call is running. */
cbb_status cbb_release_cached_memory(void);

/* Number of kernel launches the last cbb_backproject_device / cbb_pack_device
 * calls on this thread issued (for the bench's gpu_launches count). */
uint64_t cbb_launch_count(void);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* CONEBEAM_B200_H */
