// pipeline.cuh -- the staging pipeline: per-device workers (slab,
// ring slots, streams), rotating upload roots and row-band peer copies,
// resident tail pass, downloads, run statistics.
// Internal part of libconebeam_b200.so: included, in this order, by
// cbb_runtime.cu (one translation unit: runtime_common.cuh, launch.cuh,
// memory.cuh, pipeline.cuh).
#pragma once

namespace cbb {

// Raw-projection ring per device: G + 1 slots for G devices (at most
// kMaxSlots), so with rotating upload roots the next G uploads -- one per
// device -- are in flight together; with two slots they would serialise
// (2.8 ms per 153 MB batch against ~0.7 ms of kernels per batch at G = 8).
// Pinned host staging for pageable sources is a separate ring of two (a
// third did not help: those host copies contend with the DMA for host
// memory, measured on config 2).
constexpr int kMaxSlots = 17;
constexpr int kStageSlots = 2;

// ---------------------------------------------------------------------------
// Per-device worker: slab volume, raw/packed double buffers, streams, events.
// ---------------------------------------------------------------------------

struct Worker {
    int device = 0;
    int z_begin = 0, z_end = 0;
    float* d_vol = nullptr;
    float* d_raw[kMaxSlots] = {};
    void* d_packed = nullptr;          // one batch: pack and kernels share the compute stream
    int* d_err = nullptr;
    cudaStream_t copy = nullptr, compute = nullptr;
    cudaEvent_t h2d_done[kMaxSlots] = {}, raw_free[kMaxSlots] = {};
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
    cudaEvent_t head_done = nullptr, tail_done = nullptr, tail_mid_done = nullptr;
    // detector rows this worker holds / packs (RowBand::full unless set_bands)
    RowBand band;
    size_t pk_bytes = 0;               // packed bytes per projection (band rows)
    cudaEvent_t src_ready[kMaxSlots] = {}; // as root: raw slot filtered, peers may copy
    cudaEvent_t stage_read[kStageSlots] = {}; // as root: H2D from host staging slot done
    cudaEvent_t xfer_ev[2] = {};       // ChunkedXfer chunk events (copy stream)
    unsigned long long* d_counters = nullptr; // kCounterSlots culled-update counters
    bool count_culled = false;
    // raw mode (TMA kernel, bp_tma.cuh): per-projection scan flags of the
    // current batch, or of every resident projection
    unsigned* d_flags = nullptr;
    unsigned* d_flags_all = nullptr;
    TmaPlan plan;                      // this slab's staging plan (raw mode)

    ~Worker() {
        if (!copy)
            return;
        cudaSetDevice(device);
        cudaStreamSynchronize(copy);
        cudaStreamSynchronize(compute);
        auto& pool = DevicePool::get();
        pool.release(device, d_vol);
        for (int i = 0; i < kMaxSlots; ++i) {
            pool.release(device, d_raw[i]);
            if (h2d_done[i])
                cudaEventDestroy(h2d_done[i]);
            if (raw_free[i])
                cudaEventDestroy(raw_free[i]);
            if (src_ready[i])
                cudaEventDestroy(src_ready[i]);
        }
        pool.release(device, d_packed);
        for (auto e : stage_read)
            if (e)
                cudaEventDestroy(e);
        for (auto e : xfer_ev)
            cudaEventDestroy(e);
        pool.release(device, d_err);
        pool.release(device, d_counters);
        pool.release(device, d_packed_all);
        pool.release(device, d_flags);
        pool.release(device, d_flags_all);
        if (head_done)
            cudaEventDestroy(head_done);
        if (tail_done)
            cudaEventDestroy(tail_done);
        if (tail_mid_done)
            cudaEventDestroy(tail_mid_done);
        cudaEventDestroy(k_beg);
        cudaEventDestroy(k_end);
        cudaEventDestroy(c_beg);
        cudaEventDestroy(c_end);
        cudaStreamDestroy(copy);
        cudaStreamDestroy(compute);
    }
};

double elapsed_s(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.0f;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms * 1e-3;
}

// Estimated back-projection work of the 8-plane groups of [z0, z1) (group g
// starts at plane z0 + 8g): planes x (fraction of sampled (x, y, projection)
// positions that land on the detector -- warp culling skips the rest -- +
// a fixed overhead), sampled on a 12 x 12 grid at the group's centre plane for
// up to 4 of the n projections.
std::vector<double> group_work(const cbb_volume_geometry& g, int W, int H, int z0, int z1,
                               const double* mats, int n, int group = 8) {
    const int L = g.edge_voxels, S = 12, NP = std::min(n, 4);
    std::vector<double> gw;
    for (int z = z0; z < z1; z += group) {
        const int pz = std::min(group, z1 - z);
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
    }
    return gw;
}

// ng contiguous slabs of [s0, s1) with near-equal estimated work (the
// single-process counterpart of distributed.py's balanced_slabs); each gets
// at least one plane.
std::vector<int> balanced_bounds(const cbb_volume_geometry& g, int W, int H, int s0, int s1,
                                 int ng, const double* mats, int n) {
    const std::vector<double> gw = group_work(g, W, H, s0, s1, mats, n);
    std::vector<double> cum(1, 0.0); // per-plane prefix sums
    for (int z = s0; z < s1; ++z) {
        const int k = (z - s0) / 8;
        const int pz = std::min(8, s1 - (s0 + 8 * k));
        cum.push_back(cum.back() + gw[k] / pz);
    }
    std::vector<int> b(1, s0);
    for (int r = 1; r < ng; ++r) {
        const double target = cum.back() * r / ng;
        int z = (int)(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin());
        z = std::max(b.back() - s0 + 1, std::min(z, (s1 - s0) - (ng - r)));
        b.push_back(s0 + z);
    }
    b.push_back(s1);
    return b;
}

struct Pipeline {
    cbb_volume_geometry g{};
    int W = 0, H = 0;
    cbb_options opt{};
    std::vector<std::unique_ptr<Worker>> workers;
    float* h_stage[kStageSlots] = {};       // pinned staging (batch x H x W)
    int stage_owner[kStageSlots] = {-1, -1}; // worker whose H2D last read the staging slot
    ChunkedXfer xfer;                       // volume up/download for pageable buffers
    int stage_fill = 0;                     // projections staged in the current slot
    int sslot = 0;                          // current host staging slot
    int slot = 0;                           // current device ring slot
    int nslots = 2;                         // device ring slots in use
    std::vector<double> stage_mats;         // matrices of the staged batch
    uint64_t submitted = 0;
    uint64_t nbatch = 0;   // batches issued (root = nbatch mod workers)
    bool peer_pack = false; // non-root workers pack from the root's raw slot directly
    size_t raw_bytes_per_proj = 0;
    size_t packed_bytes_per_proj = 0;
    bool resident = false;         // see Worker::d_packed_all
    int resident_count = 0;
    std::vector<double> all_mats;  // resident mode: every matrix, for the tail pass
    const double* est_mats = nullptr; // matrices for choose_tails (else the first batch)
    int est_n = 0;
    // Raw mode: one device, whole stack known, detector rows 16-byte aligned
    // and footprint boxes within the shared-memory budget: the batches are
    // scanned (scan_projections) and back-projected straight from the raw
    // projections by the TMA-staged kernel -- no packing, and resident mode
    // keeps the raw stack (4.8x smaller than the packed one).
    bool raw_mode = false;
    int tail_group() const { return raw_mode ? kTR : 8; }

    // Deferred initial volume (one worker, a volume to accumulate into):
    // init() does not upload it. In raw resident mode (whole stack known)
    // it goes up in z-chunks interleaved with the first batches -- one
    // chunk ahead of each batch, the tail planes last -- and the head
    // launches cover the chunks already on the device, each chunk catching
    // up on the projections it missed (every voxel still takes the
    // projections one by one in stack order, so the bits do not change).
    // The pageable volume's upload (~14 ms for config 2's 537 MB through
    // the staging chunks) then overlaps the projection stream instead of
    // preceding it. Every other path uploads it whole before its first
    // batch (upload_volume_whole).
    const float* vol_src = nullptr; // the slab's first plane in the caller's volume
    struct VolChunk {
        int z0 = 0, z1 = 0;
        int applied = 0;            // projections already back-projected into it
        bool issued = false, tail = false;
        cudaEvent_t ready = nullptr; // copy stream: uploaded and checked
    };
    std::vector<VolChunk> vchunks;
    size_t vchunk_next = 0;
    bool tails_chosen = false;

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
                CK(cudaEventCreateWithFlags(&w->tail_mid_done, cudaEventDisableTiming));
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
    // sampled on a 12 x 12 grid at the group's centre plane for up to 4 of
    // the given projections. A dense tail keeps its D2H short while its
    // compute hides the head's D2H.
    // the tail holds the smallest plane range with `frac` of the work: its
    // compute must cover the head's download, ~50 GB/s into pinned memory
    // but ~30 GB/s into pageable memory through the staging chunks (the C++
    // adapter's volume): config 2 adapter path 110 -> 106 ms with 0.24;
    // with the deferred volume and streaming host copies the stream phase
    // is shorter and 0.16-0.20 balance it best (94.4 ms vs 96.4 at 0.24 and
    // 0.12, 100 at 0.06: there the head launches outrun the uploads)
    bool out_pageable = false; // init: the caller's volume (in and out) is pageable
    void choose_tails(const double* mats, int n) {
        if (tails_chosen) // once per stack (the volume chunks follow the tails)
            return;
        tails_chosen = true;
        // pinned: 0.10-0.18 measured within 0.3 % of each other (76.0 +- 0.2 ms,
        // profiles/e2e_tail_r2.txt); 0.14 leaves ~3 ms of tail compute beyond
        // the 8.3 ms head download, for boxes with slower D2H
        double frac = out_pageable ? 0.18 : 0.14;
        if (const char* e = std::getenv("CBB_TAIL_FRAC"))
            frac = std::atof(e);
        for (auto& w : workers) {
            const int gs = tail_group(); // head launches skip the tail: aligned to their z-blocks
            const std::vector<double> gw =
                group_work(g, W, H, w->z_begin, w->z_end, mats, n, gs);
            std::vector<int> gz;
            for (int z = w->z_begin; z < w->z_end; z += gs)
                gz.push_back(z);
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
            if (const char* e = std::getenv("CBB_TAIL_PLANES")) { // tests: "lo:hi", group-aligned
                int lo = 0, hi = 0;
                if (std::sscanf(e, "%d:%d", &lo, &hi) == 2 && lo >= w->z_begin && hi <= w->z_end &&
                    lo < hi && (lo - w->z_begin) % gs == 0 &&
                    (hi == w->z_end || (hi - w->z_begin) % gs == 0)) {
                    w->tail_lo = lo;
                    w->tail_hi = hi;
                }
            }
            if (std::getenv("CBB_TRACE"))
                std::fprintf(stderr, "cbb: device %d slab [%d, %d) tail [%d, %d)\n", w->device,
                             w->z_begin, w->z_end, w->tail_lo, w->tail_hi);
        }
    }

    ~Pipeline() {
        if (!workers.empty()) {
            cudaSetDevice(workers[0]->device);
            cudaStreamSynchronize(workers[0]->copy);
        }
        for (auto& c : vchunks)
            if (c.ready)
                cudaEventDestroy(c.ready);
        workers.clear();
        for (auto h : h_stage)
            HostPool::get().release(h);
    }

    // mats/nmats (nullable): the whole stack's matrices; with several devices
    // and culling on, the slabs are then balanced by estimated work instead
    // of equal plane counts. defer_volume: a whole-stack call (cbb_reconstruct,
    // cbb_reconstruct_images) whose volume may go up with the first batches
    // (VolChunk); sessions validate the volume at creation, so they do not.
    void init(const cbb_volume_geometry& geom, int width, int height, const cbb_options& o,
              const float* initial_volume, const double* mats = nullptr, int nmats = 0,
              bool defer_volume = false) {
        g = geom;
        W = width;
        H = height;
        opt = o;
        out_pageable = initial_volume && !is_pinned(initial_volume);
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
        packed_bytes_per_proj = (size_t)quad_pitch_cells(W) * quad_rows(H) * 16 + kMetaBytes;
        const int L = g.edge_voxels;
        const size_t plane = (size_t)L * L;
        std::vector<int> bounds;
        if (mats && nmats > 0 && ng > 1 && opt.cull)
            bounds = balanced_bounds(g, W, H, s0, s1, ng, mats, nmats);
        for (int i = 0; i < ng; ++i) {
            auto w = std::make_unique<Worker>();
            w->device = opt.device_ids ? opt.device_ids[i] : i;
            if (w->device < 0 || w->device >= ndev)
                fail(CBB_ERR_INVALID, "options: device id %d not visible", w->device);
            w->z_begin = bounds.empty() ? s0 + (int)((long long)(s1 - s0) * i / ng) : bounds[i];
            w->z_end = bounds.empty() ? s0 + (int)((long long)(s1 - s0) * (i + 1) / ng)
                                      : bounds[i + 1];
            CK(cudaSetDevice(w->device));
            {
                // the copy stream also runs the resident scan (issue_raw): high
                // priority, so its blocks take the first SM slots the
                // back-projection frees instead of waiting for the launch to drain
                int lo = 0, hi = 0;
                CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
                CK(cudaStreamCreateWithPriority(&w->copy, cudaStreamNonBlocking,
                                                std::getenv("CBB_COPY_PRIO0") ? lo : hi));
            }
            CK(cudaStreamCreateWithFlags(&w->compute, cudaStreamNonBlocking));
            nslots = std::min(kMaxSlots, std::max(2, ng + 1));
            for (int s = 0; s < nslots; ++s) {
                CK(cudaEventCreateWithFlags(&w->h2d_done[s], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&w->raw_free[s], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&w->src_ready[s], cudaEventDisableTiming));
                w->d_raw[s] = static_cast<float*>(
                    DevicePool::get().alloc(w->device, raw_bytes_per_proj * opt.batch));
            }
            w->d_packed = DevicePool::get().alloc(w->device, packed_bytes_per_proj * opt.batch);
            for (auto& e : w->stage_read)
                CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            for (auto& e : w->xfer_ev)
                CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
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
            // on the copy stream: the volume check below sets bit 4 there, and
            // the compute stream waits for c_end before its first kernel
            CK(cudaMemsetAsync(w->d_err, 0, sizeof(int), w->copy));
            const size_t cbytes = sizeof(unsigned long long) * kCounterSlots;
            w->d_counters = static_cast<unsigned long long*>(
                DevicePool::get().alloc(w->device, cbytes));
            CK(cudaMemsetAsync(w->d_counters, 0, cbytes, w->compute));
            w->count_culled = opt.count_culled != 0;
            CK(cudaEventRecord(w->c_beg, w->copy));
            if (initial_volume && !opt.volume_is_zero && ng == 1 && defer_volume &&
                !std::getenv("CBB_NO_VOL_DEFER")) {
                vol_src = initial_volume + plane * w->z_begin; // see VolChunk
            } else if (initial_volume && !opt.volume_is_zero) {
                xfer.upload(w->d_vol, initial_volume + plane * w->z_begin, slab * sizeof(float),
                            w->copy, w->xfer_ev);
                // Volume::validate (proj/src/dataset.cpp:146-151, called by
                // backproject_reference, kernel_ref.cpp:7): a non-finite voxel
                // is reported as CBB_ERR_INVALID before anything is written back
                launch_check_finite(w->d_vol, (long long)slab, w->d_err, w->copy, 4);
            } else
                CK(cudaMemsetAsync(w->d_vol, 0, slab * sizeof(float), w->copy));
            CK(cudaEventRecord(w->c_end, w->copy));
            CK(cudaStreamWaitEvent(w->compute, w->c_end, 0));
            workers.push_back(std::move(w));
        }
        stage_mats.assign(12 * (size_t)opt.batch, 0.0);
        // peer access between every pair of devices: band reads go straight
        // over NVLink; without it for some pair, band copies are staged
        peer_pack = !std::getenv("CBB_NO_PEER_PACK");
        for (auto& a : workers)
            for (auto& b : workers) {
                int can = 0;
                if (a->device == b->device)
                    continue;
                if (cudaDeviceCanAccessPeer(&can, b->device, a->device) != cudaSuccess || !can) {
                    cudaGetLastError();
                    peer_pack = false;
                    continue;
                }
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
    // upload completes (wait_stage for the staging ring).
    // stage >= 0: src is host staging slot `stage` (its reuse waits for this H2D).
    // issue() in raw mode (one worker): upload (into the resident raw stack
    // or a ring slot), optional ramp filter, scan, TMA back-projection.
    void issue_raw(const float* src, const double* mats, int n, int stage) {
        if (workers.size() > 1)
            return issue_raw_multi(src, mats, n, stage);
        NvtxRange range("cbb batch (raw)");
        Worker& w = *workers[0];
        CK(cudaSetDevice(w.device));
        const size_t bytes = raw_bytes_per_proj * n;
        float* dst;
        unsigned* flags;
        if (resident) {
            dst = static_cast<float*>(w.d_packed_all) + (size_t)submitted * W * H;
            flags = w.d_flags_all + submitted;
        } else {
            dst = w.d_raw[slot];
            flags = w.d_flags;
            CK(cudaStreamWaitEvent(w.copy, w.raw_free[slot], 0));
        }
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, w.copy));
        if (stage >= 0) {
            CK(cudaEventRecord(w.stage_read[stage], w.copy));
            stage_owner[stage] = 0;
        }
        // resident, pre-filtered stack: scan right behind the upload on the
        // (high-priority) copy stream -- per-projection flags, nothing else
        // reads them yet -- so it overlaps the back-projection instead of
        // queueing between launches (at default priority its blocks waited
        // for each launch to drain and stalled the uploads: 95 vs 78 ms)
        const bool scan_on_copy = resident && !opt.ramp_filter && !std::getenv("CBB_SCAN_COMPUTE");
        if (scan_on_copy)
            launch_scan(dst, W, H, (long long)W * H, n, flags, w.d_err, w.copy);
        CK(cudaEventRecord(w.h2d_done[slot], w.copy));
        CK(cudaStreamWaitEvent(w.compute, w.h2d_done[slot], 0));
        start_timing(w);
        if (opt.ramp_filter)
            ramp_filter_device(dst, dst, W, H, n, opt.filter_pixel_mm, w.compute);
        if (!scan_on_copy)
            launch_scan(dst, W, H, (long long)W * H, n, flags, w.d_err, w.compute);
        if (resident && submitted == 0)
            choose_tails(est_mats ? est_mats : mats, est_mats ? est_n : n);
        if (resident) {
            // the stack stays in HBM: back-project in launches of up to
            // kTmaBatch resident projections (the upload batch only sets the
            // streaming granularity, e.g. BASELINE config 4's batches of 16);
            // during the ramp-up (batches below opt.batch) launch at once
            std::memcpy(all_mats.data() + 12 * submitted, mats, 12 * sizeof(double) * n);
            // launch sizes keep growing like the upload ramp (4, 4, 8, 16,
            // 32, 64, 64, ...): never more than twice the previous launch, so
            // the device is not left waiting for a large accumulation
            const int pend = (int)(submitted + n) - raw_pending;
            // and with the upload ramp on (small slabs), every batch of the
            // first 128 projections is launched at once too: accumulating to
            // 2x the last launch there left the device waiting for uploads
            // (config 2 end to end 78.1 -> 76.5 ms; CBB_LAUNCH_RAMP: experiments)
            static const int launch_ramp_env = std::getenv("CBB_LAUNCH_RAMP")
                                                   ? std::atoi(std::getenv("CBB_LAUNCH_RAMP"))
                                                   : -1;
            const int launch_ramp = launch_ramp_env >= 0 ? launch_ramp_env
                                                         : (ramp_ < opt.batch ? 128 : 0);
            if (n < opt.batch || (int)(submitted + n) <= launch_ramp ||
                pend >= std::min(kTmaBatch, 2 * raw_last_launch))
                launch_raw_pending((int)(submitted + n));
        } else {
            w.guarded += launch_backproject_raw(w.d_vol, g, w.z_begin, w.z_end, dst,
                                               (long long)W * H, W, H, 0, H, n, mats, flags,
                                               w.plan, opt, w.d_err, w.compute, 0, 0,
                                               w.count_culled ? w.d_counters : nullptr);
            CK(cudaEventRecord(w.raw_free[slot], w.compute));
        }
        ++nbatch;
        submitted += n;
        slot = (slot + 1) % nslots;
    }

    // issue_raw with several workers: batch k is uploaded once by worker
    // k mod G; every worker holds its slab's band of raw rows -- the root
    // copies its band out of its slot (into its resident stack) or reads it in
    // place, the others copy theirs from the root's slot peer-to-peer (the
    // staged kernel reads local memory through its tensor map); each then
    // scans its rows and runs the TMA-staged kernel on them.
    void issue_raw_multi(const float* src, const double* mats, int n, int stage) {
        NvtxRange range("cbb batch (raw, multi)");
        const int G = (int)workers.size();
        Worker& root = *workers[nbatch % G];
        // slot reuse, as in issue_packed: the root's slot is read by its own
        // kernels (raw_free) and the other workers' band copies (h2d_done);
        // a non-root worker's slot is rewritten by its next band copy
        CK(cudaSetDevice(root.device));
        for (auto& o : workers) {
            CK(cudaStreamWaitEvent(root.copy, o->raw_free[slot], 0));
            if (o.get() != &root)
                CK(cudaStreamWaitEvent(root.copy, o->h2d_done[slot], 0));
        }
        for (auto& w : workers)
            if (w.get() != &root) {
                CK(cudaSetDevice(w->device));
                CK(cudaStreamWaitEvent(w->copy, w->raw_free[slot], 0));
            }
        CK(cudaSetDevice(root.device));
        CK(cudaMemcpyAsync(root.d_raw[slot], src, raw_bytes_per_proj * n, cudaMemcpyHostToDevice,
                           root.copy));
        CK(cudaEventRecord(root.h2d_done[slot], root.copy));
        if (stage >= 0) {
            CK(cudaEventRecord(root.stage_read[stage], root.copy));
            stage_owner[stage] = (int)(nbatch % G);
        }
        CK(cudaStreamWaitEvent(root.compute, root.h2d_done[slot], 0));
        start_timing(root);
        cudaEvent_t ready = root.h2d_done[slot];
        if (opt.ramp_filter) {
            ramp_filter_device(root.d_raw[slot], root.d_raw[slot], W, H, n, opt.filter_pixel_mm,
                               root.compute);
            CK(cudaEventRecord(root.src_ready[slot], root.compute));
            ready = root.src_ready[slot];
        }
        // the root sees the whole batch: it checks the pixels no band holds
        if (!root.band.is_full(H))
            launch_check_finite(root.d_raw[slot], (long long)n * W * H, root.d_err, root.compute);
        if (resident && submitted == 0)
            choose_tails(est_mats ? est_mats : mats, est_mats ? est_n : n);
        for (auto& wp : workers) {
            Worker& w = *wp;
            CK(cudaSetDevice(w.device));
            const int r0 = w.band.r0, rows = w.band.rn;
            const size_t band_bytes = (size_t)rows * W * sizeof(float);
            float* res = resident ? static_cast<float*>(w.d_packed_all) + (size_t)submitted * rows * W
                                  : nullptr;
            unsigned* flags = resident ? w.d_flags_all + submitted : w.d_flags;
            const float* rows_ptr;
            long long stride;
            if (&w == &root) {
                if (resident) {
                    CK(cudaMemcpy2DAsync(res, band_bytes, root.d_raw[slot] + (size_t)r0 * W,
                                         raw_bytes_per_proj, band_bytes, n,
                                         cudaMemcpyDeviceToDevice, w.compute));
                    rows_ptr = res;
                    stride = (long long)rows * W;
                } else {
                    rows_ptr = root.d_raw[slot] + (size_t)r0 * W;
                    stride = (long long)W * H;
                }
            } else {
                float* d = resident ? res : w.d_raw[slot];
                CK(cudaStreamWaitEvent(w.copy, ready, 0));
                copy_band_to(root, w, slot, n, d);
                CK(cudaEventRecord(w.h2d_done[slot], w.copy));
                CK(cudaStreamWaitEvent(w.compute, w.h2d_done[slot], 0));
                start_timing(w);
                rows_ptr = d;
                stride = (long long)rows * W;
            }
            launch_scan(rows_ptr, W, rows, stride, n, flags, w.d_err, w.compute);
            w.guarded += launch_backproject_raw(w.d_vol, g, w.z_begin, w.z_end, rows_ptr, stride,
                                               W, H, r0, rows, n, mats, flags, w.plan, opt,
                                               w.d_err, w.compute, resident ? w.tail_lo : 0,
                                               resident ? w.tail_hi : 0,
                                               w.count_culled ? w.d_counters : nullptr);
            CK(cudaEventRecord(w.raw_free[slot], w.compute));
        }
        ++nbatch;
        if (resident)
            std::memcpy(all_mats.data() + 12 * submitted, mats, 12 * sizeof(double) * n);
        submitted += n;
        slot = (slot + 1) % nslots;
    }

    // raw resident mode: resident projections [raw_pending, end) not yet
    // back-projected into the head planes
    int raw_pending = 0;
    int raw_last_launch = 0;

    // The deferred volume in one piece (every path but raw resident mode),
    // before the first batch or at finish.
    void upload_volume_whole() {
        if (!vol_src || !vchunks.empty())
            return;
        Worker& w = *workers[0];
        CK(cudaSetDevice(w.device));
        const size_t slab = (size_t)g.edge_voxels * g.edge_voxels * (w.z_end - w.z_begin);
        CK(cudaEventRecord(w.c_beg, w.copy));
        xfer.upload(w.d_vol, vol_src, slab * sizeof(float), w.copy, w.xfer_ev);
        launch_check_finite(w.d_vol, (long long)slab, w.d_err, w.copy, 4); // Volume::validate
        CK(cudaEventRecord(w.c_end, w.copy));
        CK(cudaStreamWaitEvent(w.compute, w.c_end, 0));
        vol_src = nullptr;
    }

    // Raw resident mode, one worker: the deferred volume's z-chunks (see
    // VolChunk). Head chunks of ~1/8 of the head planes in z order, aligned
    // to the staged kernel's z-blocks, then the tail (needed only at finish).
    void plan_volume_chunks() {
        Worker& w = *workers[0];
        choose_tails(est_mats, est_n);
        const int gs = kTR;
        int nchunks = 8;
        if (const char* e = std::getenv("CBB_VOL_CHUNKS")) // experiments
            nchunks = std::max(1, std::atoi(e));
        const int head = (w.z_end - w.z_begin) - (w.tail_hi - w.tail_lo);
        const int cp = std::max(gs, (head / nchunks + gs - 1) / gs * gs);
        auto add = [&](int a, int b, bool tail) {
            for (int z = a; z < b; z += cp) {
                VolChunk c;
                c.z0 = z;
                c.z1 = tail ? b : std::min(z + cp, b);
                c.tail = tail;
                CK(cudaEventCreateWithFlags(&c.ready, cudaEventDisableTiming));
                vchunks.push_back(c);
                if (tail)
                    break;
            }
        };
        CK(cudaSetDevice(w.device));
        add(w.z_begin, w.tail_lo, false);
        add(w.tail_hi, w.z_end, false);
        add(w.tail_lo, w.tail_hi, true);
        if (std::getenv("CBB_TRACE"))
            std::fprintf(stderr, "cbb: deferred volume in %zu chunks of %d planes (tail [%d, %d))\n",
                         vchunks.size(), cp, w.tail_lo, w.tail_hi);
    }

    // Queues the next `k` volume chunks on the copy stream (pageable: through
    // the staging chunks, this thread copying) with the finiteness check.
    void pump_volume(size_t k) {
        if (vchunks.empty())
            return;
        Worker& w = *workers[0];
        CK(cudaSetDevice(w.device));
        const size_t plane = (size_t)g.edge_voxels * g.edge_voxels;
        for (; k > 0 && vchunk_next < vchunks.size(); --k) {
            VolChunk& c = vchunks[vchunk_next++];
            const size_t off = plane * (c.z0 - w.z_begin), n = plane * (c.z1 - c.z0);
            xfer.upload_async(w.d_vol + off, vol_src + off, n * sizeof(float), w.copy, w.xfer_ev);
            // Volume::validate (proj/src/dataset.cpp:146-151): bit 4
            launch_check_finite(w.d_vol + off, (long long)n, w.d_err, w.copy, 4);
            CK(cudaEventRecord(c.ready, w.copy));
            c.issued = true;
        }
    }

    // launch_raw_pending with a chunked volume: projections [applied, end)
    // into each run of uploaded head chunks with equal `applied` (a run
    // spanning the tail skips it through the kernel's gap), i.e. one launch
    // for the chunks that kept up and one for those that just arrived.
    void launch_chunks_pending(int end) {
        Worker& w = *workers[0];
        CK(cudaSetDevice(w.device));
        const size_t plane = (size_t)g.edge_voxels * g.edge_voxels;
        for (auto& c : vchunks)
            if (c.issued && c.ready) {
                CK(cudaStreamWaitEvent(w.compute, c.ready, 0));
                // waited once: the compute stream is ordered after it from now on
                CK(cudaEventDestroy(c.ready));
                c.ready = nullptr;
            }
        size_t i = 0;
        while (i < vchunks.size()) {
            VolChunk& a = vchunks[i];
            if (a.tail || !a.issued || a.applied >= end) {
                ++i;
                continue;
            }
            size_t j = i + 1;
            int z1 = a.z1;
            while (j < vchunks.size() && !vchunks[j].tail && vchunks[j].issued &&
                   vchunks[j].applied == a.applied &&
                   (vchunks[j].z0 == z1 || (z1 == w.tail_lo && vchunks[j].z0 == w.tail_hi))) {
                z1 = vchunks[j].z1;
                ++j;
            }
            const int from = a.applied;
            const bool gap = a.z0 < w.tail_lo && z1 > w.tail_hi;
            w.guarded += launch_backproject_raw(
                w.d_vol + plane * (a.z0 - w.z_begin), g, a.z0, z1,
                static_cast<const float*>(w.d_packed_all) + (size_t)from * W * H,
                (long long)W * H, W, H, 0, H, end - from, all_mats.data() + 12 * (size_t)from,
                w.d_flags_all + from, w.plan, opt, w.d_err, w.compute, gap ? w.tail_lo : 0,
                gap ? w.tail_hi : 0, w.count_culled ? w.d_counters : nullptr);
            for (size_t k = i; k < j; ++k)
                vchunks[k].applied = end;
            i = j;
        }
    }

    void launch_raw_pending(int end) {
        if (!vchunks.empty()) {
            if (end > raw_pending)
                raw_last_launch = end - raw_pending;
            launch_chunks_pending(end);
            raw_pending = std::max(raw_pending, end);
            return;
        }
        if (end <= raw_pending)
            return;
        Worker& w = *workers[0];
        CK(cudaSetDevice(w.device));
        const int n = end - raw_pending;
        raw_last_launch = n;
        w.guarded += launch_backproject_raw(
            w.d_vol, g, w.z_begin, w.z_end,
            static_cast<const float*>(w.d_packed_all) + (size_t)raw_pending * W * H,
            (long long)W * H, W, H, 0, H, n, all_mats.data() + 12 * (size_t)raw_pending,
            w.d_flags_all + raw_pending, w.plan, opt, w.d_err, w.compute, w.tail_lo, w.tail_hi,
            w.count_culled ? w.d_counters : nullptr);
        raw_pending = end;
    }

    // host time spent issuing batches (CBB_TRACE: printed per call), the
    // single-thread issue cost that bounds a multi-GPU batch rate
    double issue_ms_sum = 0.0, issue_ms_max = 0.0;
    uint64_t issue_count = 0;

    void issue(const float* src, const double* mats, int n, int stage = -1) {
        const auto t0 = std::chrono::steady_clock::now();
        if (vol_src) { // the deferred volume goes ahead of the batch (VolChunk)
            static const int per_batch = std::getenv("CBB_VOL_PER_BATCH")
                                             ? std::max(1, std::atoi(std::getenv("CBB_VOL_PER_BATCH")))
                                             : 1;
            if (vchunks.empty())
                upload_volume_whole();
            else
                pump_volume((size_t)per_batch);
        }
        if (raw_mode)
            issue_raw(src, mats, n, stage);
        else
            issue_packed(src, mats, n, stage);
        const double ms = std::chrono::duration<double, std::milli>(
                              std::chrono::steady_clock::now() - t0).count();
        issue_ms_sum += ms;
        issue_ms_max = std::max(issue_ms_max, ms);
        ++issue_count;
    }

    void issue_packed(const float* src, const double* mats, int n, int stage) {
        NvtxRange range("cbb batch");
        const size_t bytes = raw_bytes_per_proj * n;
        // Batch k is uploaded once, by the root worker k mod G. Each other
        // worker packs its row band straight out of the root's raw slot over
        // peer memory (pack_quads' loads cross NVLink: the transfer and the
        // layout transform are one kernel), or, without peer access, first
        // copies the band rows (cudaMemcpy3DPeerAsync) and packs locally.
        const int G = (int)workers.size();
        Worker& root = *workers[nbatch % G];
        // Slot reuse. The root's raw[slot] may still be read by the previous
        // batch that used it: every worker's pack (peer packs read it
        // directly; all record raw_free[slot]) and the other workers' band
        // copies out of it (recorded as their h2d_done[slot]). A non-root
        // worker writes only its own raw[slot], and only on the band-copy
        // path, after its own pack of that slot's previous use (raw_free).
        // About 3G stream-event waits per batch (was G(2G-1): 120 at G = 8,
        // 0.17 ms of host issue time per batch, profiles/issue_time_r2.txt).
        CK(cudaSetDevice(root.device));
        for (auto& o : workers) {
            CK(cudaStreamWaitEvent(root.copy, o->raw_free[slot], 0));
            if (o.get() != &root)
                CK(cudaStreamWaitEvent(root.copy, o->h2d_done[slot], 0));
        }
        if (!peer_pack)
            for (auto& w : workers)
                if (w.get() != &root) {
                    CK(cudaSetDevice(w->device));
                    CK(cudaStreamWaitEvent(w->copy, w->raw_free[slot], 0));
                }
        CK(cudaSetDevice(root.device));
        CK(cudaMemcpyAsync(root.d_raw[slot], src, bytes, cudaMemcpyHostToDevice, root.copy));
        CK(cudaEventRecord(root.h2d_done[slot], root.copy));
        if (stage >= 0) {
            CK(cudaEventRecord(root.stage_read[stage], root.copy));
            stage_owner[stage] = (int)(nbatch % G);
        }
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
            if (peer_pack) {
                CK(cudaStreamWaitEvent(w->compute, ready, 0));
            } else {
                CK(cudaStreamWaitEvent(w->copy, ready, 0));
                copy_band(root, *w, slot, n);
                CK(cudaEventRecord(w->h2d_done[slot], w->copy));
                CK(cudaStreamWaitEvent(w->compute, w->h2d_done[slot], 0));
            }
            start_timing(*w);
        }
        // the tails are needed by the first back-projection only: choose them
        // once the first upload is already on its way
        if (resident && submitted == 0) {
            const auto t0 = std::chrono::steady_clock::now();
            choose_tails(est_mats ? est_mats : mats, est_mats ? est_n : n);
            if (std::getenv("CBB_TRACE"))
                std::fprintf(stderr, "cbb: choose_tails %.2f ms\n",
                             std::chrono::duration<double, std::milli>(
                                 std::chrono::steady_clock::now() - t0).count());
        }
        for (auto& w : workers) {
            CK(cudaSetDevice(w->device));
            void* packed = resident ? static_cast<char*>(w->d_packed_all) + w->pk_bytes * submitted
                                    : w->d_packed;
            if (w.get() == &root)
                launch_pack_band(w->d_raw[slot], 0, H, (long long)W * H, W, H, n, packed, w->band,
                                 w->compute, w->d_err);
            else if (peer_pack) // the root's full raw slot, read over peer memory
                launch_pack_band(root.d_raw[slot], 0, H, (long long)W * H, W, H, n, packed,
                                 w->band, w->compute, w->d_err);
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
        slot = (slot + 1) % nslots;
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
    void copy_band(const Worker& root, Worker& w, int s, int n) { copy_band_to(root, w, s, n, w.d_raw[s]); }
    void copy_band_to(const Worker& root, Worker& w, int s, int n, float* dst) {
        const RowBand& b = w.band;
        if (b.rn <= 0)
            return;
        cudaMemcpy3DPeerParms p = {};
        const size_t row_bytes = (size_t)b.rn * W * sizeof(float);
        p.srcPtr = make_cudaPitchedPtr(root.d_raw[s] + (size_t)b.r0 * W, raw_bytes_per_proj,
                                       row_bytes, n);
        p.srcDevice = root.device;
        p.dstPtr = make_cudaPitchedPtr(dst, row_bytes, row_bytes, n);
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
            w->pk_bytes = (size_t)quad_pitch_cells(W) * w->band.qn * 16 + kMetaBytes;
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

    // Blocks until no upload still reads the host staging slot s.
    void wait_stage(int s) {
        if (stage_owner[s] < 0)
            return;
        auto& w = *workers[stage_owner[s]];
        CK(cudaSetDevice(w.device));
        CK(cudaEventSynchronize(w.stage_read[s]));
    }

    // Pinned staging for pageable sources, allocated on first use only.
    void ensure_staging() {
        for (int s = 0; s < kStageSlots; ++s)
            if (!h_stage[s])
                h_stage[s] = HostPool::get().alloc(raw_bytes_per_proj * opt.batch);
    }

    void stage_one(const float* img, const double* m) {
        ensure_staging();
        if (stage_fill == 0)
            wait_stage(sslot);
        stream_copy(h_stage[sslot] + (size_t)stage_fill * W * H, img, raw_bytes_per_proj);
        std::memcpy(stage_mats.data() + 12 * (size_t)stage_fill, m, 12 * sizeof(double));
        if (++stage_fill == opt.batch)
            flush();
    }

    void flush() {
        if (stage_fill == 0)
            return;
        issue(h_stage[sslot], stage_mats.data(), stage_fill, sslot);
        sslot = (sslot + 1) % kStageSlots;
        stage_fill = 0;
    }

    // Size of the batch starting at projection `first` of a stream: 4, 4, 8,
    // 16, ... up to opt.batch, so the first back-projection starts after a
    // small upload instead of a full batch (pipeline fill). Batch boundaries
    // do not change any result: each voxel still accumulates the projections
    // one by one in stack order. The ramp's three extra launches each re-read
    // and re-write the slab (~2 x slab bytes at ~6.5 TB/s) while it saves the
    // upload of (batch - 4) projections (~55 GB/s): no ramp when that costs
    // more (config 3's 4.3 GB slab: 631 vs 633 ms end to end; config 2:
    // 86.0 with the ramp vs 87.9 ms without).
    int batch_at(int first, int count) const {
        if (ramp_ < 0) {
            size_t slab = 0;
            for (auto& w : workers)
                slab = std::max(slab, (size_t)(w->z_end - w->z_begin) * g.edge_voxels *
                                          g.edge_voxels * sizeof(float));
            const double cost = 3.0 * 2.0 * (double)slab / 6.5e12;
            const double gain = (double)std::max(0, opt.batch - 4) * W * H * 4.0 / 55e9;
            ramp_ = gain > cost ? 4 : opt.batch;
            if (const char* e = std::getenv("CBB_RAMP")) // experiments: first batch size
                ramp_ = std::max(1, std::atoi(e));
        }
        return std::min({opt.batch, std::max(ramp_, first), count - first});
    }
    mutable int ramp_ = -1; // smallest first batch, chosen on first use

    // Whole-stack submission straight from the caller's buffer: pinned
    // buffers are copied asynchronously in place, pageable ones are staged
    // through the pinned staging ring (kStageSlots buffers).
    // First submission of a stack whose matrices are all known: row bands,
    // resident mode, tail estimate.
    void begin_stack(const double* mats, int count) {
        if (submitted != 0)
            return;
        NvtxRange range("cbb setup (bands, resident)");
        const auto t0 = std::chrono::steady_clock::now();
        set_bands(mats, count);
        if (tma_path_enabled()) {
            raw_mode = true;
            for (auto& w : workers) {
                w->plan = plan_tma(g, W, H, w->z_begin, w->z_end, mats, count);
                raw_mode = raw_mode && w->plan.ok;
            }
            if (raw_mode) {
                for (auto& w : workers) {
                    // one device: the whole detector (uploads land in place);
                    // several: each keeps its slab's band of raw rows
                    if (workers.size() == 1)
                        w->band = RowBand::full(H);
                    if (w->band.rn < 1) { // footprint off the detector: hold one row
                        // (a tensor map needs >= 1 row; extra rows hold true pixels)
                        w->band.r0 = std::min(std::max(w->band.r0, 0), H - 1);
                        w->band.rn = 1;
                    }
                    w->pk_bytes = (size_t)w->band.rn * W * sizeof(float); // resident rows
                    CK(cudaSetDevice(w->device));
                    w->d_flags = static_cast<unsigned*>(
                        DevicePool::get().alloc(w->device, sizeof(unsigned) * opt.batch));
                }
            }
            if (std::getenv("CBB_TRACE"))
                for (auto& w : workers)
                    std::fprintf(stderr,
                                 "cbb: raw mode %d, device %d slab [%d, %d): tma pitch %d bh %d "
                                 "stages %d, rows [%d, %d)\n",
                                 (int)raw_mode, w->device, w->z_begin, w->z_end, w->plan.pitch,
                                 w->plan.bh, w->plan.stages, w->band.r0, w->band.r0 + w->band.rn);
        }
        enable_resident(count);
        if (raw_mode && resident)
            for (auto& w : workers) {
                CK(cudaSetDevice(w->device));
                w->d_flags_all = static_cast<unsigned*>(
                    DevicePool::get().alloc(w->device, sizeof(unsigned) * count));
            }
        est_mats = mats;
        est_n = count;
        if (vol_src && raw_mode && resident && workers.size() == 1)
            plan_volume_chunks();
        if (std::getenv("CBB_TRACE"))
            std::fprintf(stderr, "cbb: enable_resident %.2f ms\n",
                         std::chrono::duration<double, std::milli>(
                             std::chrono::steady_clock::now() - t0).count());
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
                wait_stage(sslot);
                parallel_memcpy(h_stage[sslot], src, raw_bytes_per_proj * n);
                issue(h_stage[sslot], mats + 12 * (size_t)first, n, sslot);
                sslot = (sslot + 1) % kStageSlots;
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
        for (int first = 0, n = 0; first < count; first += n) {
            n = batch_at(first, count);
            wait_stage(sslot);
            float* dst = h_stage[sslot];
            // gathered by the copy pool in ~2 MB pieces of the images
            const size_t per_img = std::max<size_t>(1, raw_bytes_per_proj / (size_t(2) << 20));
            const size_t piece = (raw_bytes_per_proj + per_img - 1) / per_img;
            CopyPool::get().run_pieces((size_t)n * per_img, [&](size_t i) {
                const size_t j = i / per_img, off = (i % per_img) * piece;
                if (off < raw_bytes_per_proj)
                    stream_copy(reinterpret_cast<char*>(dst + (size_t)j * W * H) + off,
                                reinterpret_cast<const char*>(imgs[first + j]) + off,
                                std::min(piece, raw_bytes_per_proj - off));
            });
            issue(dst, mats + 12 * (size_t)first, n, sslot);
            sslot = (sslot + 1) % kStageSlots;
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
        const int nt = (int)std::min<unsigned>(copy_threads(), hw);
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
            wait_stage(sslot);
            t_wait += ms_since(t0);
            t0 = now();
            float* dst = h_stage[sslot];
            std::vector<std::thread> pool;
            std::vector<int> bad(nt, 0);
            for (int t = 0; t < nt; ++t)
                pool.emplace_back([&, t] {
                    for (int j = t; j < n; j += nt) {
                        const uint64_t off = header_bytes + rec_bytes * (uint64_t)(first + j);
                        if (map) {
                            std::memcpy(mats.data() + 12 * (size_t)j, map + off, 96);
                            stream_copy(dst + (size_t)j * W * H, map + off + 96, rec_bytes - 96);
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
            issue(dst, mats.data(), n, sslot);
            sslot = (sslot + 1) % kStageSlots;
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
        // the reference validates the images (stack.validate) before the
        // volume (backproject_reference), kernel_ref.cpp:6-7, 33
        if (err_any & 2) // ProjectionImage::validate (proj/src/dataset.cpp:123-129)
            fail(CBB_ERR_INVALID, "ProjectionImage contains non-finite values");
        if (err_any & 4) // Volume::validate (proj/src/dataset.cpp:146-151)
            fail(CBB_ERR_INVALID, "Volume contains non-finite values");
        if (err_any & 1)
            fail(CBB_ERR_GEOMETRY, "backprojection hit a voxel with w == 0");
    }

    // Waits for all work, checks the error flags, downloads slabs into vol_out.
    void finish(float* vol_out) {
        NvtxRange range("cbb finish");
        flush();
        if (vol_src) { // nothing submitted, or chunks still to upload
            if (vchunks.empty())
                upload_volume_whole();
            else
                pump_volume(vchunks.size());
        }
        if (raw_mode && resident && workers.size() == 1)
            launch_raw_pending((int)submitted);
        if (std::getenv("CBB_TRACE") && issue_count)
            std::fprintf(stderr,
                         "cbb: %d worker(s), %s mode: %llu batches issued, host issue %.3f ms "
                         "mean / %.3f ms max per batch\n",
                         (int)workers.size(), raw_mode ? "raw" : "packed",
                         (unsigned long long)issue_count, issue_ms_sum / issue_count,
                         issue_ms_max);
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
        // the tail in two parts: its last 8 planes go last, so that only
        // their download (not the whole tail's) follows the final kernel --
        // when that saves more (tail download at ~50 GB/s) than the second
        // part's extra launches cost (~30 us each): config 3 625 vs 631 ms
        // end to end; configs 0 and 1 lose ~0.7 ms if split.
        const int nlaunch = (resident_count + opt.batch - 1) / opt.batch;
        // the last part is one z-block group (8 planes for the gather
        // kernel, 12 for the staged kernel: no partly empty z-blocks)
        const int gs = tail_group();
        auto tail_mid = [&](const Worker& w) {
            const double saved_ms = (double)(w.tail_hi - w.tail_lo - gs) * plane * 4.0 / 50e6;
            if (std::getenv("CBB_TAIL_NOSPLIT")) // experiments
                return w.tail_hi;
            return w.tail_hi - w.tail_lo >= 2 * gs && saved_ms > 0.03 * nlaunch ? w.tail_hi - gs
                                                                                : w.tail_hi;
        };
        for (auto& w : workers) {
            CK(cudaSetDevice(w->device));
            if (trace && w == workers.front()) {
                CK(cudaEventCreate(&t_tail));
                CK(cudaEventRecord(t_tail, w->compute));
            }
            const int mid = tail_mid(*w);
            for (const auto& part : {std::make_pair(w->tail_lo, mid),
                                     std::make_pair(mid, w->tail_hi)}) {
                if (part.second > part.first && raw_mode)
                    w->guarded += launch_backproject_raw(
                        w->d_vol + plane * (part.first - w->z_begin), g, part.first,
                        part.second, static_cast<const float*>(w->d_packed_all),
                        (long long)w->band.rn * W, W, H, w->band.r0, w->band.rn, resident_count,
                        all_mats.data(), w->d_flags_all, w->plan, opt, w->d_err, w->compute, 0,
                        0, w->count_culled ? w->d_counters : nullptr);
                else if (part.second > part.first)
                    w->guarded += launch_backproject(
                        w->d_vol + plane * (part.first - w->z_begin), g, part.first,
                        part.second, w->d_packed_all, W, H, resident_count, all_mats.data(), opt,
                        w->d_err, w->compute, 0, 0, &w->band,
                        w->count_culled ? w->d_counters : nullptr);
                if (part.second == mid)
                    CK(cudaEventRecord(w->tail_mid_done, w->compute));
            }
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
                CK(cudaStreamWaitEvent(w->copy, w->tail_mid_done, 0));
                d2h(*w, w->tail_lo, tail_mid(*w));
            }
            for (auto& w : workers) {
                CK(cudaSetDevice(w->device));
                CK(cudaStreamWaitEvent(w->copy, w->tail_done, 0));
                d2h(*w, tail_mid(*w), w->tail_hi);
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
