// memory.cuh -- device / pinned-host buffer caches and host<->device
// transfers of large pageable blocks.
// Internal part of libconebeam_b200.so: included, in this order, by
// cbb_runtime.cu (one translation unit: runtime_common.cuh, launch.cuh,
// memory.cuh, pipeline.cuh).
#pragma once

#include <immintrin.h> // stream_copy's AVX2 streaming stores

namespace cbb {

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

// Host copy into pinned staging, split over a few threads for large blocks
// (a single thread moves ~5-10 GB/s, below the PCIe H2D rate).
// Host threads for pageable <-> pinned copies: one memcpy stream reaches
// only ~5-10 GB/s, so these copies (the drop-in's pageable volume and
// per-image buffers) are spread over the host's cores; CBB_COPY_THREADS
// overrides (default: all hardware threads, at most 32).
inline unsigned copy_threads() {
    static const unsigned n = [] {
        if (const char* e = std::getenv("CBB_COPY_THREADS"))
            return (unsigned)std::max(1, std::atoi(e));
        return std::min(32u, std::max(1u, std::thread::hardware_concurrency()));
    }();
    return n;
}

// Host copies into or out of the pinned staging buffers with non-temporal
// (streaming) stores: the destination is not read back by this CPU soon
// (the DMA reads the staging buffer; a downloaded volume is far over L3), so
// the stores skip the read-for-ownership of every destination line. On the
// GPU box (16 cores, profiles/host_paths_r2.txt) 16 threads move 64.5 GB/s
// during a concurrent H2D DMA instead of glibc memcpy's 48.6, and a staged
// 1 GiB upload runs at 46.1 instead of 38.6 GB/s. Plain memcpy without AVX2.
__attribute__((target("avx2"))) static void stream_copy_avx2(char* d, const char* s, size_t n) {
    const size_t head = std::min(n, (size_t)((32 - ((uintptr_t)d & 31)) & 31));
    std::memcpy(d, s, head);
    d += head;
    s += head;
    n -= head;
    size_t i = 0;
    for (; i + 128 <= n; i += 128) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 32));
        const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 64));
        const __m256i e = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 96));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), a);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 32), b);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 64), c);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 96), e);
    }
    std::memcpy(d + i, s + i, n - i);
    _mm_sfence(); // the streamed lines are globally visible before the DMA is queued
}

inline void stream_copy(void* dst, const void* src, size_t bytes) {
    static const bool avx2 = __builtin_cpu_supports("avx2") && !std::getenv("CBB_NO_STREAM_COPY");
    if (avx2 && bytes >= 4096)
        stream_copy_avx2(static_cast<char*>(dst), static_cast<const char*>(src), bytes);
    else
        std::memcpy(dst, src, bytes);
}

// Persistent copy workers (copy_threads() - 1 of them plus the caller):
// spawning threads per call cost ~0.1-0.2 ms, too much for the 16 MB chunks
// of the staged volume transfers. One job at a time (callers serialise).
class CopyPool {
  public:
    static CopyPool& get() {
        static CopyPool* p = created() = new CopyPool(copy_threads()); // never destroyed
        return *p;
    }
    static CopyPool*& created() { // null until first use (the unload hook checks it)
        static CopyPool* p = nullptr;
        return p;
    }
    void run(void* dst, const void* src, size_t bytes, size_t piece) {
        char* d = static_cast<char*>(dst);
        const char* s = static_cast<const char*>(src);
        run_pieces((bytes + piece - 1) / piece, [=](size_t i) {
            const size_t off = i * piece;
            stream_copy(d + off, s + off, std::min(piece, bytes - off));
        });
    }
    // fn(i) for i in [0, pieces), spread over the workers and the caller
    void run_pieces(size_t pieces, const std::function<void(size_t)>& fn) {
        if (pieces == 0)
            return;
        std::lock_guard<std::mutex> one(job_mu_);
        Job j;
        j.fn = &fn;
        j.pieces = j.left = pieces;
        {
            std::lock_guard<std::mutex> lk(mu_);
            job_ = &j;
            ++gen_;
        }
        cv_.notify_all();
        work(j);
        // the job lives on this stack: return only when no worker holds it
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [&] { return j.left == 0 && j.users == 0; });
        job_ = nullptr;
    }
    // library unload (dlclose): wake the workers and wait until they left
    // this library's code
    void shutdown() {
        std::unique_lock<std::mutex> lk(mu_);
        stop_ = true;
        cv_.notify_all();
        done_.wait_for(lk, std::chrono::seconds(2), [&] { return live_ == 0; });
    }

  private:
    struct Job {
        const std::function<void(size_t)>* fn = nullptr;
        size_t pieces = 0, left = 0; // left, users: under mu_
        int users = 0;
        std::atomic<size_t> next{0};
    };
    explicit CopyPool(unsigned nt) {
        live_ = nt > 1 ? nt - 1 : 0;
        for (unsigned i = 1; i < nt; ++i)
            std::thread([this] { loop(); }).detach();
    }
    void work(Job& j) {
        size_t did = 0;
        for (size_t i; (i = j.next.fetch_add(1)) < j.pieces;) {
            (*j.fn)(i);
            ++did;
        }
        if (did) {
            std::lock_guard<std::mutex> lk(mu_);
            j.left -= did;
            if (j.left == 0)
                done_.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            Job* j = nullptr;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) {
                    --live_;
                    done_.notify_all();
                    return;
                }
                seen = gen_;
                j = job_; // null: that job already finished
                if (!j)
                    continue;
                ++j->users;
            }
            work(*j);
            std::lock_guard<std::mutex> lk(mu_);
            if (--j->users == 0 && j->left == 0)
                done_.notify_all();
        }
    }
    std::mutex job_mu_, mu_;
    std::condition_variable cv_, done_;
    Job* job_ = nullptr;
    uint64_t gen_ = 0;
    unsigned live_ = 0;
    bool stop_ = false;
};

__attribute__((destructor)) static void copy_pool_unload() {
    if (CopyPool* p = CopyPool::created())
        p->shutdown();
}

void parallel_memcpy(void* dst, const void* src, size_t bytes) {
    const size_t kPiece = size_t(2) << 20;
    if (copy_threads() <= 1 || bytes <= kPiece) {
        stream_copy(dst, src, bytes);
        return;
    }
    // pieces of 2 MB, at least ~4 per thread for balance
    const size_t piece = std::max<size_t>(256 << 10, std::min(kPiece, bytes / (4 * copy_threads())));
    CopyPool::get().run(dst, src, bytes, (piece + 63) & ~size_t(63));
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
    const size_t kChunk = [] {
        const char* e = std::getenv("CBB_XFER_CHUNK_MB"); // experiments
        return size_t(e ? std::max(1, std::atoi(e)) : 64) << 20;
    }();
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
    // returns once every chunk has reached the device (pageable src)
    void upload(void* dst, const void* src, size_t bytes, cudaStream_t st, cudaEvent_t ev[2]) {
        if (bytes == 0)
            return;
        if (is_pinned(src)) {
            CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
            return;
        }
        ensure();
        const bool trace = std::getenv("CBB_TRACE") != nullptr;
        const auto t0 = std::chrono::steady_clock::now();
        double wait_ms = 0.0, copy_ms = 0.0;
        auto ms_since = [](std::chrono::steady_clock::time_point a) {
            return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a)
                .count();
        };
        int k = 0;
        for (size_t off = 0; off < bytes; off += kChunk, k ^= 1) {
            const size_t len = std::min(kChunk, bytes - off);
            auto ta = std::chrono::steady_clock::now();
            CK(cudaEventSynchronize(ev[k])); // buf[k]'s previous DMA finished
            wait_ms += ms_since(ta);
            ta = std::chrono::steady_clock::now();
            parallel_memcpy(buf[k], static_cast<const char*>(src) + off, len);
            copy_ms += ms_since(ta);
            CK(cudaMemcpyAsync(static_cast<char*>(dst) + off, buf[k], len,
                               cudaMemcpyHostToDevice, st));
            CK(cudaEventRecord(ev[k], st));
        }
        // the staging chunks are shared by every worker of the pipeline (the
        // events are not): drain them before the next upload may refill them
        CK(cudaEventSynchronize(ev[0]));
        CK(cudaEventSynchronize(ev[1]));
        if (trace)
            std::fprintf(stderr, "cbb: pageable upload %.1f MB in %.2f ms (host copies %.2f ms, "
                                 "waits %.2f ms)\n",
                         bytes / 1e6, ms_since(t0), copy_ms, wait_ms);
    }
    // upload() without the final drain, for one worker's deferred volume
    // chunks (Pipeline::pump_volume): returns once the last piece is queued;
    // a staging chunk is refilled only after its previous DMA (ev), and the
    // chunk to fill next carries over between calls.
    int next = 0;
    void upload_async(void* dst, const void* src, size_t bytes, cudaStream_t st,
                      cudaEvent_t ev[2]) {
        if (bytes == 0)
            return;
        if (is_pinned(src)) {
            CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
            return;
        }
        ensure();
        for (size_t off = 0; off < bytes; off += kChunk, next ^= 1) {
            const size_t len = std::min(kChunk, bytes - off);
            CK(cudaEventSynchronize(ev[next]));
            parallel_memcpy(buf[next], static_cast<const char*>(src) + off, len);
            CK(cudaMemcpyAsync(static_cast<char*>(dst) + off, buf[next], len,
                               cudaMemcpyHostToDevice, st));
            CK(cudaEventRecord(ev[next], st));
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

} // namespace cbb
