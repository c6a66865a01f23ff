// Host -> device paths for PAGEABLE sources (the drop-in's per-image
// buffers and volume), measured on the GPU box:
//  1. staged: N threads memcpy pageable -> pinned (glibc memcpy vs
//     non-temporal AVX2 stores), alone and while a pinned H2D DMA runs;
//  2. the driver's own cudaMemcpy from pageable memory;
//  3. direct GPU reads of pageable memory (HMM / pageable memory access),
//     first and second touch;
//  4. cudaHostRegister cost.
// nvcc -O2 -gencode arch=compute_100a,code=sm_100a -Xcompiler -mavx2 -o host_paths host_paths.cu -lpthread
#include <immintrin.h>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#include <cuda_runtime.h>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void nt_copy(char* dst, const char* src, size_t n) {
    // dst 32-byte aligned (pinned allocations are page aligned; pieces of 2 MB)
    size_t i = 0;
    for (; i + 128 <= n; i += 128) {
        __m256i a = _mm256_loadu_si256((const __m256i*)(src + i));
        __m256i b = _mm256_loadu_si256((const __m256i*)(src + i + 32));
        __m256i c = _mm256_loadu_si256((const __m256i*)(src + i + 64));
        __m256i d = _mm256_loadu_si256((const __m256i*)(src + i + 96));
        _mm256_stream_si256((__m256i*)(dst + i), a);
        _mm256_stream_si256((__m256i*)(dst + i + 32), b);
        _mm256_stream_si256((__m256i*)(dst + i + 64), c);
        _mm256_stream_si256((__m256i*)(dst + i + 96), d);
    }
    std::memcpy(dst + i, src + i, n - i);
    _mm_sfence();
}

static double par_copy(char* dst, const char* src, size_t bytes, int nt, bool nt_store) {
    const double t0 = now();
    std::vector<std::thread> pool;
    const size_t piece = size_t(2) << 20;
    std::atomic<size_t> next{0};
    for (int t = 0; t < nt; ++t)
        pool.emplace_back([&] {
            for (size_t k; (k = next.fetch_add(1)) * piece < bytes;) {
                const size_t off = k * piece, len = std::min(piece, bytes - off);
                if (nt_store)
                    nt_copy(dst + off, src + off, len);
                else
                    std::memcpy(dst + off, src + off, len);
            }
        });
    for (auto& th : pool)
        th.join();
    return bytes / (now() - t0) / 1e9;
}

__global__ void read_kernel(const float4* __restrict__ src, float4* __restrict__ dst, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

int main() {
    const size_t bytes = size_t(1) << 30; // 1 GiB
    printf("hardware_concurrency %u\n", std::thread::hardware_concurrency());
    char* src = static_cast<char*>(aligned_alloc(4096, bytes));
    memset(src, 1, bytes);
    char* pinned = nullptr;
    cudaHostAlloc(&pinned, bytes, cudaHostAllocPortable);
    memset(pinned, 0, bytes);
    char* pinned2 = nullptr;
    cudaHostAlloc(&pinned2, bytes, cudaHostAllocPortable);
    memset(pinned2, 0, bytes);
    void* d = nullptr;
    cudaMalloc(&d, 2 * bytes);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);

    cudaEventRecord(a, st);
    cudaMemcpyAsync(d, pinned2, bytes, cudaMemcpyHostToDevice, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("H2D pinned alone: %.1f GB/s\n", bytes / (ms * 1e-3) / 1e9);

    for (bool nts : {false, true})
        for (int nt : {4, 8, 16, 32}) {
            double best = 0;
            for (int rep = 0; rep < 3; ++rep)
                best = std::max(best, par_copy(pinned, src, bytes, nt, nts));
            // with a concurrent DMA from another pinned buffer (4 x 1 GiB back to back)
            for (int k = 0; k < 4; ++k)
                cudaMemcpyAsync(d, pinned2, bytes, cudaMemcpyHostToDevice, st);
            cudaEventRecord(a, st);
            const double c = par_copy(pinned, src, bytes, nt, nts);
            cudaEventRecord(b, st);
            cudaStreamSynchronize(st);
            printf("%s threads %2d: %.1f GB/s alone, %.1f GB/s during DMA\n",
                   nts ? "nt-store" : "memcpy  ", nt, best, c);
        }

    // pipelined staged upload of 1 GiB (copy 64 MB pieces, DMA each), as ChunkedXfer
    for (bool nts : {false, true})
        for (int nt : {8, 16, 32}) {
            const size_t chunk = size_t(64) << 20;
            cudaEvent_t ev[2];
            cudaEventCreate(&ev[0]);
            cudaEventCreate(&ev[1]);
            cudaDeviceSynchronize();
            const double t0 = now();
            int k = 0;
            for (size_t off = 0; off < bytes; off += chunk, k ^= 1) {
                cudaEventSynchronize(ev[k]);
                par_copy(pinned + k * chunk, src + off, chunk, nt, nts);
                cudaMemcpyAsync((char*)d + off, pinned + k * chunk, chunk, cudaMemcpyHostToDevice, st);
                cudaEventRecord(ev[k], st);
            }
            cudaStreamSynchronize(st);
            printf("staged upload %s threads %2d: %.1f GB/s\n", nts ? "nt-store" : "memcpy  ", nt,
                   bytes / (now() - t0) / 1e9);
        }

    {
        const double t0 = now();
        cudaMemcpy(d, src, bytes, cudaMemcpyHostToDevice);
        printf("cudaMemcpy from pageable: %.1f GB/s\n", bytes / (now() - t0) / 1e9);
    }

    int dev = 0, pma = 0, pmah = 0;
    cudaDeviceGetAttribute(&pma, cudaDevAttrPageableMemoryAccess, dev);
    cudaDeviceGetAttribute(&pmah, cudaDevAttrPageableMemoryAccessUsesHostPageTables, dev);
    printf("pageableMemoryAccess %d, usesHostPageTables %d\n", pma, pmah);
    if (pma) {
        char* hm = static_cast<char*>(aligned_alloc(4096, bytes));
        memset(hm, 2, bytes);
        for (int touch = 0; touch < 3; ++touch) {
            cudaEventRecord(a, st);
            read_kernel<<<148 * 8, 512, 0, st>>>((const float4*)hm, (float4*)d, bytes / 16);
            cudaEventRecord(b, st);
            const cudaError_t e = cudaStreamSynchronize(st);
            cudaEventElapsedTime(&ms, a, b);
            printf("GPU reads pageable (touch %d): %s %.1f GB/s\n", touch, cudaGetErrorString(e),
                   bytes / (ms * 1e-3) / 1e9);
        }
        // fresh memory, touched on the host just before (the realistic case)
        char* hm2 = static_cast<char*>(aligned_alloc(4096, bytes));
        memset(hm2, 3, bytes);
        cudaEventRecord(a, st);
        read_kernel<<<148 * 8, 512, 0, st>>>((const float4*)hm2, (float4*)d, bytes / 16);
        cudaEventRecord(b, st);
        cudaStreamSynchronize(st);
        cudaEventElapsedTime(&ms, a, b);
        printf("GPU reads fresh pageable: %.1f GB/s\n", bytes / (ms * 1e-3) / 1e9);
    }
    {
        char* hr = static_cast<char*>(aligned_alloc(4096, bytes));
        memset(hr, 4, bytes);
        const double t0 = now();
        const cudaError_t e = cudaHostRegister(hr, bytes, cudaHostRegisterDefault);
        const double t1 = now();
        cudaHostUnregister(hr);
        printf("cudaHostRegister 1 GiB: %s %.1f ms, unregister %.1f ms\n", cudaGetErrorString(e),
               (t1 - t0) * 1e3, (now() - t1) * 1e3);
    }
    return 0;
}
