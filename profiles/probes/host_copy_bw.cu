// Host memcpy bandwidth on the GPU box: pageable -> pinned (cudaHostAlloc)
// with 1..32 threads, the staging copy of cbb_reconstruct's pageable paths.
// nvcc -O2 -o host_copy_bw host_copy_bw.cu -lpthread
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <cuda_runtime.h>

int main() {
    const size_t bytes = size_t(1) << 31; // 2 GiB
    char* src = static_cast<char*>(malloc(bytes));
    memset(src, 1, bytes);
    char* pinned = nullptr;
    cudaHostAlloc(&pinned, bytes, cudaHostAllocPortable);
    memset(pinned, 0, bytes);
    char* pageable = static_cast<char*>(malloc(bytes));
    memset(pageable, 0, bytes);
    printf("hardware_concurrency %u\n", std::thread::hardware_concurrency());
    for (char* dst : {pinned, pageable}) {
        for (int nt : {1, 2, 4, 8, 16, 32}) {
            double best = 1e9;
            for (int rep = 0; rep < 3; ++rep) {
                auto t0 = std::chrono::steady_clock::now();
                std::vector<std::thread> pool;
                const size_t per = bytes / nt;
                for (int t = 0; t < nt; ++t)
                    pool.emplace_back([=] { memcpy(dst + t * per, src + t * per, per); });
                for (auto& th : pool) th.join();
                best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
            }
            printf("%s threads %2d: %.1f GB/s\n", dst == pinned ? "to pinned  " : "to pageable", nt, bytes / best / 1e9);
        }
    }
    // H2D from pinned for reference
    void* d = nullptr;
    cudaMalloc(&d, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaMemcpyAsync(d, pinned, bytes, cudaMemcpyHostToDevice);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("H2D pinned: %.1f GB/s\n", bytes / (ms * 1e-3) / 1e9);
    // cudaHostRegister cost for the pageable buffer
    auto t0 = std::chrono::steady_clock::now();
    cudaError_t e = cudaHostRegister(pageable, bytes, cudaHostRegisterDefault);
    double reg = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("cudaHostRegister 2 GiB: %.1f ms (%s)\n", reg * 1e3, cudaGetErrorString(e));
    cudaEventRecord(a);
    cudaMemcpyAsync(d, pageable, bytes, cudaMemcpyHostToDevice);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("H2D registered: %.1f GB/s\n", bytes / (ms * 1e-3) / 1e9);
    t0 = std::chrono::steady_clock::now();
    cudaHostUnregister(pageable);
    printf("cudaHostUnregister: %.1f ms\n", std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() * 1e3);
    return 0;
}
