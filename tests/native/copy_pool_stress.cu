// Stress test of cbb::parallel_memcpy (the persistent copy pool of
// memory.cuh): concurrent callers, random sizes, byte-exact copies.
// Built and run on the host by tests/test_copy_pool.py (no GPU needed).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <thread>
#include <vector>
#include <random>
#include <cuda_runtime.h>
#define CK(x) (void)(x)
namespace cbb { inline void check_cuda(cudaError_t, const char*) {} }
#include "memory.cuh"
int main() {
    std::mt19937_64 rng(1);
    std::vector<char> a(64 << 20), b(64 << 20);
    for (auto& c : a) c = (char)rng();
    // concurrent callers + many sizes
    std::atomic<int> bad{0};
    auto worker = [&](int id) {
        std::vector<char> src(8 << 20), dst(8 << 20);
        std::mt19937_64 r(id);
        for (int it = 0; it < 300; ++it) {
            size_t n = 1 + r() % src.size();
            for (size_t i = 0; i < n; i += 4096) src[i] = (char)r();
            cbb::parallel_memcpy(dst.data(), src.data(), n);
            if (std::memcmp(dst.data(), src.data(), n)) ++bad;
        }
    };
    // stream_copy (AVX2 streaming stores): every destination/source
    // misalignment and sizes around the 4 KB threshold and the 128 B loop
    for (size_t n : {0ul, 1ul, 31ul, 127ul, 4095ul, 4096ul, 4097ul, 4224ul, 65537ul, 1000003ul})
        for (int da = 0; da < 64; da += 3)
            for (int sa = 0; sa < 8; ++sa) {
                std::memset(b.data(), 0x5a, n + 256);
                cbb::stream_copy(b.data() + 64 + da, a.data() + sa, n);
                if (std::memcmp(b.data() + 64 + da, a.data() + sa, n)) ++bad;
                for (int i = 0; i < 64 + da; ++i) // nothing written before dst
                    if (b[i] != 0x5a) { ++bad; break; }
                for (int i = 0; i < 64; ++i) // nor after dst + n
                    if (b[64 + da + n + i] != 0x5a) { ++bad; break; }
            }
    std::vector<std::thread> ts;
    for (int i = 0; i < 4; ++i) ts.emplace_back(worker, i);
    for (int it = 0; it < 50; ++it) {
        cbb::parallel_memcpy(b.data(), a.data(), a.size());
        if (std::memcmp(a.data(), b.data(), a.size())) ++bad;
    }
    for (auto& t : ts) t.join();
    printf("bad %d threads %u\n", bad.load(), cbb::copy_threads());
    return bad != 0;
}
