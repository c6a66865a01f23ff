// tma_unit.cu -- standalone check of the TMA box load used by bp_tma.cuh
// (cuTensorMapEncodeTiled + cp.async.bulk.tensor.3d + mbarrier), outside the
// library: loads a PITCH x BH box of a 3-D float tensor (with out-of-bounds
// parts) and compares it with the expected values on the host.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tma_unit tma_unit.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                         const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                         CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                         CUtensorMapFloatOOBfill);

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}

template <int VARIANT>
__global__ void k(const __grid_constant__ CUtensorMap map, const CUtensorMap* gmap, float* out,
                  int pitch, int bh, int x, int y, int z) {
    extern __shared__ __align__(1024) unsigned char sm[];
    float* dst = reinterpret_cast<float*>(sm);
    unsigned long long& bar = *reinterpret_cast<unsigned long long*>(sm + pitch * bh * 4);
    const CUtensorMap* mp = VARIANT == 5 ? gmap : &map;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
        if (VARIANT != 1)
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0 && VARIANT == 3) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar)) : "memory");
    } else if (threadIdx.x == 0 && VARIANT == 6) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                     "r"(0u)
                     : "memory");
    } else if (threadIdx.x == 0 && VARIANT == 7) {
        unsigned long long st;
        asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)),
                     "r"((unsigned)(pitch * bh * 4))
                     : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
                     "l"(reinterpret_cast<unsigned long long>(mp)), "r"(smem_u32(&bar)),
                     "r"(x), "r"(y), "r"(z)
                     : "memory");
        asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];" : "=l"(st) : "r"(smem_u32(&bar)) : "memory");
    } else if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                     "r"((unsigned)(pitch * bh * 4))
                     : "memory");
        if (VARIANT == 4)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                         " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
                         "l"(reinterpret_cast<unsigned long long>(mp)), "r"(smem_u32(&bar)),
                         "r"(x), "r"(y)
                         : "memory");
        else if (VARIANT == 2)
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                         " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
                         "l"(reinterpret_cast<unsigned long long>(mp)), "r"(smem_u32(&bar)),
                         "r"(x), "r"(y), "r"(z)
                         : "memory");
        else
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                         " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
                         "l"(reinterpret_cast<unsigned long long>(mp)), "r"(smem_u32(&bar)),
                         "r"(x), "r"(y), "r"(z)
                         : "memory");
    }
    asm volatile("{\n\t.reg .pred P1;\nWAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                 "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(&bar)),
                 "r"(0u)
                 : "memory");
    for (int i = threadIdx.x; i < pitch * bh; i += blockDim.x)
        out[i] = dst[i];
}

int main(int argc, char** argv) {
    const int variant = argc > 1 ? atoi(argv[1]) : 0;
    const int W = 1248, H = 960, N = 3;
    const int pitch = argc > 2 ? atoi(argv[2]) : 80, bh = argc > 3 ? atoi(argv[3]) : 34;
    const int x = argc > 4 ? atoi(argv[4]) : -7, y = argc > 5 ? atoi(argv[5]) : 940, z = 1;
    std::vector<float> h((size_t)W * H * N);
    for (size_t i = 0; i < h.size(); ++i)
        h[i] = (float)(i % 100003) + 0.5f;
    float *d, *o;
    cudaMalloc(&d, h.size() * 4);
    cudaMalloc(&o, pitch * bh * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    CUtensorMap map;
    const cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    const cuuint64_t strides[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4};
    const cuuint32_t box[3] = {(cuuint32_t)pitch, (cuuint32_t)bh, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r = ((Enc)f)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    const size_t smem = pitch * bh * 4 + 64;
    CUtensorMap* gmap;
    cudaMalloc(&gmap, sizeof map);
    cudaMemcpy(gmap, &map, sizeof map, cudaMemcpyHostToDevice);
    CUtensorMap map2 = map;
    if (variant == 4) { // rank-2 map over projection z only
        const cuuint64_t d2[2] = {(cuuint64_t)W, (cuuint64_t)H};
        const cuuint64_t s2[1] = {(cuuint64_t)W * 4};
        const cuuint32_t b2[2] = {(cuuint32_t)pitch, (cuuint32_t)bh};
        r = ((Enc)f)(&map2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d + (size_t)z * W * H, d2, s2, b2,
                     es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("encode2 %d\n", (int)r);
    }
    switch (variant) {
    case 0: k<0><<<1, 256, smem>>>(map, gmap, o, pitch, bh, x, y, z); break;
    case 1: k<1><<<1, 256, smem>>>(map, gmap, o, pitch, bh, x, y, z); break;
    case 2: k<2><<<1, 256, smem>>>(map, gmap, o, pitch, bh, x, y, z); break;
    case 3: k<3><<<1, 256, smem>>>(map, gmap, o, pitch, bh, x, y, z); break;
    case 4: k<4><<<1, 256, smem>>>(map2, gmap, o, pitch, bh, x, y, z); break;
    default: k<5><<<1, 256, smem>>>(map, gmap, o, pitch, bh, x, y, z); break;
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d kernel: %s\n", variant, cudaGetErrorString(e));
    if (e != cudaSuccess)
        return 1;
    std::vector<float> got(pitch * bh);
    cudaMemcpy(got.data(), o, got.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r2 = 0; r2 < bh; ++r2)
        for (int c = 0; c < pitch; ++c) {
            const int gx = x + c, gy = y + r2;
            const float want = (gx >= 0 && gx < W && gy >= 0 && gy < H)
                                   ? h[((size_t)z * H + gy) * W + gx]
                                   : 0.0f;
            bad += got[r2 * pitch + c] != want;
        }
    printf("variant %d mismatches %d of %d\n", variant, bad, pitch * bh);
    return bad != 0;
}
