// FP64 FMA throughput of the B200 (the ramp filter's roofline denominator):
// 8 independent DFMA chains per thread, 148 x 8 blocks of 256 threads.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
        x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            x[k] = fma(x[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
        s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    double* out;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    const double flops = 2.0 * 8 * iters * (double)blocks * threads;
    printf("FP64 FMA: %.2f TFLOP/s (%d SMs, best of 5, %.3f ms)\n", flops / (best * 1e-3) / 1e12, sms,
           best);
    return 0;
}
