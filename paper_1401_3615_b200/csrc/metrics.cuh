// metrics.cuh -- volume comparison on the GPU: the
// reference harness's quality_metrics (MSE, PSNR against max_ref,
// proj/src/bench.cpp:65-82) and max_relative_error (:92-102), plus the parity
// figures north_star states (relative L2, max |d| / (max r - min r)) and the
// count of bitwise-different voxels, without copying volumes to the host.
// Deterministic: fixed grid, per-block partials reduced in a fixed order.
#pragma once

#include <cfloat>

namespace cbb {

constexpr int kMetricBlocks = 592; // 148 SMs x 4
constexpr int kMetricThreads = 256;

struct MetricPartial {
    double sum_sq_diff, sum_sq_ref, max_abs, max_rel, ref_min, ref_max;
    unsigned long long bit_diff;
    double pad;
};

__global__ void __launch_bounds__(kMetricThreads)
metrics_partial(const float* __restrict__ test, const float* __restrict__ ref, long long n,
                double floor, MetricPartial* __restrict__ part) {
    double ssd = 0.0, ssr = 0.0, mabs = 0.0, mrel = 0.0, rmin = DBL_MAX, rmax = -DBL_MAX;
    unsigned long long nd = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const float tf = test[i], rf = ref[i];
        const double r = rf, d = (double)tf - r, ad = fabs(d);
        ssd += d * d;
        ssr += r * r;
        mabs = fmax(mabs, ad);
        mrel = fmax(mrel, ad / (fabs(r) + floor));
        rmin = fmin(rmin, r);
        rmax = fmax(rmax, r);
        nd += __float_as_uint(tf) != __float_as_uint(rf);
    }
    __shared__ double s[6][kMetricThreads];
    __shared__ unsigned long long sn[kMetricThreads];
    const int t = threadIdx.x;
    s[0][t] = ssd; s[1][t] = ssr; s[2][t] = mabs; s[3][t] = mrel; s[4][t] = rmin; s[5][t] = rmax;
    sn[t] = nd;
    __syncthreads();
    for (int w = kMetricThreads / 2; w > 0; w >>= 1) {
        if (t < w) {
            s[0][t] += s[0][t + w];
            s[1][t] += s[1][t + w];
            s[2][t] = fmax(s[2][t], s[2][t + w]);
            s[3][t] = fmax(s[3][t], s[3][t + w]);
            s[4][t] = fmin(s[4][t], s[4][t + w]);
            s[5][t] = fmax(s[5][t], s[5][t + w]);
            sn[t] += sn[t + w];
        }
        __syncthreads();
    }
    if (t == 0)
        part[blockIdx.x] = MetricPartial{s[0][0], s[1][0], s[2][0], s[3][0], s[4][0], s[5][0],
                                         sn[0], 0.0};
}

} // namespace cbb
