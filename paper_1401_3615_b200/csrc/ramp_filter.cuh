// ramp_filter.cuh -- FDK filtering step upstream of the back-projection
// (SURVEY 8(f) rank 1): row-wise Shepp-Logan ramp filter
//     h[n] = -2 / (pi^2 * tau * (4 n^2 - 1)),  tau = detector pixel pitch,
// applied as a linear convolution through a zero-padded float64 FFT of
// length nfft >= 2W (power of two), then rounded to float32 -- the same
// definition the synthetic-input generator uses (paper_1401_3615_b200/synth.py).
// The reference treats projections as pre-filtered, so this stage
// has no reference counterpart; its parity check is a float64 numpy FFT.
//
// Device work: rows are widened to float64 into the padded buffer, cuFFT
// D2Z, pointwise multiply by the cached spectrum of h, Z2D, then scale 1/nfft
// and narrow the first W samples to float32.
#pragma once

#include <cmath>
#include <cstdlib>
#include <cufft.h>
#include <map>
#include <mutex>
#include <tuple>

#include "../../include/conebeam_b200.h"
#include "ramp_fft.cuh"

namespace cbb {

// defined in cbb_runtime.cu
[[noreturn]] void fail(cbb_status s, const char* fmt, ...);
void check_cuda(cudaError_t e, const char* what);
extern thread_local uint64_t g_launches;

__global__ void rf_widen(const float* __restrict__ raw, double* __restrict__ pad, int W, int nfft,
                         long long rows) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long total = rows * nfft;
    if (i >= total)
        return;
    const long long r = i / nfft;
    const int c = (int)(i - r * nfft);
    pad[i] = c < W ? (double)raw[r * W + c] : 0.0;
}

__global__ void rf_multiply(double2* __restrict__ spec, const double2* __restrict__ h, int nc,
                            long long rows) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= rows * nc)
        return;
    const double2 a = spec[i];
    const double2 b = h[i % nc];
    spec[i] = make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__global__ void rf_narrow(const double* __restrict__ pad, float* __restrict__ out, int W, int nfft,
                          long long rows, double scale) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= rows * W)
        return;
    const long long r = i / W;
    const int c = (int)(i - r * W);
    out[i] = (float)(pad[r * nfft + c] * scale);
}

// h[n] at wrapped index (n in (-nfft/2, nfft/2]).
__global__ void rf_kernel_taps(double* h, int nfft, double tau) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nfft)
        return;
    const double n = i <= nfft / 2 ? (double)i : (double)(i - nfft);
    h[i] = -2.0 / (M_PI * M_PI * tau * (4.0 * n * n - 1.0));
}

inline int rf_nfft(int W) {
    int n = 1;
    while (n < 2 * W)
        n *= 2;
    return n;
}

// Cached per (device, nfft, rows, tau): plans, work buffers, spectrum of h.
// The work buffers (and cuFFT's own work areas) are shared by every stream of
// the device, so uses are chained on the GPU: each use waits for `last` (the
// previous use, possibly on another stream) and records it when done.
struct RampPlan {
    cudaEvent_t last = nullptr;
    cufftHandle fwd = 0, inv = 0;
    double* pad = nullptr;
    double2* spec = nullptr;
    double2* h = nullptr;
    int nfft = 0;
    long long rows = 0;
};

class RampPlans {
  public:
    static RampPlans& get() {
        static RampPlans p;
        return p;
    }
    // Returns a plan for up to `rows` rows of width W; caller holds the lock.
    RampPlan& plan(int device, int W, long long rows, double tau, cudaStream_t st) {
        const int nfft = rf_nfft(W);
        auto key = std::make_tuple(device, nfft, rows, tau);
        auto it = plans_.find(key);
        if (it != plans_.end())
            return it->second;
        RampPlan p;
        p.nfft = nfft;
        p.rows = rows;
        const int nc = nfft / 2 + 1;
        check_cuda(cudaMalloc(&p.pad, sizeof(double) * nfft * rows), "cudaMalloc(ramp pad)");
        check_cuda(cudaMalloc(&p.spec, sizeof(double2) * nc * rows), "cudaMalloc(ramp spec)");
        check_cuda(cudaMalloc(&p.h, sizeof(double2) * nc), "cudaMalloc(ramp h)");
        int n[1] = {nfft};
        if (cufftPlanMany(&p.fwd, 1, n, nullptr, 1, nfft, nullptr, 1, nc, CUFFT_D2Z, (int)rows) !=
                CUFFT_SUCCESS ||
            cufftPlanMany(&p.inv, 1, n, nullptr, 1, nc, nullptr, 1, nfft, CUFFT_Z2D, (int)rows) !=
                CUFFT_SUCCESS)
            fail(CBB_ERR_INTERNAL, "cufftPlanMany failed (nfft %d, rows %lld)", nfft, rows);
        // spectrum of h: taps -> first row of pad, one-row D2Z
        cufftHandle one = 0;
        if (cufftPlan1d(&one, nfft, CUFFT_D2Z, 1) != CUFFT_SUCCESS)
            fail(CBB_ERR_INTERNAL, "cufftPlan1d failed");
        cufftSetStream(one, st);
        rf_kernel_taps<<<(nfft + 255) / 256, 256, 0, st>>>(p.pad, nfft, tau);
        if (cufftExecD2Z(one, p.pad, p.h) != CUFFT_SUCCESS)
            fail(CBB_ERR_INTERNAL, "cufftExecD2Z(h) failed");
        check_cuda(cudaStreamSynchronize(st), "ramp spectrum");
        cufftDestroy(one);
        check_cuda(cudaEventCreateWithFlags(&p.last, cudaEventDisableTiming), "ramp event");
        return plans_.emplace(key, p).first->second;
    }
    std::mutex mu;

  private:
    std::map<std::tuple<int, int, long long, double>, RampPlan> plans_;
};

constexpr long long kRampRows = 8192; // rows per FFT call (~0.5 GB of float64 work space)

// raw and out: count*H rows of W floats (device); may alias. cuFFT path,
// kept for detectors wider than the fused kernel's 2048 pixels (and as the
// comparison baseline, CBB_RAMP_CUFFT=1).
inline void ramp_filter_cufft(const float* raw, float* out, int W, int H, int count, double tau,
                              cudaStream_t st) {
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    const long long rows_total = (long long)H * count;
    auto& pl = RampPlans::get();
    std::lock_guard<std::mutex> lk(pl.mu);
    RampPlan& p = pl.plan(dev, W, kRampRows, tau, st);
    cufftSetStream(p.fwd, st);
    cufftSetStream(p.inv, st);
    check_cuda(cudaStreamWaitEvent(st, p.last, 0), "ramp: wait previous use");
    const int nc = p.nfft / 2 + 1;
    for (long long r0 = 0; r0 < rows_total; r0 += kRampRows) {
        const long long rows = std::min(kRampRows, rows_total - r0);
        const long long nw = rows * p.nfft;
        rf_widen<<<(unsigned)((nw + 255) / 256), 256, 0, st>>>(raw + r0 * W, p.pad, W, p.nfft, rows);
        if (rows < kRampRows) // zero the unused rows so the fixed-batch plan stays finite
            check_cuda(cudaMemsetAsync(p.pad + nw, 0, sizeof(double) * (kRampRows - rows) * p.nfft, st),
                       "cudaMemsetAsync(ramp)");
        if (cufftExecD2Z(p.fwd, p.pad, p.spec) != CUFFT_SUCCESS)
            fail(CBB_ERR_INTERNAL, "cufftExecD2Z failed");
        const long long nm = rows * nc;
        rf_multiply<<<(unsigned)((nm + 255) / 256), 256, 0, st>>>(p.spec, p.h, nc, rows);
        if (cufftExecZ2D(p.inv, p.spec, p.pad) != CUFFT_SUCCESS)
            fail(CBB_ERR_INTERNAL, "cufftExecZ2D failed");
        const long long no = rows * W;
        rf_narrow<<<(unsigned)((no + 255) / 256), 256, 0, st>>>(p.pad, out + r0 * W, W, p.nfft, rows,
                                                               1.0 / p.nfft);
        check_cuda(cudaGetLastError(), "ramp filter kernels");
        g_launches += 3;
    }
    check_cuda(cudaEventRecord(p.last, st), "ramp: record use");
}

} // namespace cbb

namespace cbb {

// The FDK filter stage: the fused shared-memory FFT kernel (ramp_fft.cuh)
// when the detector fits its N = 4096 transform, else cuFFT.
inline void ramp_filter_device(const float* raw, float* out, int W, int H, int count, double tau,
                               cudaStream_t st) {
    static const bool force_cufft = std::getenv("CBB_RAMP_CUFFT") != nullptr;
    if (ramp_fft_supported(W) && !force_cufft)
        ramp_fft_device(raw, out, W, H, count, tau, st);
    else
        ramp_filter_cufft(raw, out, W, H, count, tau, st);
}

} // namespace cbb
