// ramp_fft.cuh -- hand-written sm_100a FDK ramp filter: one fused kernel per
// stack, FP64 FFT convolution in shared memory.
//
// Same definition as ramp_filter.cuh (and the input generator,
// paper_1401_3615_b200/synth.py): every detector row is linearly convolved
// with the Shepp-Logan kernel h[n] = -2 / (pi^2 tau (4 n^2 - 1)), tau = pixel
// pitch, in float64, and rounded to float32. The cuFFT path it replaces
// (ramp_filter.cuh: widen rows to 4096 doubles in HBM, D2Z, spectrum
// multiply, Z2D, narrow) moved ~130 GB through HBM for config 2's 476k rows
// (27.7 ms, 34 % of a back-projection step; BENCH r2a). Here each row is read
// once and written once (8 B per pixel):
//
//   * two rows form one complex sequence z = x1 + i x2 (zero-padded to
//     N = 4096 >= 2W - 1, so the circular convolution equals the linear one on
//     the W outputs); h is real and even, so its spectrum H is real and
//     IFFT(FFT(z) H) = (x1 * h) + i (x2 * h): the two filtered rows come back
//     as the real and imaginary parts, with no split/merge step;
//   * the FFT is a radix-16 Stockham transform (16^3 = 4096) by 256 threads,
//     16 points per thread in registers: pass 1 loads the rows straight from
//     global memory (coalesced), the forward transform's last pass leaves
//     every thread holding exactly the 16 frequencies the inverse transform's
//     first pass needs, so the spectrum multiply and that pass happen in
//     registers; the inverse's last pass stores the W outputs (scaled by 1/N,
//     folded into H) straight to global memory. Shared memory (one complex
//     double plane, one pad element per 16) carries only the 4 remaining
//     exchanges.
//
// FP64 (64 lanes/clk/SM on B200) bounds it: ~370k FP64 ops per row pair.
// Detectors wider than 2048 pixels keep the cuFFT path.
#pragma once

#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "../../include/conebeam_b200.h"

namespace cbb {

[[noreturn]] void fail(cbb_status s, const char* fmt, ...);
void check_cuda(cudaError_t e, const char* what);
extern thread_local uint64_t g_launches;

constexpr int kRfN = 4096;                     // FFT length
constexpr int kRfT = 256;                      // threads per FFT (N / 16)
constexpr int kRfMaxW = 2048;                  // N >= 2W - 1
// XOR swizzle of the complex plane (16-byte elements, 8 per 128-byte bank
// row): the stride-16 writes of the first pass, the stride-256 reads and the
// Ns = 16 writes all hit 8 distinct bank groups per 8-lane phase, with no pad.
__host__ __device__ constexpr int rf_sw(int i) { return i ^ ((i >> 4) & 7); }
constexpr int kRfPlane = kRfN;                 // complex elements in the plane
// complex plane, spectrum (N/2 + 1, padded to N/2 + 2), 272 twiddle bases,
// then (STAGE) two stages of two prefetched rows of NZ * 256 floats
constexpr int kRfFixedBytes = kRfPlane * 16 + (kRfN / 2 + 2) * 8 + 272 * 16; // 86288 B
__host__ __device__ constexpr bool rf_stage(int nz) { return nz <= 6; }
__host__ __device__ constexpr int rf_smem_bytes(int nz) {
    return kRfFixedBytes + (rf_stage(nz) ? 2 * 2 * nz * kRfT * 4 : 0);
}

struct cd {
    double x, y;
};
__device__ __forceinline__ cd operator+(cd a, cd b) { return {a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ cd operator-(cd a, cd b) { return {a.x - b.x, a.y - b.y}; }
__device__ __forceinline__ cd cmul(cd a, cd b) {
    return {fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x)};
}

// DFT of 4 points in place; forward uses W4 = -i, inverse +i.
template <bool INV>
__device__ __forceinline__ void dft4(cd& a0, cd& a1, cd& a2, cd& a3) {
    const cd t0 = a0 + a2, t1 = a0 - a2, t2 = a1 + a3, t3 = a1 - a3;
    const cd rt3 = INV ? cd{-t3.y, t3.x} : cd{t3.y, -t3.x}; // (+-i) * t3
    a0 = t0 + t2;
    a2 = t0 - t2;
    a1 = t1 + rt3;
    a3 = t1 - rt3;
}

// v[m] *= W16^e (forward: exp(-2 pi i e / 16), inverse: conjugate), e < 16.
template <bool INV, int E>
__device__ __forceinline__ void w16(cd& v) {
    constexpr double C1 = 0.92387953251128674, S1 = 0.38268343236508978;
    constexpr double R2 = 0.70710678118654752;
    constexpr int e = E % 16;
    // exp(-2 pi i e/16) = cos - i sin; inverse flips the sign of sin
    constexpr double sg = INV ? -1.0 : 1.0;
    if (e == 0)
        return;
    if (e == 4) { // -i (forward) / +i (inverse)
        v = INV ? cd{-v.y, v.x} : cd{v.y, -v.x};
        return;
    }
    if (e == 8) {
        v = cd{-v.x, -v.y};
        return;
    }
    if (e == 2 || e == 6) { // (1 -+ i)/sqrt2 rotations
        const double c = e == 2 ? R2 : -R2, s = sg * R2;
        v = cd{fma(v.x, c, v.y * s), fma(v.y, c, -v.x * s)};
        return;
    }
    const double c = (e == 1 || e == 15) ? C1 : (e == 3 || e == 13) ? S1
                   : (e == 5 || e == 11) ? -S1 : (e == 7 || e == 9) ? -C1 : 0.0;
    const double s0 = (e == 1 || e == 7) ? S1 : (e == 3 || e == 5) ? C1
                    : (e == 9 || e == 15) ? -S1 : (e == 11 || e == 13) ? -C1 : 0.0;
    const double s = sg * s0;
    // (x + i y)(c - i s) = (x c + y s) + i (y c - x s)
    v = cd{fma(v.x, c, v.y * s), fma(v.y, c, -v.x * s)};
}

// 16-point DFT of v[0..15] (input in natural order). Output X[k] lands in
// v[4 (k % 4) + k / 4] (radix-4 x radix-4, n = 4 n1 + n2, k = k1 + 4 k2).
// NZ: inputs v[NZ..15] are known to be zero (the zero-padded half of the
// forward transform's first pass): step 1 skips them. QN: only outputs
// X[0..QN) are needed (the inverse's last pass keeps the W < N samples):
// step 3 computes only those.
template <bool INV, int NZ = 16, int QN = 16>
__device__ __forceinline__ void dft16(cd (&v)[16]) {
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) {
        const int nz = (NZ > n2) + (NZ > 4 + n2) + (NZ > 8 + n2) + (NZ > 12 + n2);
        if (nz >= 3) {
            dft4<INV>(v[n2], v[4 + n2], v[8 + n2], v[12 + n2]); // v[4 k1 + n2] = A[n2][k1]
        } else if (nz == 2) { // (a, b, 0, 0): a + b, a -+ i b, a - b, a +- i b
            const cd a = v[n2], b = v[4 + n2];
            const cd ib = INV ? cd{-b.y, b.x} : cd{b.y, -b.x};
            v[n2] = a + b;
            v[4 + n2] = a + ib;
            v[8 + n2] = a - b;
            v[12 + n2] = a - ib;
        } else if (nz == 1) { // (a, 0, 0, 0): a everywhere
            v[4 + n2] = v[n2];
            v[8 + n2] = v[n2];
            v[12 + n2] = v[n2];
        } else {
            v[n2] = v[4 + n2] = v[8 + n2] = v[12 + n2] = cd{0.0, 0.0};
        }
    }
    w16<INV, 1>(v[5]);
    w16<INV, 2>(v[6]);
    w16<INV, 3>(v[7]);
    w16<INV, 2>(v[9]);
    w16<INV, 4>(v[10]);
    w16<INV, 6>(v[11]);
    w16<INV, 3>(v[13]);
    w16<INV, 6>(v[14]);
    w16<INV, 9>(v[15]);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
        // outputs k = k1 + 4 k2 for k2 = 0..3 (QN: only those < QN)
        const int nk = (QN > k1) + (QN > 4 + k1) + (QN > 8 + k1) + (QN > 12 + k1);
        if (nk >= 3) {
            dft4<INV>(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
        } else if (nk >= 1) {
            const cd a0 = v[4 * k1], a1 = v[4 * k1 + 1], a2 = v[4 * k1 + 2], a3 = v[4 * k1 + 3];
            const cd t0 = a0 + a2, t2 = a1 + a3;
            v[4 * k1] = t0 + t2;
            if (nk == 2) {
                const cd t1 = a0 - a2, t3 = a1 - a3;
                const cd rt3 = INV ? cd{-t3.y, t3.x} : cd{t3.y, -t3.x};
                v[4 * k1 + 1] = t1 + rt3;
            }
        }
    }
}
__device__ __forceinline__ constexpr int x16(int k) { return 4 * (k % 4) + k / 4; }

// One Stockham pass over shared memory: read 16 points at stride 256,
// twiddle by w1^r (w1 = exp(-+2 pi i (j % NS) / (16 NS)), precomputed per
// thread), DFT16, write at stride NS (or leave the outputs in registers in
// natural order: v[q] = X[j + 256 q]).
template <bool INV, int NS, bool READ, bool WRITE, int NZ = 16, int QN = 16>
__device__ __forceinline__ void rf_pass(cd (&v)[16], double2* buf, const double2* tws, int j) {
    if (READ) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const double2 x = buf[rf_sw(j + r * kRfT)];
            v[r] = cd{x.x, x.y};
        }
        __syncthreads(); // every read done before this pass's writes
    }
    if (NS > 1) {
        // w1 = exp(-+2 pi i (j % NS) / (16 NS)) from the block's table
        const double2 t = tws[NS == 16 ? (j % 16) : 16 + j];
        const cd w1{t.x, INV ? -t.y : t.y};
        cd w = w1;
#pragma unroll
        for (int r = 1; r < 16; ++r) {
            v[r] = cmul(v[r], w);
            if (r < 15)
                w = cmul(w, w1);
        }
    }
    dft16<INV, NZ, QN>(v);
    if (WRITE) {
        const int base = (j / NS) * NS * 16 + (j % NS);
#pragma unroll
        for (int q = 0; q < 16; ++q)
            buf[rf_sw(base + q * NS)] = make_double2(v[x16(q)].x, v[x16(q)].y);
        __syncthreads();
    } else {
        cd o[16];
#pragma unroll
        for (int q = 0; q < 16; ++q)
            o[q] = v[x16(q)];
#pragma unroll
        for (int q = 0; q < 16; ++q)
            v[q] = o[q];
    }
}

// rows: `rows` rows of W floats (row-major, row r at raw + r * W); pairs of
// rows (2p, 2p+1) per iteration; grid-stride over pairs. spec: the real
// spectrum of h for k <= N/2 (it is even: H[N-k] = H[k]), scaled by 1/N.
// tw: exp(-2 pi i e / N), e < N. NZ = ceil(W / 256): inputs j + 256 r with
// r >= NZ are padding (and so are outputs with q >= NZ).
template <int NZ>
__global__ void __launch_bounds__(kRfT, 2)
ramp_fft_rows(const float* raw, float* out, int W, long long rows,
              const double* __restrict__ spec, const double2* __restrict__ tw) {
    extern __shared__ double2 rf_smem[];
    // complex plane (XOR-swizzled, see rf_sw)
    double2* buf = rf_smem;
    double* hs = reinterpret_cast<double*>(rf_smem + kRfPlane); // N/2 + 1 spectrum values
    // twiddle bases of the two twiddled passes: [0, 16) for Ns = 16
    // (exp(-2 pi i m / 256)), [16, 272) for Ns = 256 (exp(-2 pi i j / 4096))
    double2* tws = reinterpret_cast<double2*>(hs + kRfN / 2 + 2);
    // prefetch stages: rows of the next pair are copied while this one is
    // transformed (cp.async, 4-byte granules: any W)
    float* stg = reinterpret_cast<float*>(tws + 272);
    constexpr bool STAGE = rf_stage(NZ);
    constexpr int SROW = NZ * kRfT;
    const int j = threadIdx.x;
    for (int k = j; k <= kRfN / 2; k += kRfT)
        hs[k] = spec[k];
    tws[16 + j] = __ldg(tw + j);
    if (j < 16)
        tws[j] = __ldg(tw + j * (kRfN / 256));
    const long long pairs = (rows + 1) / 2;
    auto prefetch = [&](long long p, int s) {
        if (p < pairs) {
            const float* r1 = raw + (2 * p) * (long long)W;
            const int nrow = 2 * p + 1 < rows ? 2 : 1;
            for (int e = j; e < nrow * W; e += kRfT) {
                const int row = e >= W, n = e - row * W;
                const unsigned dst = (unsigned)__cvta_generic_to_shared(stg + (2 * s + row) * SROW + n);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(r1 + e));
            }
        }
        asm volatile("cp.async.commit_group;");
    };
    if (STAGE)
        prefetch(blockIdx.x, 0);
    __syncthreads();
    int s = 0;
    for (long long p = blockIdx.x; p < pairs; p += gridDim.x, s ^= 1) {
        const float* r1 = raw + (2 * p) * (long long)W;
        const bool two = 2 * p + 1 < rows;
        const float* r2 = r1 + W;
        cd v[16];
        if (STAGE) {
            prefetch(p + gridDim.x, s ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
            __syncthreads(); // this pair's rows are in stage s for every thread
            const float* a = stg + 2 * s * SROW;
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const int n = j + r * kRfT;
                const bool in = r < NZ && n < W;
                v[r] = cd{in ? (double)a[n] : 0.0, (in && two) ? (double)a[SROW + n] : 0.0};
            }
        } else {
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const int n = j + r * kRfT;
                const bool in = r < NZ && n < W;
                v[r] = cd{in ? (double)__ldg(r1 + n) : 0.0,
                          (in && two) ? (double)__ldg(r2 + n) : 0.0};
            }
        }
        // forward: Ns = 1 (from registers), 16, 256 (ends in registers)
        rf_pass<false, 1, false, true, NZ>(v, buf, tws, j);
        rf_pass<false, 16, true, true>(v, buf, tws, j);
        rf_pass<false, 256, true, false>(v, buf, tws, j);
        // spectrum multiply: thread j holds Z[j + 256 q] in v[q] -- exactly
        // the inverse's first-pass inputs (stride N/16 = 256)
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int k = j + q * kRfT;
            const double h = hs[k <= kRfN / 2 ? k : kRfN - k];
            v[q] = cd{v[q].x * h, v[q].y * h};
        }
        rf_pass<true, 1, false, true>(v, buf, tws, j);
        rf_pass<true, 16, true, true>(v, buf, tws, j);
        rf_pass<true, 256, true, false, 16, NZ>(v, buf, tws, j);
        float* o1 = out + (2 * p) * (long long)W;
#pragma unroll
        for (int q = 0; q < NZ; ++q) {
            const int n = j + q * kRfT;
            if (n < W) {
                o1[n] = (float)v[q].x;
                if (two)
                    o1[W + n] = (float)v[q].y;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// N = 2560 = 10 x 16 x 16 for detectors up to 1280 pixels (BASELINE configs
// 0-3: W = 1248): 0.59x the FP64 work of N = 4096. Mixed-radix Stockham,
// forward passes radix 10, 16, 16 and inverse passes 16, 16, 10, so the
// forward transform's last pass (radix 16, thread j < 160 holds
// Z[j + 160 q]) is again exactly the inverse's first pass, in registers, and
// the inverse's last pass (radix 10, stride 256) hands thread j the outputs
// y[j + 256 q] -- the same store pattern as the N = 4096 kernel.
// ---------------------------------------------------------------------------
constexpr int kRf2N = 2560;
constexpr int kRf2T16 = kRf2N / 16; // 160 threads in the radix-16 passes
constexpr int kRf2MaxW = 1280;      // N >= 2W - 1 and W <= 5 * 256

// 5-point DFT in place (forward W5 = exp(-2 pi i / 5); inverse conjugate).
template <bool INV>
__device__ __forceinline__ void dft5(cd& x0, cd& x1, cd& x2, cd& x3, cd& x4) {
    constexpr double C1 = 0.30901699437494745, C2 = -0.80901699437494742;
    constexpr double S1 = 0.95105651629515357, S2 = 0.58778525229247314;
    const cd t1 = x1 + x4, t2 = x2 + x3, t3 = x1 - x4, t4 = x2 - x3;
    const cd a1{fma(C2, t2.x, fma(C1, t1.x, x0.x)), fma(C2, t2.y, fma(C1, t1.y, x0.y))};
    const cd a2{fma(C1, t2.x, fma(C2, t1.x, x0.x)), fma(C1, t2.y, fma(C2, t1.y, x0.y))};
    const cd b1{fma(S2, t4.x, S1 * t3.x), fma(S2, t4.y, S1 * t3.y)};
    const cd b2{fma(-S1, t4.x, S2 * t3.x), fma(-S1, t4.y, S2 * t3.y)};
    // forward: X1 = a1 - i b1, X4 = a1 + i b1, X2 = a2 - i b2, X3 = a2 + i b2
    const cd ib1 = INV ? cd{-b1.y, b1.x} : cd{b1.y, -b1.x}; // -+ i b1
    const cd ib2 = INV ? cd{-b2.y, b2.x} : cd{b2.y, -b2.x};
    x0 = x0 + t1 + t2;
    x1 = a1 + ib1;
    x4 = a1 - ib1;
    x2 = a2 + ib2;
    x3 = a2 - ib2;
}

// v *= W10^e (forward exp(-2 pi i e / 10), inverse conjugate), 1 <= e <= 4.
template <bool INV, int E>
__device__ __forceinline__ void w10(cd& v) {
    constexpr double C[5] = {1.0, 0.80901699437494745, 0.30901699437494742,
                             -0.30901699437494734, -0.80901699437494734};
    constexpr double S[5] = {0.0, 0.58778525229247314, 0.95105651629515357,
                             0.95105651629515364, 0.58778525229247325};
    const double c = C[E], sn = INV ? -S[E] : S[E];
    // (x + i y)(c - i s) = (x c + y s) + i (y c - x s)
    v = cd{fma(v.x, c, v.y * sn), fma(v.y, c, -v.x * sn)};
}

// 10-point DFT of v[0..9] as 2 x 5 (n = 5 n1 + n2, k = k1 + 2 k2); output
// X[k] lands in v[5 (k % 2) + k / 2]. ZHI: inputs v[5..9] are zero (the
// zero-padded half of the forward transform's first pass).
template <bool INV, bool ZHI>
__device__ __forceinline__ void dft10(cd (&v)[16]) {
#pragma unroll
    for (int n2 = 0; n2 < 5; ++n2) {
        if (ZHI) {
            v[5 + n2] = v[n2];
        } else {
            const cd a = v[n2], b = v[5 + n2];
            v[n2] = a + b;
            v[5 + n2] = a - b;
        }
    }
    w10<INV, 1>(v[6]);
    w10<INV, 2>(v[7]);
    w10<INV, 3>(v[8]);
    w10<INV, 4>(v[9]);
    dft5<INV>(v[0], v[1], v[2], v[3], v[4]);
    dft5<INV>(v[5], v[6], v[7], v[8], v[9]);
}
__device__ __forceinline__ constexpr int x10(int k) { return 5 * (k % 2) + k / 2; }

// smem layout of the N = 2560 kernel: plane, spectrum (N/2 + 1 -> N/2 + 2),
// twiddle bases tw[0..256), tw[16 m] (m < 10), tw[10 m] (m < 16), then two
// prefetch stages of two 1280-float rows
constexpr int kRf2Bytes = kRf2N * 16 + (kRf2N / 2 + 2) * 8 + (256 + 10 + 16) * 16 +
                          2 * 2 * kRf2MaxW * 4; // 76208 B

template <bool INV, int NS>
__device__ __forceinline__ void rf2_twiddle16(cd (&v)[16], cd w1) {
    if (INV)
        w1.y = -w1.y;
    cd w = w1;
#pragma unroll
    for (int r = 1; r < 16; ++r) {
        v[r] = cmul(v[r], w);
        if (r < 15)
            w = cmul(w, w1);
    }
}

__global__ void __launch_bounds__(kRfT, 2)
ramp_fft2560_rows(const float* raw, float* out, int W, long long rows,
                  const double* __restrict__ spec, const double2* __restrict__ tw) {
    extern __shared__ double2 rf_smem[];
    double2* buf = rf_smem;
    double* hs = reinterpret_cast<double*>(rf_smem + kRf2N);
    double2* tw256 = reinterpret_cast<double2*>(hs + kRf2N / 2 + 2);
    double2* tw16x = tw256 + 256; // tw[16 m], m < 10: forward radix-16 pass, Ns = 10
    double2* tw10x = tw16x + 10;  // tw[10 m], m < 16: inverse radix-16 pass, Ns = 16
    float* stg = reinterpret_cast<float*>(tw10x + 16);
    constexpr int SROW = kRf2MaxW;
    const int j = threadIdx.x;
    const bool act16 = j < kRf2T16; // the radix-16 passes use 160 threads
    for (int k = j; k <= kRf2N / 2; k += kRfT)
        hs[k] = spec[k];
    tw256[j] = __ldg(tw + j);
    if (j < 10)
        tw16x[j] = __ldg(tw + 16 * j);
    if (j < 16)
        tw10x[j] = __ldg(tw + 10 * j);
    const long long pairs = (rows + 1) / 2;
    auto prefetch = [&](long long p, int s) {
        if (p < pairs) {
            const float* r1 = raw + (2 * p) * (long long)W;
            const int nrow = 2 * p + 1 < rows ? 2 : 1;
            for (int e = j; e < nrow * W; e += kRfT) {
                const int row = e >= W, n = e - row * W;
                const unsigned dst = (unsigned)__cvta_generic_to_shared(stg + (2 * s + row) * SROW + n);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(r1 + e));
            }
        }
        asm volatile("cp.async.commit_group;");
    };
    prefetch(blockIdx.x, 0);
    __syncthreads();
    int s = 0;
    for (long long p = blockIdx.x; p < pairs; p += gridDim.x, s ^= 1) {
        const bool two = 2 * p + 1 < rows;
        cd v[16];
        prefetch(p + gridDim.x, s ^ 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();
        {
            const float* a = stg + 2 * s * SROW;
#pragma unroll
            for (int r = 0; r < 10; ++r) {
                const int n = j + r * kRfT;
                const bool in = r < 5 && n < W;
                v[r] = cd{in ? (double)a[n] : 0.0, (in && two) ? (double)a[SROW + n] : 0.0};
            }
        }
        // forward A: radix 10, Ns = 1 (256 threads): -> buf[10 j + q]
        dft10<false, true>(v);
#pragma unroll
        for (int q = 0; q < 10; ++q)
            buf[rf_sw(10 * j + q)] = make_double2(v[x10(q)].x, v[x10(q)].y);
        __syncthreads();
        // forward B: radix 16, Ns = 10
        if (act16) {
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const double2 x = buf[rf_sw(j + kRf2T16 * r)];
                v[r] = cd{x.x, x.y};
            }
        }
        __syncthreads();
        if (act16) {
            const double2 t = tw16x[j % 10];
            rf2_twiddle16<false, 10>(v, cd{t.x, t.y});
            dft16<false>(v);
            const int base = (j / 10) * 160 + (j % 10);
#pragma unroll
            for (int q = 0; q < 16; ++q)
                buf[rf_sw(base + 10 * q)] = make_double2(v[x16(q)].x, v[x16(q)].y);
        }
        __syncthreads();
        // forward C: radix 16, Ns = 160 -> registers: v[q] = Z[j + 160 q]
        if (act16) {
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const double2 x = buf[rf_sw(j + kRf2T16 * r)];
                v[r] = cd{x.x, x.y};
            }
        }
        __syncthreads();
        if (act16) {
            const double2 t = tw256[j];
            rf2_twiddle16<false, 160>(v, cd{t.x, t.y});
            dft16<false>(v);
            cd o[16];
#pragma unroll
            for (int q = 0; q < 16; ++q)
                o[q] = v[x16(q)];
            // spectrum multiply, then inverse A: radix 16, Ns = 1 -> buf[16 j + q]
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const int k = j + kRf2T16 * q;
                const double h = hs[k <= kRf2N / 2 ? k : kRf2N - k];
                v[q] = cd{o[q].x * h, o[q].y * h};
            }
            dft16<true>(v);
#pragma unroll
            for (int q = 0; q < 16; ++q)
                buf[rf_sw(16 * j + q)] = make_double2(v[x16(q)].x, v[x16(q)].y);
        }
        __syncthreads();
        // inverse B: radix 16, Ns = 16
        if (act16) {
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const double2 x = buf[rf_sw(j + kRf2T16 * r)];
                v[r] = cd{x.x, x.y};
            }
        }
        __syncthreads();
        if (act16) {
            const double2 t = tw10x[j % 16];
            rf2_twiddle16<true, 16>(v, cd{t.x, t.y});
            dft16<true>(v);
            const int base = (j / 16) * 256 + (j % 16);
#pragma unroll
            for (int q = 0; q < 16; ++q)
                buf[rf_sw(base + 16 * q)] = make_double2(v[x16(q)].x, v[x16(q)].y);
        }
        __syncthreads();
        // inverse C: radix 10, Ns = 256 (256 threads): y[j + 256 q]
#pragma unroll
        for (int r = 0; r < 10; ++r) {
            const double2 x = buf[rf_sw(j + kRfT * r)];
            v[r] = cd{x.x, x.y};
        }
        {
            const double2 t = tw256[j];
            const cd w1{t.x, -t.y};
            cd w = w1;
#pragma unroll
            for (int r = 1; r < 10; ++r) {
                v[r] = cmul(v[r], w);
                if (r < 9)
                    w = cmul(w, w1);
            }
        }
        dft10<true, false>(v);
        float* o1 = out + (2 * p) * (long long)W;
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            const int n = j + q * kRfT;
            if (n < W) {
                o1[n] = (float)v[x10(q)].x;
                if (two)
                    o1[W + n] = (float)v[x10(q)].y;
            }
        }
        __syncthreads(); // buf reused by the next pair's first pass
    }
}

// ramp_fft2560_rows with 160 threads per CTA (kRf2T16), 3 CTAs per SM: the
// four radix-16 passes (most of the FP64 work) use every thread instead of
// 160 of 256, and the two radix-10 passes (256 butterflies) take two rounds
// on threads 0-95. Same operations in the same order on the same values, so
// the same bits as ramp_fft2560_rows.
constexpr int kRf2T = kRf2T16;
__global__ void __launch_bounds__(kRf2T, 3)
ramp_fft2560_rows160(const float* raw, float* out, int W, long long rows,
                     const double* __restrict__ spec, const double2* __restrict__ tw) {
    extern __shared__ double2 rf_smem[];
    double2* buf = rf_smem;
    double* hs = reinterpret_cast<double*>(rf_smem + kRf2N);
    double2* tw256 = reinterpret_cast<double2*>(hs + kRf2N / 2 + 2);
    double2* tw16x = tw256 + 256; // tw[16 m], m < 10: forward radix-16 pass, Ns = 10
    double2* tw10x = tw16x + 10;  // tw[10 m], m < 16: inverse radix-16 pass, Ns = 16
    float* stg = reinterpret_cast<float*>(tw10x + 16);
    constexpr int SROW = kRf2MaxW;
    const int j = threadIdx.x;
    for (int k = j; k <= kRf2N / 2; k += kRf2T)
        hs[k] = spec[k];
    for (int k = j; k < 256; k += kRf2T)
        tw256[k] = __ldg(tw + k);
    if (j < 10)
        tw16x[j] = __ldg(tw + 16 * j);
    if (j < 16)
        tw10x[j] = __ldg(tw + 10 * j);
    const long long pairs = (rows + 1) / 2;
    auto prefetch = [&](long long p, int s) {
        if (p < pairs) {
            const float* r1 = raw + (2 * p) * (long long)W;
            const int nrow = 2 * p + 1 < rows ? 2 : 1;
            for (int e = j; e < nrow * W; e += kRf2T) {
                const int row = e >= W, n = e - row * W;
                const unsigned dst = (unsigned)__cvta_generic_to_shared(stg + (2 * s + row) * SROW + n);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(r1 + e));
            }
        }
        asm volatile("cp.async.commit_group;");
    };
    prefetch(blockIdx.x, 0);
    __syncthreads();
    int s = 0;
    for (long long p = blockIdx.x; p < pairs; p += gridDim.x, s ^= 1) {
        const bool two = 2 * p + 1 < rows;
        cd v[16];
        prefetch(p + gridDim.x, s ^ 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();
        // forward A: radix 10, Ns = 1, butterflies b = j, j + 160 (< 256): -> buf[10 b + q]
        {
            const float* a = stg + 2 * s * SROW;
            for (int b = j; b < 256; b += kRf2T) {
#pragma unroll
                for (int r = 0; r < 10; ++r) {
                    const int n = b + r * 256;
                    const bool in = r < 5 && n < W;
                    v[r] = cd{in ? (double)a[n] : 0.0, (in && two) ? (double)a[SROW + n] : 0.0};
                }
                dft10<false, true>(v);
#pragma unroll
                for (int q = 0; q < 10; ++q)
                    buf[rf_sw(10 * b + q)] = make_double2(v[x10(q)].x, v[x10(q)].y);
            }
        }
        __syncthreads();
        // forward B: radix 16, Ns = 10
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const double2 x = buf[rf_sw(j + kRf2T16 * r)];
            v[r] = cd{x.x, x.y};
        }
        __syncthreads();
        {
            const double2 t = tw16x[j % 10];
            rf2_twiddle16<false, 10>(v, cd{t.x, t.y});
            dft16<false>(v);
            const int base = (j / 10) * 160 + (j % 10);
#pragma unroll
            for (int q = 0; q < 16; ++q)
                buf[rf_sw(base + 10 * q)] = make_double2(v[x16(q)].x, v[x16(q)].y);
        }
        __syncthreads();
        // forward C: radix 16, Ns = 160 -> registers: v[q] = Z[j + 160 q]
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const double2 x = buf[rf_sw(j + kRf2T16 * r)];
            v[r] = cd{x.x, x.y};
        }
        __syncthreads();
        {
            const double2 t = tw256[j];
            rf2_twiddle16<false, 160>(v, cd{t.x, t.y});
            dft16<false>(v);
            cd o[16];
#pragma unroll
            for (int q = 0; q < 16; ++q)
                o[q] = v[x16(q)];
            // spectrum multiply, then inverse A: radix 16, Ns = 1 -> buf[16 j + q]
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const int k = j + kRf2T16 * q;
                const double h = hs[k <= kRf2N / 2 ? k : kRf2N - k];
                v[q] = cd{o[q].x * h, o[q].y * h};
            }
            dft16<true>(v);
#pragma unroll
            for (int q = 0; q < 16; ++q)
                buf[rf_sw(16 * j + q)] = make_double2(v[x16(q)].x, v[x16(q)].y);
        }
        __syncthreads();
        // inverse B: radix 16, Ns = 16
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const double2 x = buf[rf_sw(j + kRf2T16 * r)];
            v[r] = cd{x.x, x.y};
        }
        __syncthreads();
        {
            const double2 t = tw10x[j % 16];
            rf2_twiddle16<true, 16>(v, cd{t.x, t.y});
            dft16<true>(v);
            const int base = (j / 16) * 256 + (j % 16);
#pragma unroll
            for (int q = 0; q < 16; ++q)
                buf[rf_sw(base + 16 * q)] = make_double2(v[x16(q)].x, v[x16(q)].y);
        }
        __syncthreads();
        // inverse C: radix 10, Ns = 256, butterflies b = j, j + 160: y[b + 256 q]
        float* o1 = out + (2 * p) * (long long)W;
        for (int b = j; b < 256; b += kRf2T) {
#pragma unroll
            for (int r = 0; r < 10; ++r) {
                const double2 x = buf[rf_sw(b + 256 * r)];
                v[r] = cd{x.x, x.y};
            }
            {
                const double2 t = tw256[b];
                const cd w1{t.x, -t.y};
                cd w = w1;
#pragma unroll
                for (int r = 1; r < 10; ++r) {
                    v[r] = cmul(v[r], w);
                    if (r < 9)
                        w = cmul(w, w1);
                }
            }
            dft10<true, false>(v);
#pragma unroll
            for (int q = 0; q < 5; ++q) {
                const int n = b + q * 256;
                if (n < W) {
                    o1[n] = (float)v[x10(q)].x;
                    if (two)
                        o1[W + n] = (float)v[x10(q)].y;
                }
            }
        }
        __syncthreads(); // buf reused by the next pair's first pass
    }
}

// spec[k] = (1/N) sum_n hc[n] cos(2 pi k n / N), hc the wrapped kernel
// (n <= N/2: h(n), else h(n - N)); tw[e] = exp(-2 pi i e / N).
__global__ void ramp_fft_tables(double* spec, double2* tw, int N, double tau) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= N)
        return;
    double s = 0.0;
    for (int n = 0; n < N; ++n) {
        const double m = n <= N / 2 ? (double)n : (double)(n - N);
        const double h = -2.0 / (M_PI * M_PI * tau * (4.0 * m * m - 1.0));
        const long long e = ((long long)k * n) % N;
        s += h * cospi(2.0 * (double)e / (double)N);
    }
    spec[k] = s / (double)N;
    double sn, cs;
    sincospi(2.0 * (double)k / (double)N, &sn, &cs);
    tw[k] = make_double2(cs, -sn);
}

struct RampFftTables {
    double* spec = nullptr;
    double2* tw = nullptr;
};

class RampFftCache {
  public:
    static RampFftCache& get() {
        static RampFftCache c;
        return c;
    }
    // tables for (device, tau, N); built once on stream st (synchronously)
    RampFftTables tables(int device, double tau, cudaStream_t st, int N = kRfN) {
        std::lock_guard<std::mutex> lk(mu_);
        auto key = std::make_tuple(device, tau, N);
        auto it = map_.find(key);
        if (it != map_.end())
            return it->second;
        RampFftTables t;
        check_cuda(cudaMalloc(&t.spec, sizeof(double) * N), "cudaMalloc(ramp spectrum)");
        check_cuda(cudaMalloc(&t.tw, sizeof(double2) * N), "cudaMalloc(ramp twiddles)");
        ramp_fft_tables<<<(N + 127) / 128, 128, 0, st>>>(t.spec, t.tw, N, tau);
        check_cuda(cudaGetLastError(), "ramp_fft_tables");
        check_cuda(cudaStreamSynchronize(st), "ramp_fft_tables");
        ++g_launches;
        return map_.emplace(key, t).first->second;
    }

  private:
    std::mutex mu_;
    std::map<std::tuple<int, double, int>, RampFftTables> map_;
};

template <int NZ>
void launch_ramp_fft(int dev, unsigned grid, const float* raw, float* out, int W, long long rows,
                     const RampFftTables& t, cudaStream_t st) {
    static bool attr_set[64] = {};
    if (dev < 64 && !attr_set[dev]) {
        check_cuda(cudaFuncSetAttribute(ramp_fft_rows<NZ>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        rf_smem_bytes(NZ)),
                   "cudaFuncSetAttribute(ramp_fft_rows)");
        attr_set[dev] = true;
    }
    ramp_fft_rows<NZ><<<grid, kRfT, rf_smem_bytes(NZ), st>>>(raw, out, W, rows, t.spec, t.tw);
}

inline bool ramp_fft_supported(int W) { return W >= 1 && W <= kRfMaxW; }

// raw, out: count*H rows of W floats on the device (may alias).
inline void ramp_fft_device(const float* raw, float* out, int W, int H, int count, double tau,
                            cudaStream_t st) {
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    const long long rows = (long long)H * count;
    const long long pairs = (rows + 1) / 2;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const long long grid = std::min<long long>(pairs, (long long)nsm * 2); // 2 CTAs/SM
    if (grid < 1)
        return;
    static const bool no2560 = std::getenv("CBB_RAMP_4096") != nullptr; // comparisons
    if (W <= kRf2MaxW && !no2560) {
        const RampFftTables t2 = RampFftCache::get().tables(dev, tau, st, kRf2N);
        static bool attr2[64] = {};
        if (dev < 64 && !attr2[dev]) {
            check_cuda(cudaFuncSetAttribute(ramp_fft2560_rows,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, kRf2Bytes),
                       "cudaFuncSetAttribute(ramp_fft2560_rows)");
            attr2[dev] = true;
        }
        const bool use256 = std::getenv("CBB_RAMP_256") != nullptr; // comparisons (tests)
        if (use256) {
            ramp_fft2560_rows<<<(unsigned)grid, kRfT, kRf2Bytes, st>>>(raw, out, W, rows, t2.spec,
                                                                      t2.tw);
        } else {
            static bool attr3[64] = {};
            if (dev < 64 && !attr3[dev]) {
                check_cuda(cudaFuncSetAttribute(ramp_fft2560_rows160,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                kRf2Bytes),
                           "cudaFuncSetAttribute(ramp_fft2560_rows160)");
                attr3[dev] = true;
            }
            const long long grid3 = std::min<long long>(pairs, (long long)nsm * 3); // 3 CTAs/SM
            ramp_fft2560_rows160<<<(unsigned)grid3, kRf2T, kRf2Bytes, st>>>(raw, out, W, rows,
                                                                            t2.spec, t2.tw);
        }
        check_cuda(cudaGetLastError(), "ramp_fft2560_rows");
        ++g_launches;
        return;
    }
    const RampFftTables t = RampFftCache::get().tables(dev, tau, st);
    const int nz = (W + kRfT - 1) / kRfT;
    if (nz <= 5)
        launch_ramp_fft<5>(dev, (unsigned)grid, raw, out, W, rows, t, st);
    else if (nz == 6)
        launch_ramp_fft<6>(dev, (unsigned)grid, raw, out, W, rows, t, st);
    else
        launch_ramp_fft<8>(dev, (unsigned)grid, raw, out, W, rows, t, st);
    check_cuda(cudaGetLastError(), "ramp_fft_rows");
    ++g_launches;
}

} // namespace cbb
