// bp_tma.cuh -- back-projection from RAW projections staged in shared memory
// by TMA (sm_100a), the alternative to the packed-quad gather kernel of
// bp_kernels.cuh.
//
// Why: bp_kernel gathers each voxel's four taps with one scattered LDG.128
// from the packed quad layout. Those gathers miss L1 (ncu r1v12e: L1 hit
// 4.9 %), so every update waits on an L2 round trip (top stall
// long_scoreboard) and moves ~14 B from L2 (L1/TEX data pipe 76 %), and the
// quad layout costs a pack pass writing 4.8x the raw bytes.
//
// Here a block owns a 16 x 16 x 8 voxel tile (8 warps of 8 x 4 x 8, R = 8
// voxels per thread along z). For each projection of the batch that touches
// the tile, one elected thread asks the TMA unit for the tile's detector
// footprint -- a PITCH x BH box of the raw row-major projection
// (cp.async.bulk.tensor.3d, zero fill outside the detector, which is
// exactly the guarded sampler's per-tap zero) -- into an S-stage ring of
// shared-memory buffers, signalled by mbarriers (full: TMA transaction
// bytes; empty: one arrive per warp). Warps read their taps with four LDS
// (rows iy, iy + 1 at immediate offsets 0, 4, 4 PITCH, 4 PITCH + 4 from one
// address), ~30 cycles instead of an L2 round trip, and the L2 -> SM traffic
// drops to the footprint boxes (~5 B per update).
//
// The per-voxel arithmetic is bp_kernels.cuh's, operation for operation
// (exact mode bitwise = reference): only the source of the four tap values
// changes, and they are the same values (the box holds raw pixels, zero off
// the detector). A (block, projection) whose footprint does not fit the box
// (the host sizes the box from sampled footprints; the device checks every
// block) reads its taps from global memory with per-tap bounds checks --
// same values again, just slower.
#pragma once

#include <cuda.h>

namespace cbb {

constexpr int kTBX = 16, kTBY = 16;   // block tile in x, y (voxels)
#ifndef CBB_TMA_R
#define CBB_TMA_R 12
#endif
constexpr int kTR = CBB_TMA_R;        // voxels per thread along z
// Voxel-pair body (bp_project_p): every per-voxel quantity of two z-neighbours
// in one f32x2 register, taps included; 0 = bp_project_f (pairs within a voxel).
#ifndef CBB_TMA_PAIRS
#define CBB_TMA_PAIRS 1
#endif
// guarded kernel: voxels per thread along z -- the same z-blocks as the staged
// kernel, so a resident tail gap (aligned to kTR) maps identically
constexpr int kGR = kTR;
constexpr int kTThreads = 256;        // 8 warps of 8 x 4 voxel columns
constexpr int kTMaxStages = 8;        // TMA ring depth limit (the host picks 2..8 stages)

struct TmaArgs {
    float* vol;             // slab base: voxel (0, 0, z_begin)
    const float* raw;       // raw projection 0 of this launch (band row raw_row0 first)
    long long raw_stride;   // floats per projection in the raw buffer
    const unsigned* flags;  // per projection of this launch: bit 0 = a tap >= 2^86
    int* err;               // bit 0: w == 0 (guarded kernel)
    unsigned long long neg_zero2;
    unsigned long long* counters; // nullable: culled-update counters
    int L, z_begin, z_end, count;
    float O, MM;
    float Wf, Hf;           // detector size (cull test)
    int W, H;               // detector size (fallback fetch)
    int raw_row0, raw_rows; // detector rows held by the raw buffer
    int tz0;                // TMA z coordinate of projection 0 of this launch
    int bh;                 // box rows (TMA box height); box width = PITCH
    int cull;
    int gap_at, gap;        // skipped planes (resident tail), as in BpArgs
    int stages;             // TMA ring depth (2..kTMaxStages)
    unsigned magic_off;     // -4 kMagic (mod 2^32), passed at run time so that ptxas cannot
                            // split it off the stage base into four load-address adds
};

constexpr int kTmaBatch = 64;         // projections per staged launch (64-bit masks)

struct TmaMats {
    float a[kTmaBatch][12]; // parameter-bank layout of bp_kernels.cuh (store_matrix)
};

// block_setup (bp_kernels.cuh) for up to kTmaBatch projections: the batch's
// matrices and the block-uniform z-products in shared memory.
template <int R>
__device__ BlockTables<R> tma_block_setup(const TmaArgs& args, const TmaMats& mats, int zoff) {
    __shared__ float s_m[kTmaBatch * 12];
    __shared__ __align__(16) f2 s_zuv[kTmaBatch * R];
    __shared__ f2 s_zw[kTmaBatch * (R / 2)];
    const float* flat = &mats.a[0][0];
    for (int i = threadIdx.x; i < args.count * 12; i += blockDim.x)
        s_m[i] = flat[i];
    const int z0 = args.z_begin + zoff, zl = args.z_end - 1;
    for (int i = threadIdx.x; i < args.count * R; i += blockDim.x) {
        const int p = i / R, r = i % R;
        const float* a = flat + 12 * p;
#if CBB_TMA_PAIRS
        // voxel pairs: entry 2k + c = (wz_2k * a[6 + c], wz_2k+1 * a[6 + c])
        const int k = r / 2, c = r % 2;
        const float wz0 = __fadd_rn(args.O, __fmul_rn((float)min(z0 + 2 * k, zl), args.MM));
        const float wz1 = __fadd_rn(args.O, __fmul_rn((float)min(z0 + 2 * k + 1, zl), args.MM));
        s_zuv[i] = pk(__fmul_rn(wz0, a[M67 + c]), __fmul_rn(wz1, a[M67 + c]));
#else
        const float wz = __fadd_rn(args.O, __fmul_rn((float)min(z0 + r, zl), args.MM));
        s_zuv[i] = pk(__fmul_rn(wz, a[M67]), __fmul_rn(wz, a[M67 + 1]));
#endif
    }
    for (int i = threadIdx.x; i < args.count * (R / 2); i += blockDim.x) {
        const int p = i / (R / 2), k = i % (R / 2);
        const float wz0 = __fadd_rn(args.O, __fmul_rn((float)min(z0 + 2 * k, zl), args.MM));
        const float wz1 = __fadd_rn(args.O, __fmul_rn((float)min(z0 + 2 * k + 1, zl), args.MM));
        const float a8 = flat[12 * p + M8];
        s_zw[i] = pk(__fmul_rn(wz0, a8), __fmul_rn(wz1, a8));
    }
    __syncthreads();
    return BlockTables<R>{s_m, s_zuv, s_zw};
}

// ---------------------------------------------------------------------------
// mbarrier / TMA primitives
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Waits on the mbarrier at shared address `addr` (32-bit window address).
__device__ __forceinline__ void mbar_wait_a(unsigned addr, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(addr),
        "r"(parity)
        : "memory");
}
// Single-thread shared atomic add returning the old value (no warp
// aggregation code around it).
__device__ __forceinline__ unsigned atom_add_shared(unsigned addr, unsigned v) {
    unsigned old;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void mbar_arrive_a(unsigned addr) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ bool mbar_test_a(unsigned addr, unsigned parity) {
    unsigned r;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n}"
        : "=r"(r)
        : "r"(addr), "r"(parity)
        : "memory");
    return r != 0u;
}
// Non-blocking probe: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(unsigned long long* bar, unsigned parity) {
    unsigned r;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n}"
        : "=r"(r)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return r != 0u;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 3-D tile load (x, y, projection) into shared memory, completion counted on bar.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map,
                                            unsigned long long* bar, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
        : "memory");
}

// ---------------------------------------------------------------------------
// Tap fetchers: {bl, tl, br, tr} of truncated position (ixt, iyt), the
// quad layout of bp_kernels.cuh, so the lerp code is shared.
// ---------------------------------------------------------------------------

// From a staged box. sbase = shared address of the stage - 4 kMagic (so the
// biased float index bits address it with one IMAD); bias = 2^23 - by0 *
// PITCH - bx0. The loads are volatile asm: they stay between the stage's
// full-barrier wait and the warp's empty-barrier arrive (both volatile asm)
// and take immediate offsets for the three other taps.
template <int PITCH>
struct SmemFetch {
    unsigned sbase;
    float bias;
    __device__ __forceinline__ float4 operator()(float ixt, float iyt) const {
        const int bits = __float_as_int(__fmaf_rn(iyt, (float)PITCH, __fadd_rn(ixt, bias)));
        unsigned a;
        asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(a) : "r"(bits), "r"(sbase));
        float bl, br, tl, tr;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(bl) : "r"(a));
        asm volatile("ld.shared.f32 %0, [%1+4];" : "=f"(br) : "r"(a));
        asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(tl) : "r"(a), "n"(PITCH * 4));
        asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(tr) : "r"(a), "n"(PITCH * 4 + 4));
        return make_float4(bl, tl, br, tr);
    }
    // Taps of two voxels as pairs (bl0, bl1), (tl0, tl1), ... : the cell
    // indices of both in one FADD2 + FFMA2 (integer-valued, exact).
    __device__ __forceinline__ void pair(f2 ixt, f2 iyt, f2& bl, f2& tl, f2& br, f2& tr) const {
        const f2 idx = fma2(iyt, bc((float)PITCH), add2(ixt, bc(bias)));
        float i0, i1;
        upk(idx, i0, i1);
        unsigned a0, a1;
        asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(a0) : "r"(__float_as_int(i0)), "r"(sbase));
        asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(a1) : "r"(__float_as_int(i1)), "r"(sbase));
        float b0, b1, r0, r1, t0, t1, q0, q1;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(b0) : "r"(a0));
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(b1) : "r"(a1));
        asm volatile("ld.shared.f32 %0, [%1+4];" : "=f"(r0) : "r"(a0));
        asm volatile("ld.shared.f32 %0, [%1+4];" : "=f"(r1) : "r"(a1));
        asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(t0) : "r"(a0), "n"(PITCH * 4));
        asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(t1) : "r"(a1), "n"(PITCH * 4));
        asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(q0) : "r"(a0), "n"(PITCH * 4 + 4));
        asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(q1) : "r"(a1), "n"(PITCH * 4 + 4));
        bl = pk(b0, b1);
        br = pk(r0, r1);
        tl = pk(t0, t1);
        tr = pk(q0, q1);
    }
};

// From the raw projection in global memory with the reference's per-tap
// bounds (kernel_ref.hpp:33-44); rows outside the held band read as 0 (the
// host sizes bands so that this only happens off the detector).
struct RawFetch {
    const float* img; // row raw_row0 of the projection
    int W, H, r0, rn;
    __device__ __forceinline__ float tap(int x, int y) const {
        const bool in = x >= 0 && x < W && y >= 0 && y < H && y >= r0 && y < r0 + rn;
        return in ? __ldg(img + (long long)(y - r0) * W + x) : 0.0f;
    }
    __device__ __forceinline__ float4 operator()(float ixt, float iyt) const {
        const int x = (int)ixt, y = (int)iyt;
        return make_float4(tap(x, y), tap(x, y + 1), tap(x + 1, y), tap(x + 1, y + 1));
    }
    __device__ __forceinline__ void pair(f2 ixt, f2 iyt, f2& bl, f2& tl, f2& br, f2& tr) const {
        float x0, x1, y0, y1;
        upk(ixt, x0, x1);
        upk(iyt, y0, y1);
        const float4 a = (*this)(x0, y0), b = (*this)(x1, y1);
        bl = pk(a.x, b.x);
        tl = pk(a.y, b.y);
        br = pk(a.z, b.z);
        tr = pk(a.w, b.w);
    }
};

// exact mode: 1/(w*w) from RN(y*y) instead of a second MUFU.RCP (below)
#ifndef CBB_TMA_YY
#define CBB_TMA_YY 1
#endif

// bp_project (bp_kernels.cuh) with the taps from `fetch` (no clamping: the
// fetcher covers every tap position of the tile). Operation for operation
// the same arithmetic.
template <int R, int MODE, class Fetch>
__device__ __forceinline__ void bp_project_f(const TmaArgs& args, const float* m, float wx,
                                             float wy, const f2* zuv, const f2* zw,
                                             f2 (&accp)[R / 2], unsigned& vmin,
                                             const Fetch& fetch) {
    const f2 NZ = args.neg_zero2;
    const f2 ONE2 = bc(1.0f);
    const f2 ZERO2 = bc(0.0f);
    const f2 a910 = ld2(m, M910);
    const f2 tuv = add2(MUL2(ld2(m, M01), bc(wx)), MUL2(ld2(m, M34), bc(wy)));
    const float tw = __fadd_rn(__fmul_rn(wx, m[M2]), __fmul_rn(wy, m[M5]));
    constexpr int G = R % 4 == 0 ? 4 : 2;
    constexpr int GP = G / 2;
#pragma unroll
    for (int g = 0; g < R / G; ++g) {
        f2 wpair[GP], ypair[GP], sxy[G];
        float4 quad[G];
#pragma unroll
        for (int k = 0; k < GP; ++k) {
            const f2 w01 = add2(add2(bc(tw), zw[g * GP + k]), bc(m[M11]));
            wpair[k] = w01;
            float w0, w1;
            upk(w01, w0, w1);
            const f2 r01 = pk(rcp_approx(w0), rcp_approx(w1));
            const f2 y01 = fma2(r01, fma2(neg2(w01), r01, ONE2), r01);
            ypair[k] = y01;
            float yv[2];
            upk(y01, yv[0], yv[1]);
            const float wv[2] = {w0, w1};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int r = 2 * k + h;
                const f2 uv = add2(add2(tuv, zuv[g * G + r]), a910);
                const f2 q0 = fma2(uv, bc(yv[h]), ZERO2);
                const f2 rem = fma2(bc(-wv[h]), q0, uv);
                const f2 ixy = fma2(bc(yv[h]), rem, q0);
                float ix, iy;
                upk(ixy, ix, iy);
                const float ixt = truncf(ix);
                const float iyt = truncf(iy);
                sxy[r] = add2(ixy, pk(-ixt, -iyt));
                quad[r] = fetch(ixt, iyt);
            }
        }
#pragma unroll
        for (int k = 0; k < GP; ++k) {
            float val[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int r = 2 * k + h;
                float sx, sy;
                upk(sxy[r], sx, sy);
                const f2 oms = add2(ONE2, neg2(sxy[r]));
                float omsx, omsy;
                upk(oms, omsx, omsy);
                const f2 bt = add2(MUL2(pk(quad[r].x, quad[r].y), bc(omsx)),
                                   MUL2(pk(quad[r].z, quad[r].w), bc(sx)));
                float valb, valt;
                upk(bt, valb, valt);
                val[h] = __fadd_rn(__fmul_rn(omsy, valb), __fmul_rn(sy, valt));
            }
            const f2 vv = pk(val[0], val[1]);
            f2 c;
            if (MODE == 0) {
                const f2 ww = MUL2(wpair[k], wpair[k]);
                float ww0, ww1;
                upk(ww, ww0, ww1);
#if CBB_TMA_YY
                // 1/(w*w) seeded with RN(y*y) (y: the refined 1/w) instead of
                // a second MUFU.RCP, then the same Newton step: as accurate
                // (error squared by the step), one XU op fewer per voxel;
                // bitwise the IEEE quotient on 4e10 random operand pairs
                // (profiles/probes/weight_div_check.cu)
                (void)ww0;
                (void)ww1;
                const f2 r2 = MUL2(ypair[k], ypair[k]);
#else
                const f2 r2 = pk(rcp_approx(ww0), rcp_approx(ww1));
#endif
                const f2 y2 = fma2(r2, fma2(neg2(ww), r2, ONE2), r2);
                const f2 q0 = MUL2(vv, y2);
                c = fma2(neg2(y2), fma2(ww, q0, neg2(vv)), q0);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const unsigned e = __float_as_uint(val[h]) << 1;
                    vmin = min(vmin, e - 1u);
                }
            } else {
                c = MUL2(vv, MUL2(ypair[k], ypair[k]));
            }
            accp[g * GP + k] = add2(accp[g * GP + k], c);
        }
    }
}

// bp_project_f with voxel pairs in the lanes: (u0, u1), (v0, v1), (ix0, ix1),
// ..., the taps (bl0, bl1), ... and the two lerps, so the y-lerp and the tap
// addresses pack too (~3 instructions fewer per voxel). Same operations on
// the same operands as bp_project_f, so the same bits. zuv: the pair layout
// of tma_block_setup (CBB_TMA_PAIRS).
template <int R, int MODE, class Fetch>
__device__ __forceinline__ void bp_project_p(const TmaArgs& args, const float* m, float wx,
                                             float wy, const f2* zuv, const f2* zw,
                                             f2 (&accp)[R / 2], unsigned& vmin,
                                             const Fetch& fetch) {
    const f2 NZ = args.neg_zero2;
    const f2 ONE2 = bc(1.0f);
    const f2 ZERO2 = bc(0.0f);
    const f2 tuv = add2(MUL2(ld2(m, M01), bc(wx)), MUL2(ld2(m, M34), bc(wy)));
    float tu, tv;
    upk(tuv, tu, tv);
    const float tw = __fadd_rn(__fmul_rn(wx, m[M2]), __fmul_rn(wy, m[M5]));
#ifdef CBB_TMA_GP
    constexpr int GP = CBB_TMA_GP;         // voxel pairs in flight (tuning hook)
#else
    constexpr int GP = R % 4 == 0 ? 2 : 1; // voxel pairs in flight
#endif
    static_assert((R / 2) % GP == 0, "pairs per group");
#pragma unroll
    for (int g = 0; g < R / (2 * GP); ++g) {
        f2 wpair[GP], ypair[GP], sx[GP], sy[GP], bl[GP], tl[GP], br[GP], tr[GP];
#pragma unroll
        for (int k = 0; k < GP; ++k) {
            const int kk = g * GP + k;
            const f2 w01 = add2(add2(bc(tw), zw[kk]), bc(m[M11]));
            wpair[k] = w01;
            float w0, w1;
            upk(w01, w0, w1);
            const f2 r01 = pk(rcp_approx(w0), rcp_approx(w1));
            const f2 y01 = fma2(r01, fma2(neg2(w01), r01, ONE2), r01);
            ypair[k] = y01;
            const float4 z4 = *reinterpret_cast<const float4*>(zuv + 2 * kk);
            const f2 u01 = add2(add2(bc(tu), pk(z4.x, z4.y)), bc(m[M910]));
            const f2 v01 = add2(add2(bc(tv), pk(z4.z, z4.w)), bc(m[M910 + 1]));
            const f2 qu = fma2(u01, y01, ZERO2);
            const f2 ix01 = fma2(y01, fma2(neg2(w01), qu, u01), qu);
            const f2 qv = fma2(v01, y01, ZERO2);
            const f2 iy01 = fma2(y01, fma2(neg2(w01), qv, v01), qv);
            float ix0, ix1, iy0, iy1;
            upk(ix01, ix0, ix1);
            upk(iy01, iy0, iy1);
            const f2 ixt = pk(truncf(ix0), truncf(ix1));
            const f2 iyt = pk(truncf(iy0), truncf(iy1));
            sx[k] = add2(ix01, neg2(ixt));
            sy[k] = add2(iy01, neg2(iyt));
            fetch.pair(ixt, iyt, bl[k], tl[k], br[k], tr[k]);
        }
#pragma unroll
        for (int k = 0; k < GP; ++k) {
            const f2 omsx = add2(ONE2, neg2(sx[k]));
            const f2 omsy = add2(ONE2, neg2(sy[k]));
            const f2 vb = add2(MUL2(bl[k], omsx), MUL2(br[k], sx[k]));
            const f2 vt = add2(MUL2(tl[k], omsx), MUL2(tr[k], sx[k]));
            const f2 vv = add2(MUL2(omsy, vb), MUL2(sy[k], vt));
            f2 c;
            if (MODE == 0) {
                const f2 ww = MUL2(wpair[k], wpair[k]);
#if CBB_TMA_YY
                const f2 r2 = MUL2(ypair[k], ypair[k]);
#else
                float ww0, ww1;
                upk(ww, ww0, ww1);
                const f2 r2 = pk(rcp_approx(ww0), rcp_approx(ww1));
#endif
                const f2 y2 = fma2(r2, fma2(neg2(ww), r2, ONE2), r2);
                const f2 q0 = MUL2(vv, y2);
                c = fma2(neg2(y2), fma2(ww, q0, neg2(vv)), q0);
                float val[2];
                upk(vv, val[0], val[1]);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const unsigned e = __float_as_uint(val[h]) << 1;
                    vmin = min(vmin, e - 1u);
                }
            } else {
                c = MUL2(vv, MUL2(ypair[k], ypair[k]));
            }
            accp[g * GP + k] = add2(accp[g * GP + k], c);
        }
    }
}

// update_ieee (bp_kernels.cuh) with raw taps: IEEE divisions, optional
// reference guards.
template <int MODE, bool GUARD>
__device__ __forceinline__ float update_ieee_raw(const RawFetch& f, float u, float v, float w) {
    const float ix = __fdiv_rn(u, w);
    const float iy = __fdiv_rn(v, w);
    float val = 0.0f;
    if (!GUARD || (fabsf(ix) < 1.0e9f && fabsf(iy) < 1.0e9f)) {
        const float ixt = truncf(ix);
        const float iyt = truncf(iy);
        val = lerp_quad(f(ixt, iyt), __fsub_rn(ix, ixt), __fsub_rn(iy, iyt));
    }
    if (MODE == 0)
        return __fdiv_rn(val, __fmul_rn(w, w));
    const float rw = __frcp_rn(w);
    return __fmul_rn(val, __fmul_rn(rw, rw));
}

__device__ __forceinline__ RawFetch raw_fetch(const TmaArgs& a, int p) {
    return RawFetch{a.raw + (long long)p * a.raw_stride, a.W, a.H, a.raw_row0, a.raw_rows};
}

// Projects the 8 corners of the box [x0,x1] x [y0,y1] x [z0,z1] (world mm)
// with matrix a (parameter-bank layout), approximate arithmetic; w > 0 on
// the box is guaranteed for unguarded batches.
__device__ __forceinline__ void corner_extent(const float* a, const float cx[2],
                                              const float cy[2], const float cz[2], float& minx,
                                              float& maxx, float& miny, float& maxy) {
    minx = miny = 3.0e38f;
    maxx = maxy = -3.0e38f;
#pragma unroll
    for (int yi = 0; yi < 2; ++yi) {
#pragma unroll
        for (int zi = 0; zi < 2; ++zi) {
            const float bu = fmaf(a[M34], cy[yi], fmaf(a[M67], cz[zi], a[M910]));
            const float bv = fmaf(a[M34 + 1], cy[yi], fmaf(a[M67 + 1], cz[zi], a[M910 + 1]));
            const float bw = fmaf(a[M5], cy[yi], fmaf(a[M8], cz[zi], a[M11]));
#pragma unroll
            for (int xi = 0; xi < 2; ++xi) {
                const float rw = rcp_approx(fmaf(a[M2], cx[xi], bw));
                const float ix = fmaf(a[M01], cx[xi], bu) * rw;
                const float iy = fmaf(a[M01 + 1], cx[xi], bv) * rw;
                minx = fminf(minx, ix);
                maxx = fmaxf(maxx, ix);
                miny = fminf(miny, iy);
                maxy = fmaxf(maxy, iy);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// The kernel. Grid (ceil(L/16), ceil(L/16), z-blocks of 8 planes), 256
// threads, dynamic shared memory: S stages of PITCH * bh floats, then 2 S
// mbarriers.
// ---------------------------------------------------------------------------
#ifndef CBB_TMA_MINB
#define CBB_TMA_MINB 3
#endif
#if CBB_TMA_PAIRS
#define CBB_TMA_BODY bp_project_p
#else
#define CBB_TMA_BODY bp_project_f
#endif
template <int MODE, int PITCH, bool CNT>
__global__ void __launch_bounds__(kTThreads, CBB_TMA_MINB)
bp_tma_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ TmaArgs args,
              const __grid_constant__ TmaMats mats) {
    constexpr int R = kTR, P = R / 2;
    extern __shared__ __align__(128) unsigned char tsm[];
    const int S = args.stages;
    const int stage_floats = PITCH * args.bh;
    float* stages = reinterpret_cast<float*>(tsm);
    __shared__ unsigned long long full[kTMaxStages];
    __shared__ unsigned long long empty[kTMaxStages]; // one arrive per warp and use
    __shared__ int s_claim[kTMaxStages];    // staged index whose refill was claimed
    __shared__ int s_tlist[kTmaBatch];      // staged projections in order
    __shared__ int2 s_box[kTmaBatch];
    __shared__ float s_bias[kTmaBatch];
    __shared__ unsigned s_fit2[2];          // per half: projections whose box fits
    __shared__ unsigned long long s_wmask[kTThreads / 32];
    __shared__ unsigned s_culled;

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int tx0 = blockIdx.x * kTBX + (warp & 1) * 8;
    const int ty0 = blockIdx.y * kTBY + (warp >> 1) * 4;
    const int x = tx0 + (lane & 7);
    const int y = ty0 + (lane >> 3);
    const int bz = blockIdx.z;
    const int zoff = bz * R >= args.gap_at ? bz * R + args.gap : bz * R;
    const int L = args.L;
    const float O = args.O, MM = args.MM;
    const bool in_xy = x < L && y < L;
    const float wx = __fadd_rn(O, __fmul_rn((float)min(x, L - 1), MM));
    const float wy = __fadd_rn(O, __fmul_rn((float)min(y, L - 1), MM));
    const int zfirst = args.z_begin + zoff;
    const int nvalid = in_xy ? max(0, min(R, args.z_end - zfirst)) : 0;

    float acc[R];
    const size_t plane = (size_t)L * L;
    float* volp = args.vol + (size_t)zoff * plane + (size_t)y * L + x;
#pragma unroll
    for (int r = 0; r < R; ++r)
        acc[r] = r < nvalid ? volp[(size_t)r * plane] : 0.0f;
    f2 accp[P];
    bool negz = false;
#pragma unroll
    for (int k = 0; k < P; ++k) {
        accp[k] = pk(acc[2 * k], acc[2 * k + 1]);
        negz |= __float_as_uint(acc[2 * k]) == 0x80000000u ||
                __float_as_uint(acc[2 * k + 1]) == 0x80000000u;
    }
    if (CNT && threadIdx.x == 0)
        s_culled = 0u;
    const BlockTables<R> tabs = tma_block_setup<R>(args, mats, zoff);
    const float* s_m = tabs.m;

    // ---- per-warp culling (lane = projection) and per-block footprint boxes
    const int z0 = zfirst, z1 = min(zfirst + R - 1, args.z_end - 1);
    const float cz[2] = {O + (float)z0 * MM, O + (float)z1 * MM};
    unsigned long long todo = 0ull, bigm = 0ull;
    for (int half = 0; half < 2 && 32 * half < args.count; ++half) {
        const int p = 32 * half + lane;
        bool active = false, big = false;
        if (p < args.count && tx0 < L && ty0 < L) {
            const float cx[2] = {O + (float)tx0 * MM, O + (float)min(tx0 + 7, L - 1) * MM};
            const float cy[2] = {O + (float)ty0 * MM, O + (float)min(ty0 + 3, L - 1) * MM};
            float minx, maxx, miny, maxy;
            corner_extent(s_m + 12 * p, cx, cy, cz, minx, maxx, miny, maxy);
            const float mg = 0.05f, rel = 1e-5f;
            active = !(maxx < -2.0f - mg - rel * fabsf(maxx) ||
                       minx > args.Wf + mg + rel * fabsf(minx) ||
                       maxy < -2.0f - mg - rel * fabsf(maxy) ||
                       miny > args.Hf + mg + rel * fabsf(miny));
        }
        if (MODE == 0 && p < args.count)
            big = (__ldg(args.flags + p) & 1u) != 0u;
        todo |= (unsigned long long)__ballot_sync(0xffffffffu, active) << (32 * half);
        bigm |= (unsigned long long)__ballot_sync(0xffffffffu, big) << (32 * half);
    }
    if (!args.cull || __any_sync(0xffffffffu, negz))
        todo = args.count == 64 ? ~0ull : ((1ull << args.count) - 1ull);
    if (warp < 2 && 32 * warp < args.count) {
      // warps 0 and 1: projections 0-31 and 32-63
      {
        const int half = warp;
        // block box for projection p: taps of every voxel of the tile
        // (padding voxels sit on real ones) lie in [floor(min ix), floor(max ix) + 2]
        const int p = 32 * half + lane;
        bool fits = false;
        int bx0 = 0, by0 = 0;
        if (p < args.count) {
            const int bxa = blockIdx.x * kTBX, bya = blockIdx.y * kTBY;
            const float cx[2] = {O + (float)min(bxa, L - 1) * MM,
                                 O + (float)min(bxa + kTBX - 1, L - 1) * MM};
            const float cy[2] = {O + (float)min(bya, L - 1) * MM,
                                 O + (float)min(bya + kTBY - 1, L - 1) * MM};
            float minx, maxx, miny, maxy;
            corner_extent(s_m + 12 * p, cx, cy, cz, minx, maxx, miny, maxy);
            const float mg = 0.05f, rel = 1e-5f;
            // the TMA box's innermost start coordinate must be 16-byte aligned
            // (a multiple of 4 floats; other starts raise an illegal
            // instruction on B200 -- profiles/probes/tma_unit.cu)
            const float lx = 4.0f * floorf(floorf(minx - mg - rel * fabsf(minx)) * 0.25f);
            const float hx = floorf(maxx + mg + rel * fabsf(maxx)) + 2.0f;
            const float ly = floorf(miny - mg - rel * fabsf(miny));
            const float hy = floorf(maxy + mg + rel * fabsf(maxy)) + 2.0f;
            // box in range for the float index bias (exact below 2^22) and TMA
            fits = hx - lx + 1.0f <= (float)PITCH && hy - ly + 1.0f <= (float)args.bh &&
                   fabsf(lx) < 1.0e6f && fabsf(ly) < 1.0e6f &&
                   fabsf(ly) * (float)PITCH + fabsf(lx) < 4194304.0f;
            if (fits) {
                bx0 = (int)lx;
                by0 = (int)ly;
            }
        }
        s_box[p] = make_int2(bx0, by0);
        // SmemFetch bias: 2^23 - (by0 * PITCH + bx0), exact (|.| < 2^22)
        s_bias[p] = 8388608.0f - (float)(by0 * PITCH + bx0);
        const unsigned fm = __ballot_sync(0xffffffffu, fits);
        if (lane == 0)
            s_fit2[half] = fm;
      }
    }
    if (lane == 0)
        s_wmask[warp] = todo;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kTThreads / 32);
            s_claim[s] = -1;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    unsigned long long act = 0ull;
#pragma unroll
    for (int w = 0; w < kTThreads / 32; ++w)
        act |= s_wmask[w];
    const unsigned long long s_fit =
        args.count > 32 ? ((unsigned long long)s_fit2[1] << 32) | s_fit2[0] : s_fit2[0];
    const unsigned long long tma_mask = act & s_fit;
    const unsigned stage_bytes = (unsigned)stage_floats * 4u;
    const int ntma = __popcll(tma_mask);
    // Staged projection t (t-th bit of tma_mask) goes to slot t % S. Thread 0
    // fills the first S slots; afterwards the LAST warp to finish with a slot
    // (shared counter) refills it with projection t + S at once, so every
    // load is issued as soon as the slowest warp allows, S - 1 projections
    // ahead, and no warp ever waits for another to issue.
    auto issue = [&](int slot, int p) {
        const int2 b = s_box[p];
        mbar_expect_tx(&full[slot], stage_bytes);
        tma_load_3d(stages + (size_t)slot * stage_floats, &tmap, &full[slot], b.x,
                    b.y - args.raw_row0, args.tz0 + p);
    };
    if (MODE == 0 && warp == 0) {
        // the staged list in parallel: lane l places projections l and
        // l + 32 at their rank among the staged ones; the first S go out at
        // once from their lanes (exact mode 9.55 -> 9.45 ms per config-2
        // launch; fast mode measured 8.15 -> 8.21 ms, so it keeps the loop)
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const int p = 32 * half + lane;
            if ((tma_mask >> p) & 1ull) {
                const int t = __popcll(tma_mask & ((1ull << p) - 1ull));
                s_tlist[t] = p;
                if (t < S)
                    issue(t, p);
            }
        }
    }
    if (MODE != 0 && threadIdx.x == 0) {
        unsigned long long pm = tma_mask;
        for (int t = 0; pm; ++t, pm &= pm - 1ull) {
            const int p = __ffsll(pm) - 1;
            s_tlist[t] = p;
            if (t < S)
                issue(t, p);
        }
    }
    __syncthreads(); // s_tlist
    if (CNT) {
        const unsigned nv = __reduce_add_sync(0xffffffffu, (unsigned)nvalid);
        const unsigned culled = (unsigned)args.count - __popcll(todo);
        if (lane == 0 && nv && culled)
            atomicAdd(&s_culled, nv * culled);
    }

    unsigned vmin = bigm ? 0u : ~0u;
    const unsigned sb0 = smem_u32(stages) + args.magic_off;
    const unsigned full0 = smem_u32(full), empty0 = smem_u32(empty);
    unsigned sbc = sb0;      // biased shared address of the consumer's slot
    int k = 0, cslot = 0;    // consumer position among the staged projections
    unsigned cph = 0u;       // parity of the consumer slot's current use
    // one staged projection: wait for its box, compute (if this warp's tile
    // touches it), release the slot
    auto staged = [&](int p) {
        mbar_wait_a(full0 + 8u * (unsigned)cslot, cph);
        if ((todo >> p) & 1ull) {
            const SmemFetch<PITCH> f{sbc, s_bias[p]};
            CBB_TMA_BODY<R, MODE>(args, mats.a[p], wx, wy, tabs.zuv + p * R,
                                  tabs.zw + p * (R / 2), accp, vmin, f);
        }
        __syncwarp();
        if (lane == 0) {
            // the warp's reads of the slot are done (issued before, in
            // order). Every warp arrives on the slot's empty barrier; a warp
            // that then sees the phase complete (its own arrival was the
            // last, or a concurrent one was) claims the refill -- normally
            // one warp, so the claim's atomic is rare.
            const unsigned eb = empty0 + 8u * (unsigned)cslot;
            mbar_arrive_a(eb);
            if (k + S < ntma && mbar_test_a(eb, cph) && atomicExch(&s_claim[cslot], k) != k)
                issue(cslot, s_tlist[k + S]);
        }
        ++k;
        if (++cslot == S) {
            cslot = 0;
            cph ^= 1u;
            sbc = sb0;
        } else {
            sbc += stage_bytes;
        }
    };
    if (act == tma_mask) {
        // common case: every active projection is staged
#if defined(CBB_TMA_UNROLL) && CBB_TMA_UNROLL == 2
#pragma unroll 2
#endif
        for (int t = 0; t < ntma; ++t)
            staged(s_tlist[t]);
    } else {
        for (unsigned long long rem = act; rem; rem &= rem - 1ull) {
            const int p = __ffsll(rem) - 1;
            if ((tma_mask >> p) & 1ull)
                staged(p);
            else if ((todo >> p) & 1ull)
                CBB_TMA_BODY<R, MODE>(args, mats.a[p], wx, wy, tabs.zuv + p * R,
                                      tabs.zw + p * (R / 2), accp, vmin, raw_fetch(args, p));
        }
    }
    bool redo = false;
    if (MODE == 0)
        redo = vmin < 0x43000000u - 1u;
#pragma unroll
    for (int q = 0; q < P; ++q)
        upk(accp[q], acc[2 * q], acc[2 * q + 1]);
    if (MODE == 0 && redo) {
        // numerator outside the fast division's proven range: recompute the
        // thread's voxels over the batch with IEEE divisions
#pragma unroll
        for (int r = 0; r < R; ++r)
            acc[r] = r < nvalid ? volp[(size_t)r * plane] : 0.0f;
        for (int p = 0; p < args.count; ++p) {
            const float* m = mats.a[p];
            const RawFetch f = raw_fetch(args, p);
            const float tu = __fadd_rn(__fmul_rn(wx, m[M01]), __fmul_rn(wy, m[M34]));
            const float tv = __fadd_rn(__fmul_rn(wx, m[M01 + 1]), __fmul_rn(wy, m[M34 + 1]));
            const float tw = __fadd_rn(__fmul_rn(wx, m[M2]), __fmul_rn(wy, m[M5]));
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const float wz = __fadd_rn(O, __fmul_rn((float)min(zfirst + r, args.z_end - 1), MM));
                const float u = __fadd_rn(__fadd_rn(tu, __fmul_rn(wz, m[M67])), m[M910]);
                const float v = __fadd_rn(__fadd_rn(tv, __fmul_rn(wz, m[M67 + 1])), m[M910 + 1]);
                const float w = __fadd_rn(__fadd_rn(tw, __fmul_rn(wz, m[M8])), m[M11]);
                acc[r] = __fadd_rn(acc[r], update_ieee_raw<0, false>(f, u, v, w));
            }
        }
    }
    if (act) {
#pragma unroll
        for (int r = 0; r < R; ++r)
            if (r < nvalid)
                volp[(size_t)r * plane] = acc[r];
    }
    if (CNT) {
        __syncthreads();
        if (threadIdx.x == 0 && s_culled) {
            const unsigned slot = (blockIdx.x + 7u * blockIdx.y + 13u * blockIdx.z) % kCounterSlots;
            atomicAdd(args.counters + slot, (unsigned long long)s_culled);
        }
    }
}

// Guarded batches (the host could not prove w > 0 and bounded coordinates
// over the slab): the reference's scalar per-voxel body with IEEE divisions,
// the 1e9 guard and the w == 0 flag, taps straight from the raw projection.
// Grid (ceil(L/32), ceil(L/8), ceil(nz/R)), 256 threads.
template <int MODE>
__global__ void __launch_bounds__(256)
bp_guarded_raw(const __grid_constant__ TmaArgs args, const __grid_constant__ TmaMats mats) {
    constexpr int R = kGR;
    const int x = blockIdx.x * 32 + (threadIdx.x & 31);
    const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
    const int zoff = blockIdx.z * R >= args.gap_at ? blockIdx.z * R + args.gap : blockIdx.z * R;
    const int L = args.L;
    if (x >= L || y >= L)
        return;
    const int zfirst = args.z_begin + zoff;
    const int nvalid = max(0, min(R, args.z_end - zfirst));
    const float wx = __fadd_rn(args.O, __fmul_rn((float)x, args.MM));
    const float wy = __fadd_rn(args.O, __fmul_rn((float)y, args.MM));
    const size_t plane = (size_t)L * L;
    float* volp = args.vol + (size_t)zoff * plane + (size_t)y * L + x;
    float acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r)
        acc[r] = r < nvalid ? volp[(size_t)r * plane] : 0.0f;
    bool zero_w = false;
    for (int p = 0; p < args.count; ++p) {
        const float* m = mats.a[p];
        const RawFetch f = raw_fetch(args, p);
        const float tu = __fadd_rn(__fmul_rn(wx, m[M01]), __fmul_rn(wy, m[M34]));
        const float tv = __fadd_rn(__fmul_rn(wx, m[M01 + 1]), __fmul_rn(wy, m[M34 + 1]));
        const float tw = __fadd_rn(__fmul_rn(wx, m[M2]), __fmul_rn(wy, m[M5]));
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const float wz =
                __fadd_rn(args.O, __fmul_rn((float)min(zfirst + r, args.z_end - 1), args.MM));
            const float u = __fadd_rn(__fadd_rn(tu, __fmul_rn(wz, m[M67])), m[M910]);
            const float v = __fadd_rn(__fadd_rn(tv, __fmul_rn(wz, m[M67 + 1])), m[M910 + 1]);
            const float w = __fadd_rn(__fadd_rn(tw, __fmul_rn(wz, m[M8])), m[M11]);
            zero_w |= r < nvalid && w == 0.0f;
            acc[r] = __fadd_rn(acc[r], update_ieee_raw<MODE, true>(f, u, v, w));
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
        if (r < nvalid)
            volp[(size_t)r * plane] = acc[r];
    if (zero_w)
        atomicOr(args.err, 1);
}

// Per-projection scan of the raw batch (replaces pack_quads' side duties):
// flags[p] bit 0 when some pixel has |value| >= 2^86 (the fast weight
// division's numerator bound, see kBigBits), err bit 2 on a non-finite
// pixel (ProjectionImage::validate, proj/src/dataset.cpp:123-129).
// Grid (blocks per projection, count), 256 threads, float4 loads when the
// projection stride allows.
__global__ void __launch_bounds__(256)
scan_projections(const float* __restrict__ raw, long long n, long long stride,
                 unsigned* __restrict__ flags, int* __restrict__ err) {
    const float* img = raw + (long long)blockIdx.y * stride;
    unsigned big = 0u;
    bool bad = false;
    const bool vec = ((reinterpret_cast<unsigned long long>(img) | (unsigned long long)n) & 3) == 0;
    if (vec) {
        const float4* v4 = reinterpret_cast<const float4*>(img);
        for (long long i = blockIdx.x * 256ll + threadIdx.x; i < n / 4; i += gridDim.x * 256ll) {
            const float4 q = __ldg(v4 + i);
            big = max(big, max(max(__float_as_uint(q.x) & 0x7FFFFFFFu, __float_as_uint(q.y) & 0x7FFFFFFFu),
                               max(__float_as_uint(q.z) & 0x7FFFFFFFu, __float_as_uint(q.w) & 0x7FFFFFFFu)));
        }
    } else {
        for (long long i = blockIdx.x * 256ll + threadIdx.x; i < n; i += gridDim.x * 256ll)
            big = max(big, __float_as_uint(__ldg(img + i)) & 0x7FFFFFFFu);
    }
    // non-finite <=> exponent all ones <=> |bits| >= 0x7F800000
    bad = big >= 0x7F800000u;
    const bool any_big = __syncthreads_or(big >= kBigBits);
    const bool any_bad = __syncthreads_or(bad);
    if (threadIdx.x == 0) {
        if (any_big)
            atomicOr(flags + blockIdx.y, 1u);
        if (any_bad && err)
            atomicOr(err, 2);
    }
}

} // namespace cbb
