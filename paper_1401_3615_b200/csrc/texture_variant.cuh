// texture_variant.cuh -- hardware-texture bilinear back-projection, the
// north_star's "side number" variant: the texture unit interpolates with
// 8-bit fractional weights and floor (not truncation) addressing, and the
// coordinates use FMA + approximate reciprocal, so it does NOT meet parity
// with the reference; it is reported beside the exact/fast results with its
// measured deviation. Raw projections are copied into a layered 2D CUDA
// array (border addressing -> taps off the detector read 0).
#pragma once

#include <cuda_runtime.h>

namespace cbb {

template <int R>
__global__ void __launch_bounds__(256, 2)
bp_texture_kernel(float* __restrict__ vol, int L, int z_begin, int z_end, float O, float MM,
                  cudaTextureObject_t tex, int layer0, int count,
                  const __grid_constant__ BpMats mats) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int x = blockIdx.x * kBlockX + (warp & 3) * 8 + (lane & 7);
    const int y = blockIdx.y * kBlockY + (warp >> 2) * 4 + (lane >> 3);
    const int zfirst = z_begin + blockIdx.z * R;
    if (x >= L || y >= L)
        return;
    const int nvalid = max(0, min(R, z_end - zfirst));
    const float wx = O + (float)x * MM, wy = O + (float)y * MM;
    const size_t plane = (size_t)L * L;
    float* volp = vol + (size_t)(zfirst - z_begin) * plane + (size_t)y * L + x;
    float acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r)
        acc[r] = r < nvalid ? volp[(size_t)r * plane] : 0.0f;
    for (int p = 0; p < count; ++p) {
        const float* m = mats.a[p];
        const float tu = fmaf(wy, m[M34], wx * m[M01]);
        const float tv = fmaf(wy, m[M34 + 1], wx * m[M01 + 1]);
        const float tw = fmaf(wy, m[M5], wx * m[M2]);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const float wz = O + (float)(zfirst + r) * MM;
            const float u = fmaf(wz, m[M67], tu) + m[M910];
            const float v = fmaf(wz, m[M67 + 1], tv) + m[M910 + 1];
            const float w = fmaf(wz, m[M8], tw) + m[M11];
            const float rw = __frcp_rn(w);
            const float val = tex2DLayered<float>(tex, u * rw + 0.5f, v * rw + 0.5f, layer0 + p);
            acc[r] = fmaf(val, rw * rw, acc[r]);
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
        if (r < nvalid)
            volp[(size_t)r * plane] = acc[r];
}

} // namespace cbb
