// common.cuh — shared device definitions for the sm_100a hot path.
//
// Data layout in HBM:
//   * parameters, f64 SoA [14][Gp]  (row k = flat-layout parameter k, types.hpp:15-20)
//   * CG / P-vectors, f32 SoA [14][Gp]
//   * per (view, Gaussian) splat record, f32 x 12 (48 B, float4-aligned):
//       {mx, my, A, B, C, opacity, r, g, b, -, -, -}
//     A, B, C are the conic pre-scaled to the log2 domain
//     (A = -0.5*ca*log2e, B = -cb*log2e, C = -0.5*cc*log2e) so the raster
//     evaluates alpha = o * 2^(A dx^2 + B dx dy + C dy^2) with one MUFU.EX2.
//   * per (view, Gaussian) tangent record (Jv probe), f32 x 12:
//       {A1, A2, A3, A4, A5, dopacity, dr, dg, db, -, -, -}
//     where d(power) = A1 dx + A2 dy + A3 dx^2 + A4 dx dy + A5 dy^2, i.e.
//     A1 = -(ca dmx + cb dmy), A2 = -(cb dmx + cc dmy), A3 = -dca/2,
//     A4 = -dcb, A5 = -dcc/2 (pre-combined by k_tangents)
//   * per (view, Gaussian) J^T accumulator, f32 x 12:
//       {g_mx, g_my, g_ca, g_cb, g_cc, g_opacity, g_r, g_g, g_b, -, -, -}
//     (the 9-float intermediate of jacobian.cpp:63-65)
#pragma once

#include "layout.hpp"

namespace slm {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ int warp_max_i(int v) {
    return __reduce_max_sync(0xffffffffu, v);
}

// The single gate/alpha evaluation every raster kernel shares, so the forward
// render and all derivative passes make identical FP32 decisions
// (blend_pixel rasterizer.hpp:110-124).  Explicit _rn intrinsics pin the
// rounding: no kernel may contract these differently.
struct Alpha {
    float alpha;
    float e;  // 2^q = exp(power): the falloff before opacity, = alpha/o when not clamped
    float dx, dy;
    bool clamped;
};

__device__ __forceinline__ bool eval_alpha(const float4 r0, const float4 r1, float pxc, float pyc,
                                           Alpha& a) {
    // r0 = {mx, my, A, B}, r1 = {C, opacity, r, g}
    const float dx = __fsub_rn(r0.x, pxc);
    const float dy = __fsub_rn(r0.y, pyc);
    const float q = __fmaf_rn(__fmul_rn(r0.z, dx), dx,
                              __fmaf_rn(__fmul_rn(r1.x, dy), dy, __fmul_rn(__fmul_rn(r0.w, dx), dy)));
    a.dx = dx;
    a.dy = dy;
    if (q > 0.0f) return false;  // power > 0: skip
    float e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(q));
    a.e = e;
    float alpha = __fmul_rn(r1.y, e);
    a.clamped = alpha > 0.99f;
    if (a.clamped) alpha = 0.99f;
    a.alpha = alpha;
    return alpha >= (float)(1.0 / 255.0);  // alpha < 1/255: skip
}

// Termination test (rasterizer.hpp:121-122): the entry that would push T
// under 1e-4 is not blended and ends the pixel.
__device__ __forceinline__ bool terminates(float T, float alpha, float& test_t) {
    test_t = __fmul_rn(T, __fsub_rn(1.0f, alpha));
    return test_t < 1e-4f;
}

}  // namespace slm
