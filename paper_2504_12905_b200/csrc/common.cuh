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

// The single gate / alpha evaluation every raster kernel shares (blend_pixel,
// rasterizer.hpp:110-124), so the forward render, the blend masks, the alpha
// stream and the diag make identical FP32 decisions.  Per (entry, tile) the
// log2 of the unclamped alpha is a quadratic in the pixel centre (x, y)
// relative to the tile centre:
//   q' = log2(o) + power log2(e) = (g0 + g1 x + g3 x^2) + (g2 + g4 x) y + g5 y^2
// (A, B, C of the record are the conic pre-scaled to the log2 domain), so
// alpha = 2^q' takes one MUFU.EX2, the skip gate alpha < 1/255 is
// q' < log2(1/255) -- no exponential for the ~85% of pairs it rejects -- and
// power > 0 is q' > log2(o).  Explicit _rn intrinsics pin the rounding: no
// kernel may contract these differently.
struct Gate {
    float g0, g1, g2, g3, g4, g5, lo;  // lo = log2(o)
};
// Packed FP32 FMA (sm_100 FFMA2): d = a * b + c on two lanes of a float2.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}

__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}

__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}

__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}

constexpr float kLog2Skip = -7.99435343685885793f;  // log2(1/255)

__device__ __forceinline__ Gate make_gate(const float4 r0, const float4 r1, float ox, float oy) {
    // r0 = {mx, my, A, B}, r1 = {C, opacity, r, g}
    const float mx = __fsub_rn(r0.x, ox), my = __fsub_rn(r0.y, oy);
    const float A = r0.z, B = r0.w, C = r1.x;
    Gate g;
    g.lo = log2f(r1.y);
    const float ax = __fmul_rn(A, mx), cy = __fmul_rn(C, my);
    g.g0 = __fadd_rn(__fmaf_rn(ax, mx, __fmaf_rn(__fmul_rn(B, mx), my, __fmul_rn(cy, my))), g.lo);
    g.g1 = -__fmaf_rn(B, my, __fmul_rn(2.0f, ax));
    g.g2 = -__fmaf_rn(B, mx, __fmul_rn(2.0f, cy));
    g.g3 = A;
    g.g4 = B;
    g.g5 = C;
    return g;
}

struct PixQ {  // pixel centre relative to the tile centre (half-integers) and its squares
    float x, y, xx, yy;
};
__device__ __forceinline__ PixQ pix_q(float x, float y) { return PixQ{x, y, __fmul_rn(x, x), __fmul_rn(y, y)}; }
// q' factored by column: the x-only parts (gx0 = g0 + g1 x + g3 x^2, gx1 = g2 + g4 x)
// are shared by every pixel of a column (the render evaluates 4 pixels of one
// column per entry); every kernel uses exactly these operations.
__device__ __forceinline__ float gate_x0(const Gate& g, float x, float xx) {
    return __fmaf_rn(g.g3, xx, __fmaf_rn(g.g1, x, g.g0));
}
__device__ __forceinline__ float gate_x1(const Gate& g, float x) { return __fmaf_rn(g.g4, x, g.g2); }
__device__ __forceinline__ float gate_qy(const Gate& g, float gx0, float gx1, float y, float yy) {
    return __fmaf_rn(g.g5, yy, __fmaf_rn(gx1, y, gx0));
}
__device__ __forceinline__ float gate_q(const Gate& g, const PixQ& p) {
    return gate_qy(g, gate_x0(g, p.x, p.xx), gate_x1(g, p.x), p.y, p.yy);
}
// alpha (clamped at 0.99, rasterizer.hpp:15) of a pair from q'; false: a gate skips it.
__device__ __forceinline__ bool gate_alpha(float q, float lo, float& alpha, bool& clamped) {
    if (q > lo || q < kLog2Skip) return false;  // power > 0, or alpha < 1/255
    float e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(q));
    clamped = e > 0.99f;
    alpha = clamped ? 0.99f : e;
    return true;
}

// alpha of a pair the FP64 decision (k_masks) already blends: no gate test,
// so a pair sitting within FP32 rounding of a gate keeps its alpha.
__device__ __forceinline__ void blended_alpha(float q, float& alpha, bool& clamped) {
    float e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(q));
    clamped = e > 0.99f;
    alpha = clamped ? 0.99f : e;
}

// Termination test (rasterizer.hpp:121-122): the entry that would push T
// under 1e-4 is not blended and ends the pixel.
__device__ __forceinline__ bool terminates(float T, float alpha, float& test_t) {
    test_t = __fmul_rn(T, __fsub_rn(1.0f, alpha));
    return test_t < 1e-4f;
}

// ---- TMA bulk copies (cp.async.bulk global -> shared, mbarrier completion)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// One lane: arm the barrier with the byte count and start the copy.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// Copy only (the barrier is armed separately).
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

}  // namespace slm
