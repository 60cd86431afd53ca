// raster.cu — FP32 tile rasterizers.
//
//  * k_render          full-image forward (render_with_context, rasterizer.cpp:62-91),
//                      one CTA per 16x16 tile, splat records staged in smem; writes
//                      RGB, final T, contrib count and `last` (the list position
//                      where blend_pixel stopped) and per-tile SSE vs ground truth.
//  * k_masks           once per (state, plan): for every sampled pixel one bit per
//                      tile-list entry saying whether blend_pixel blends it (alpha
//                      gates passed and before `last`).  The gates depend only on the
//                      state, not on the probe p, so the per-product passes never
//                      re-evaluate the ~85% of (pixel, entry) pairs that are skipped.
//  * k_sample_raster   the sampled-pixel products, one warp per group of <=32 samples
//                      of one tile, walking the list in windows of 32 entries:
//        JVP   Jv      dual blend (jvp, jacobian.cpp:191-211)
//        VJP   J^T u   reverse blend into the 9-float intermediate (vjp :219-247)
//        GN    J^T W J p fused: Jv, *W, J^T in one kernel (gn_apply :339-344)
//        RHS   J^T(-W r) with r read from the forward render (lm.cpp:99-121)
//  * k_diag_raster     diag(J^T W J) accumulators (jtj_diag :272-337), factored as a
//                      per-(tile, Gaussian) 5x5 quadratic form.
//
// Window walk (all sampled passes).  In window w every lane iterates only over
// ITS OWN blended entries (its mask word), so lanes do blend work instead of
// idling through a shared entry loop.  The J^T reduction over the 32 pixels
// of an entry is done without atomics or 32-lane shuffles: phase A (lane =
// pixel) keeps T and the colour prefix and writes two scalars per blended
// (pixel, entry) pair into a smem [pixel][entry] tile; the 32x32 mask matrix is
// transposed with a 5-stage shuffle bit transpose; phase B (lane = entry)
// gathers its column of pixels, rebuilds the intermediate in registers and
// adds it to HBM with vector red.global.add (one per 4 floats per entry).
// The next window's mask and splat records are prefetched into registers
// while the current window runs.
//
// The J^T passes sweep front-to-back: the reference's reverse sweep needs
// suffix_c = sum_{j>k} w_j c_j (backward_pixel_vjp :67-94); with the pixel's
// final colour C from the forward render, suffix = C - prefix_incl(k), and
// prefix is accumulated with the very same FP32 operations as the forward
// render, so gate decisions and sums replay exactly.
#include <cstdint>

#include <atomic>

#include "common.cuh"

namespace slm { extern std::atomic<long long> g_launches; }

namespace slm {

// ------------------------------------------------------------------ K6
// One CTA of 64 threads per 16x16 tile; warp w owns the 16x8 half-tile of rows
// 8w..8w+7, thread (lane l) the 4 pixels of column l & 15 at rows
// 8w + (l >> 4) + 2i, so every broadcast read of a staged splat record serves
// 4 pixels.  Per staged entry, the bounding box of its alpha >= 1/255 ellipse
// (conservatively widened) lets a warp skip the entry when the box misses its
// half-tile: every pixel there would fail the reference's alpha gate anyway.
// Per pixel the arithmetic is blend_pixel's (eval_alpha).
constexpr int kRenderThreads = 64;
constexpr int kRenderPix = 4;      // pixels per thread
constexpr int kRenderStage = 128;  // records staged per round
#ifndef SLM_LOSS_ENTRIES
#define SLM_LOSS_ENTRIES 2
#endif
constexpr int kLossE = SLM_LOSS_ENTRIES;  // list entries per iteration of the loss render

// Bounding box of {alpha >= 1/255} for a record (A, B, C: log2-domain conic,
// o: opacity): q = A dx^2 + B dx dy + C dy^2 >= L = log2(1/(255 o)).
__device__ __forceinline__ float4 alpha_box(float4 r0, float4 r1) {
    const float A = r0.z, B = r0.w, C = r1.x, o = r1.y;
    const float det = A * C - 0.25f * B * B;  // > 0 for a valid (negative-definite) conic
    const float L = -__log2f(255.0f * o);     // <= 0 when o >= 1/255
    if (!(det > 0.0f) || !(L < 0.0f)) return make_float4(1e30f, -1e30f, 1e30f, -1e30f);  // never blends
    // half-widths sqrt(L * C / det), sqrt(L * A / det) (all three signs negative),
    // widened by 0.1% + 0.05 px, which also covers sqrt.approx's few-ulp error
    const float ld = L / det;
    float hx, hy;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(hx) : "f"(fmaxf(ld * C, 0.0f)));
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(hy) : "f"(fmaxf(ld * A, 0.0f)));
    hx = hx * 1.001f + 0.05f;
    hy = hy * 1.001f + 0.05f;
    return make_float4(r0.x - hx, r0.x + hx, r0.y - hy, r0.y + hy);
}

// Maximum of the (concave) gate polynomial q'(x, y) over the rectangle
// [x0, x1] x [y0, y1] (tile-centred coordinates): the stationary point when it
// lies inside, else the best of the four edges (each a 1-D concave quadratic).
__device__ __forceinline__ float gate_rect_max(const Gate& g, float x0, float x1, float y0, float y1) {
    const float det = 4.0f * g.g3 * g.g5 - g.g4 * g.g4;
    if (det > 0.0f) {
        const float xs = (g.g4 * g.g2 - 2.0f * g.g5 * g.g1) / det, ys = (g.g4 * g.g1 - 2.0f * g.g3 * g.g2) / det;
        if (xs >= x0 && xs <= x1 && ys >= y0 && ys <= y1)
            return g.g0 + g.g1 * xs + g.g2 * ys + g.g3 * xs * xs + g.g4 * xs * ys + g.g5 * ys * ys;
    }
    float best = -1e30f;
    auto along_y = [&](float x) {  // x fixed, maximise over y
        const float a = g.g0 + g.g1 * x + g.g3 * x * x, b = g.g2 + g.g4 * x;
        const float y = g.g5 < 0.0f ? fminf(fmaxf(-b / (2.0f * g.g5), y0), y1) : (b > 0.0f ? y1 : y0);
        best = fmaxf(best, a + b * y + g.g5 * y * y);
    };
    auto along_x = [&](float y) {
        const float a = g.g0 + g.g2 * y + g.g5 * y * y, b = g.g1 + g.g4 * y;
        const float x = g.g3 < 0.0f ? fminf(fmaxf(-b / (2.0f * g.g3), x0), x1) : (b > 0.0f ? x1 : x0);
        best = fmaxf(best, a + b * x + g.g3 * x * x);
    };
    along_y(x0);
    along_y(x1);
    along_x(y0);
    along_x(y1);
    return best;
}

#ifndef SLM_RENDER_MINB
#define SLM_RENDER_MINB 16
#endif
// The 4 pixels of a thread are two packed pairs (rows 0,1 and 2,3 of its
// column); each entry is blended branch-free: a pixel whose gate fails gets
// alpha = 0, which leaves T (T (1 - 0) = T) and the colour (fma(0, c, C) = C)
// bit-identical, so only the rare termination takes a branch, and every
// packed op (fma/mul/sub .rn.f32x2) rounds each pixel like the scalar
// blend_pixel arithmetic.  FULL: also write T, contrib and `last` (the
// drop-in render); the LM step's loss renders need only colour + SSE.
template <bool STATS, bool FULL>
__global__ void __launch_bounds__(kRenderThreads, SLM_RENDER_MINB) k_render(
    const DevCam* __restrict__ cams, const int* __restrict__ tile_view,
    const int* __restrict__ tile_offsets, const int* __restrict__ entries,
    const float4* __restrict__ rec, int Gp, const float* __restrict__ gt,
    float* __restrict__ image, float* __restrict__ trans, int* __restrict__ contrib,
    int* __restrict__ last_out, double* __restrict__ sse_tile, unsigned long long* __restrict__ stats) {
    __shared__ float4 s_rec[kRenderStage + 1][3];  // + a zero-alpha record (the loss loop's odd-count pad)
    __shared__ float4 s_box[STATS ? kRenderStage : 1];
    __shared__ unsigned s_wm[kRenderStage];  // bit w: the entry's alpha box meets warp w's half-tile
    __shared__ unsigned char s_list[kRenderThreads / 32][kRenderStage + 4];  // per warp: its staged entries (+ pads)
    __shared__ double s_red[kRenderThreads / 32];
    const int tile = blockIdx.x;
    const int v = tile_view[tile];
    const DevCam& cam = cams[v];
    const int lt = tile - cam.tile_base;
    const int tx = lt % cam.tiles_x, ty = lt / cam.tiles_x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int x = tx * kTile + (lane & 15);
    const int y0 = ty * kTile + 8 * warp + (lane >> 4);
    const float pxc = (float)x + 0.5f;
    // this warp's half-tile in pixel-centre coordinates
    const float wx0 = (float)(tx * kTile) + 0.5f, wx1 = wx0 + 15.0f;
    const float wy0 = (float)(ty * kTile + 8 * warp) + 0.5f, wy1 = wy0 + 7.0f;
    const int b = tile_offsets[tile], n = tile_offsets[tile + 1] - b;
    const size_t vbase = static_cast<size_t>(v) * Gp;

    const float tcx = (float)(tx * kTile + kTile / 2), tcy = (float)(ty * kTile + kTile / 2);
    const float qx = pxc - tcx, qxx = __fmul_rn(qx, qx);
    // pair p holds pixels 2p, 2p+1 (rows y0 + 4p, y0 + 4p + 2)
    float2 T[2], C0[2], C1[2], C2[2], qy[2], qyy[2];
    int cnt[4], last[4];
    unsigned live = 0u;  // bit i: pixel i still blending
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        T[p] = make_float2(1.0f, 1.0f);
        C0[p] = C1[p] = C2[p] = make_float2(0.0f, 0.0f);
        float yv[2], yy[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int i = 2 * p + h, y = y0 + 2 * i;
            cnt[i] = 0;
            last[i] = n;
            yv[h] = (float)y + 0.5f - tcy;
            yy[h] = __fmul_rn(yv[h], yv[h]);
            if (x < cam.width && y < cam.height) live |= 1u << i;
            else {  // a dead pixel's gate is -huge: every pair skips it
                yv[h] = 0.0f;
                yy[h] = 1e30f;
            }
        }
        qy[p] = make_float2(yv[0], yv[1]);
        qyy[p] = make_float2(yy[0], yy[1]);
    }
    unsigned long long st_iter = 0, st_box = 0, st_live = 0, st_blend = 0, st_stage = 0, st_exact = 0, st_useful = 0;
    constexpr bool kLoss = !FULL && !STATS;
    if (kLoss && threadIdx.x < 3)  // q' = -1e30 at every pixel: alpha 0, colour 0
        s_rec[kRenderStage][threadIdx.x] = make_float4(threadIdx.x == 0 ? -1e30f : 0.f, 0.f, 0.f, 0.f);
    for (int start = 0; start < n; start += kRenderStage) {
        if (__syncthreads_count(live != 0u) == 0) break;
        if (STATS) st_stage += min(kRenderStage, n - start);
        for (int j = threadIdx.x; j < kRenderStage && start + j < n; j += kRenderThreads) {
            const float4* r = rec + 3 * (vbase + entries[b + start + j]);
            const float4 r0 = r[0], r1 = r[1], r2 = r[2];
            const Gate g = make_gate(r0, r1, tcx, tcy);
            s_rec[j][0] = make_float4(g.g0, g.g1, g.g2, g.g3);
            s_rec[j][1] = make_float4(g.g4, g.g5, g.lo, r1.z);
            s_rec[j][2] = make_float4(r1.w, r2.x, 0.f, 0.f);
            const float4 bx = alpha_box(r0, r1);
            if (STATS) s_box[j] = bx;
            // the half-tiles span x in [tx 16 + .5, + 15], y in [ty 16 + 8 w + .5, + 7]
            const float x0 = (float)(tx * kTile) + 0.5f, y0h = (float)(ty * kTile) + 0.5f;
            const bool inx = !(bx.y < x0 || bx.x > x0 + 15.0f);
            const unsigned m0 = (inx && !(bx.w < y0h || bx.z > y0h + 7.0f)) ? 1u : 0u;
            const unsigned m1 = (inx && !(bx.w < y0h + 8.0f || bx.z > y0h + 15.0f)) ? 2u : 0u;
            s_wm[j] = m0 | m1;
        }
        __syncthreads();
        const int m = min(kRenderStage, n - start);
        // this warp's list of the staged entries whose alpha box meets its
        // half-tile (ballot compaction, in list order): the walk below never
        // visits an entry it would skip
        int nk = 0;
        for (int j0 = 0; j0 < m; j0 += 32) {
            const int j = j0 + lane;
            const bool hit = j < m && ((s_wm[j] >> warp) & 1u);
            const unsigned bal = __ballot_sync(0xffffffffu, hit);
            if (hit) s_list[warp][nk + __popc(bal & ((1u << lane) - 1u))] = static_cast<unsigned char>(j);
            nk += __popc(bal);
        }
        if (kLoss && lane == 0)
            for (int j = nk; j < ((nk + kLossE - 1) / kLossE) * kLossE; ++j)
                s_list[warp][j] = static_cast<unsigned char>(kRenderStage);
        __syncwarp();
        if (STATS && live) st_iter += m;
        if constexpr (kLoss) {
            // loss render: kLossE entries per iteration, one loop test and one
            // termination test per group (a list ends on zero-alpha records)
            for (int ii = 0; ii < nk && live; ii += kLossE) {
                float2 a[kLossE][2];  // [entry][pixel pair]
                float4 cc[kLossE];    // the entries' colours
#pragma unroll
                for (int e = 0; e < kLossE; ++e) {
                    const int k = s_list[warp][ii + e];
                    const float4 q0 = s_rec[k][0], q1 = s_rec[k][1], q2 = s_rec[k][2];
                    cc[e] = make_float4(q1.w, q2.x, q2.y, 0.f);
                    const float gx0 = __fmaf_rn(q0.w, qxx, __fmaf_rn(q0.y, qx, q0.x)), gx1 = __fmaf_rn(q1.x, qx, q0.z);
#pragma unroll
                    for (int p = 0; p < 2; ++p) {
                        const float2 q = ffma2(make_float2(q1.y, q1.y), qyy[p],
                                               ffma2(make_float2(gx1, gx1), qy[p], make_float2(gx0, gx0)));
                        float e0, e1;
                        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(q.x));
                        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(q.y));
                        // the alpha < 1/255 skip; the clamp at 0.99 (power > 0: see below)
                        a[e][p] = make_float2(q.x >= kLog2Skip ? fminf(e0, 0.99f) : 0.0f,
                                              q.y >= kLog2Skip ? fminf(e1, 0.99f) : 0.0f);
                    }
                }
                float2 w[kLossE][2], Te[kLossE][2];
                float tmin = 1.0f;
#pragma unroll
                for (int e = 0; e < kLossE; ++e)
#pragma unroll
                    for (int p = 0; p < 2; ++p) {
                        w[e][p] = fmul2(a[e][p], T[p]);
                        T[p] = fsub2(T[p], w[e][p]);
                        Te[e][p] = T[p];
                        tmin = fminf(tmin, fminf(T[p].x, T[p].y));
                    }
                // termination (rasterizer.hpp:121-122): the entry that would push T
                // under 1e-4 is not blended and the pixel stops there (rare)
                if (tmin < 1e-4f) {
#pragma unroll
                    for (int p = 0; p < 2; ++p) {
                        bool l = false, h = false;
#pragma unroll
                        for (int e = 0; e < kLossE; ++e) {
                            l = l || Te[e][p].x < 1e-4f;
                            h = h || Te[e][p].y < 1e-4f;
                            w[e][p] = make_float2(l ? 0.0f : w[e][p].x, h ? 0.0f : w[e][p].y);
                        }
                        if (l) live &= ~(1u << (2 * p));
                        if (h) live &= ~(1u << (2 * p + 1));
                        T[p] = make_float2(l ? 1.0f : T[p].x, h ? 1.0f : T[p].y);
                        qy[p] = make_float2(l ? 0.0f : qy[p].x, h ? 0.0f : qy[p].y);
                        qyy[p] = make_float2(l ? 1e30f : qyy[p].x, h ? 1e30f : qyy[p].y);
                    }
                }
#pragma unroll
                for (int e = 0; e < kLossE; ++e)
#pragma unroll
                    for (int p = 0; p < 2; ++p) {
                        C0[p] = ffma2(w[e][p], make_float2(cc[e].x, cc[e].x), C0[p]);
                        C1[p] = ffma2(w[e][p], make_float2(cc[e].y, cc[e].y), C1[p]);
                        C2[p] = ffma2(w[e][p], make_float2(cc[e].z, cc[e].z), C2[p]);
                    }
            }
            continue;
        }
        for (int ii = 0; ii < nk && live; ++ii) {
            const int k = s_list[warp][ii];
            const float4 q0 = s_rec[k][0], q1 = s_rec[k][1], q2 = s_rec[k][2];
            const Gate g{q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z};
            const float gx0 = gate_x0(g, qx, qxx), gx1 = gate_x1(g, qx);  // shared by the column
            // q' of the 4 pixels as two packed FMA chains (fma.rn.f32x2 rounds each
            // lane like __fmaf_rn: gate_qy's q'); dead pixels carry qyy = 1e30
            float2 a[2];
            bool ps[4];
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                const float2 q = ffma2(make_float2(g.g5, g.g5), qyy[p],
                                       ffma2(make_float2(gx1, gx1), qy[p], make_float2(gx0, gx0)));
                const float qv[2] = {q.x, q.y};
                float av[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    float e;
                    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(qv[h]));
                    e = fminf(e, 0.99f);  // clamp (rasterizer.hpp:15)
                    // the alpha < 1/255 skip only: power > 0 (q' > log2 o) cannot happen
                    // for a valid splat (positive definite conic) except by the FP32
                    // rounding of q' within ~1e-3 px of a centre, so that test of
                    // blend_pixel is left to the exact FP64 passes (k_masks,
                    // k_render_exact); STATS keeps it for the work counters
                    if (STATS) {
                        ps[2 * p + h] = !(qv[h] > g.lo || qv[h] < kLog2Skip);
                        av[h] = ps[2 * p + h] ? e : 0.0f;
                    } else {
                        ps[2 * p + h] = qv[h] >= kLog2Skip;
                        av[h] = ps[2 * p + h] ? e : 0.0f;
                    }
                }
                a[p] = make_float2(av[0], av[1]);
            }
            if constexpr (!FULL && !STATS) {
                // loss render (colour only): w = alpha T, T' = T - w (one rounding
                // each; the loss is compared to the f64 reference within tolerance),
                // updated in place; a terminated pixel gets w = 0 and T = 1 (its T is
                // not an output, and T = 1 never triggers the test again)
                float2 w[2];
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    w[p] = fmul2(a[p], T[p]);
                    T[p] = fsub2(T[p], w[p]);
                }
                if (fminf(fminf(T[0].x, T[0].y), fminf(T[1].x, T[1].y)) < 1e-4f) {
                    // termination (rasterizer.hpp:121-122): not blended, the pixel stops (rare)
#pragma unroll
                    for (int p = 0; p < 2; ++p) {
                        const bool l = T[p].x < 1e-4f, h = T[p].y < 1e-4f;
                        if (l) live &= ~(1u << (2 * p));
                        if (h) live &= ~(1u << (2 * p + 1));
                        w[p] = make_float2(l ? 0.0f : w[p].x, h ? 0.0f : w[p].y);
                        T[p] = make_float2(l ? 1.0f : T[p].x, h ? 1.0f : T[p].y);
                        qy[p] = make_float2(l ? 0.0f : qy[p].x, h ? 0.0f : qy[p].y);
                        qyy[p] = make_float2(l ? 1e30f : qyy[p].x, h ? 1e30f : qyy[p].y);
                    }
                }
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    C0[p] = ffma2(w[p], make_float2(q1.w, q1.w), C0[p]);
                    C1[p] = ffma2(w[p], make_float2(q2.x, q2.x), C1[p]);
                    C2[p] = ffma2(w[p], make_float2(q2.y, q2.y), C2[p]);
                }
            } else {
                float2 tt[2];
    #pragma unroll
                for (int p = 0; p < 2; ++p) tt[p] = fmul2(T[p], fsub2(make_float2(1.0f, 1.0f), a[p]));
                // a pixel that fails the gate keeps tt = T >= 1e-4 (alpha = 0), so
                // tt < 1e-4 alone marks a termination
                if (fminf(fminf(tt[0].x, tt[0].y), fminf(tt[1].x, tt[1].y)) < 1e-4f) {
                    // termination (rasterizer.hpp:121-122): not blended, the pixel stops (rare)
                    const bool tm0 = tt[0].x < 1e-4f, tm1 = tt[0].y < 1e-4f, tm2 = tt[1].x < 1e-4f, tm3 = tt[1].y < 1e-4f;
                    const bool tm[4] = {tm0, tm1, tm2, tm3};
    #pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if (tm[i]) {
                            ps[i] = false;
                            live &= ~(1u << i);
                            if (FULL) last[i] = start + k;
                        }
    #pragma unroll
                    for (int p = 0; p < 2; ++p) {
                        const bool l = tm[2 * p], h = tm[2 * p + 1];
                        a[p] = make_float2(l ? 0.0f : a[p].x, h ? 0.0f : a[p].y);
                        tt[p] = make_float2(l ? T[p].x : tt[p].x, h ? T[p].y : tt[p].y);
                        qy[p] = make_float2(l ? 0.0f : qy[p].x, h ? 0.0f : qy[p].y);
                        qyy[p] = make_float2(l ? 1e30f : qyy[p].x, h ? 1e30f : qyy[p].y);
                    }
                }
    #pragma unroll
                for (int p = 0; p < 2; ++p) {
                    const float2 w = fmul2(a[p], T[p]);
                    C0[p] = ffma2(w, make_float2(q1.w, q1.w), C0[p]);
                    C1[p] = ffma2(w, make_float2(q2.x, q2.x), C1[p]);
                    C2[p] = ffma2(w, make_float2(q2.y, q2.y), C2[p]);
                    T[p] = tt[p];
                }
            }
            if (FULL) {
#pragma unroll
                for (int i = 0; i < 4; ++i) cnt[i] += ps[i] ? 1 : 0;
            }
            if (STATS) {
                const int nb = (ps[0] ? 1 : 0) + (ps[1] ? 1 : 0) + (ps[2] ? 1 : 0) + (ps[3] ? 1 : 0);
                ++st_box;
                st_live += __popc(live);
                st_blend += nb;
                const unsigned act = __activemask();
                const bool leader = (threadIdx.x & 31) == __ffs(act) - 1;  // one count per warp
                if (leader && gate_rect_max(g, wx0 - tcx, wx1 - tcx, wy0 - tcy, wy1 - tcy) >= kLog2Skip - 0.01f)
                    ++st_exact;
                if (__any_sync(act, nb > 0) && leader) ++st_useful;
            }
        }
    }
    double sq = 0.0;
#pragma unroll
    for (int i = 0; i < kRenderPix; ++i) {
        const int y = y0 + 2 * i;
        const float c0 = (i & 1) ? C0[i >> 1].y : C0[i >> 1].x;
        const float c1 = (i & 1) ? C1[i >> 1].y : C1[i >> 1].x;
        const float c2 = (i & 1) ? C2[i >> 1].y : C2[i >> 1].x;
        if (x < cam.width && y < cam.height) {
            const size_t pix = cam.pix_base + static_cast<size_t>(y) * cam.width + x;
            image[3 * pix] = c0;
            image[3 * pix + 1] = c1;
            image[3 * pix + 2] = c2;
            if (FULL) {
                trans[pix] = (i & 1) ? T[i >> 1].y : T[i >> 1].x;
                contrib[pix] = cnt[i];
                last_out[pix] = last[i];
            }
            if (gt) {
                const float* gp = gt + 3 * pix;
                const double d0 = (double)c0 - (double)gp[0], d1 = (double)c1 - (double)gp[1],
                             d2 = (double)c2 - (double)gp[2];
                sq += d0 * d0 + d1 * d1 + d2 * d2;
            }
        }
    }
    if (STATS) {  // diagnostic counters (slm_debug_render_stats): per thread, summed per warp
        unsigned long long v[7] = {st_iter, st_box, st_live, st_blend, st_stage, st_exact, st_useful};
        for (int q = 0; q < 7; ++q) {
            unsigned long long x = v[q];
            for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            if ((threadIdx.x & 31) == 0) atomicAdd(stats + (q < 5 ? q : q + 3), x);
        }
    }
    if (sse_tile) {
        sq = warp_sum_d(sq);
        if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = sq;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int i = 0; i < kRenderThreads / 32; ++i) s += s_red[i];
            sse_tile[tile] = s;
        }
    }
}

// Per-view SSE in fixed order (deterministic): one warp per view.
__global__ void k_sse_views(const DevCam* __restrict__ cams, int V, int n_tiles_total,
                            const double* __restrict__ sse_tile, double* __restrict__ sse_view) {
    const int v = blockIdx.x;
    if (v >= V) return;
    const int base = cams[v].tile_base, nt = cams[v].tiles_x * cams[v].tiles_y;
    double s = 0.0;
    for (int i = threadIdx.x; i < nt; i += 32) s += sse_tile[base + i];
    s = warp_sum_d(s);
    if (threadIdx.x == 0) sse_view[v] = s;
}

// ------------------------------------------------------------------ group setup
// One warp per group of <= 32 samples of one tile; lane = sample pixel.
struct GroupCtx {
    bool active;
    int s, orig;
    size_t pix, vbase;
    float pxc, pyc;  // pixel centre (x + 0.5, y + 0.5), rasterizer.cpp:82
    float ox, oy;    // tile centre: origin of the local pixel coordinates of the J^T moments
    int tile;        // batch tile index
};

__device__ __forceinline__ bool setup_group(const Group* groups, int n_groups, const DevCam* cams,
                                            const int* spix, const int* sorig, int Gp, int gi, int lane,
                                            GroupCtx& c) {
    if (gi >= n_groups) return false;
    const Group grp = groups[gi];
    const DevCam& cam = cams[grp.view];
    c.active = lane < grp.count;
    c.s = grp.begin + (c.active ? lane : 0);
    const int packed = spix[c.s];
    const int px = packed & 0xffff, py = packed >> 16;
    c.orig = sorig ? sorig[c.s] : 0;
    c.pix = cam.pix_base + static_cast<size_t>(py) * cam.width + px;
    c.vbase = static_cast<size_t>(grp.view) * Gp;
    c.pxc = (float)px + 0.5f;
    c.pyc = (float)py + 0.5f;
    const int tx = grp.tile % cam.tiles_x, ty = grp.tile / cam.tiles_x;
    c.ox = (float)(tx * kTile + kTile / 2);
    c.oy = (float)(ty * kTile + kTile / 2);
    c.tile = cam.tile_base + grp.tile;
    return true;
}

// 32x32 bit-matrix transpose across the warp: in, lane l holds row l (bit k =
// column k); out, lane k holds column k (bit l = row l).  5 shuffle stages.
__device__ __forceinline__ unsigned transpose32(unsigned x, int lane) {
    const unsigned masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const int j = 16 >> i;
        const unsigned y = __shfl_xor_sync(0xffffffffu, x, j);
        if (lane & j) x ^= ((y >> j) ^ x) & masks[i];
        else x ^= (((x >> j) ^ y) & masks[i]) << j;
    }
    return x;
}

// ------------------------------------------------------------------ masks
// Once per (state, plan), one warp per group.  Walks the tile list up to the
// group's furthest `last` in windows of 32 entries; bit k of a pixel's word =
// entry k is blended there (same eval_alpha as k_render, and k < last).  The
// window stream is then COMPACTED to the entries at least one of the group's
// pixels blends (~72% at configs[2]): their Gaussian indices go to glist in
// list order and the pixel bits are re-packed (column compaction through two
// bit transposes) into 32-entry windows, so the per-product passes walk dense
// windows and never stage an entry no lane uses.
__global__ void __launch_bounds__(128, 8) k_masks(SampleArgs A) {  // 64 registers: 8 CTAs per SM
    __shared__ double s_r[4][32][6];  // staged entries: FP64 mx, my, a, b, c, o
    __shared__ double s_thr[4][32];   // power below which alpha < 1/255 for sure
    // FP32 gate polynomials (pre-filter), entry pairs interleaved so one packed
    // FFMA2 chain evaluates two entries: [pair][q] = (g_2q(a), g_2q(b), g_2q+1(a), g_2q+1(b))
    __shared__ float4 s_g[4][16][3];
    __shared__ float s_c[4][32][3];   // their colours
    __shared__ unsigned s_col[4][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gi = blockIdx.x * 4 + warp;
    GroupCtx c;
    if (!setup_group(A.groups, A.n_groups, A.cams, A.spix, nullptr, A.Gp, gi, lane, c)) return;
    // blend_pixel (rasterizer.hpp:100-130) in FP64 with the reference's operation
    // order (no contraction), so blended sets, termination and C_final are the
    // reference's decisions, not the FP32 render's
    const double px = static_cast<double>(c.pxc), py = static_cast<double>(c.pyc);
    const PixQ pq = pix_q(c.pxc - c.ox, c.pyc - c.oy);
    const int* tl = A.entries + A.tile_offsets[c.tile];
    const int n = A.tile_offsets[c.tile + 1] - A.tile_offsets[c.tile];
    const long long off = A.mask_off[gi];
    int* glist = A.glist_out + off;
    unsigned* mout = A.masks_out + off;
    int run = 0, nb = 0, cw = 0, rows = 0;
    unsigned long long buf = 0ull;
    bool live = c.active;
    double T = 1.0, C0 = 0.0, C1 = 0.0, C2 = 0.0;
    for (int base = 0; base < n; base += 32) {
        if (!__any_sync(0xffffffffu, live)) break;
        const int j = base + lane;
        int g = 0;
        if (j < n) {
            g = tl[j];
            const float4* rf = A.rec + 3 * (c.vbase + g);
            const float4 r0 = rf[0], r1 = rf[1];
            s_c[warp][lane][0] = r1.z;
            s_c[warp][lane][1] = r1.w;
            s_c[warp][lane][2] = rf[2].x;
            const Gate gt = make_gate(r0, r1, c.ox, c.oy);
            float* pg = reinterpret_cast<float*>(&s_g[warp][lane >> 1][0]) + (lane & 1);
            pg[0] = gt.g0;
            pg[2] = gt.g1;
            pg[4] = gt.g2;
            pg[6] = gt.g3;
            pg[8] = gt.g4;
            pg[10] = gt.g5;
        }
        __syncwarp();
        const int mn = min(32, n - base);
        // FP32 pre-filter (the shared gate): a pair whose q' is below log2(1/255) by
        // far more than FP32 rounding cannot blend; the others are decided in FP64,
        // and only entries some lane may blend get their FP64 record staged
        // two entries per packed chain (fma.rn.f32x2 rounds each lane like the
        // scalar gate_q); an odd last entry evaluates stale coefficients, masked off
        unsigned cand = 0u;
        if (live) {
            const float2 X = make_float2(pq.x, pq.x), XX = make_float2(pq.xx, pq.xx);
            const float2 Y = make_float2(pq.y, pq.y), YY = make_float2(pq.yy, pq.yy);
            for (int k = 0; k < mn; k += 2) {
                const float4 a = s_g[warp][k >> 1][0], b = s_g[warp][k >> 1][1], d = s_g[warp][k >> 1][2];
                const float2 gx0 = ffma2(make_float2(b.z, b.w), XX, ffma2(make_float2(a.z, a.w), X, make_float2(a.x, a.y)));
                const float2 gx1 = ffma2(make_float2(d.x, d.y), X, make_float2(b.x, b.y));
                const float2 q = ffma2(make_float2(d.z, d.w), YY, ffma2(gx1, Y, gx0));
                const unsigned two = (q.x >= kLog2Skip - 0.5f ? 1u : 0u) | (q.y >= kLog2Skip - 0.5f ? 2u : 0u);
                cand |= two << k;  // FP32 q' error < 1e-3 measured
            }
            if (mn < 32) cand &= (1u << mn) - 1u;
        }
        const unsigned any_cand = __reduce_or_sync(0xffffffffu, cand);
        if (j < n && ((any_cand >> lane) & 1u)) {
            const double* r = A.rec64 + 6 * (c.vbase + g);
#pragma unroll
            for (int q = 0; q < 6; ++q) s_r[warp][lane][q] = r[q];
            // o exp(power) < 1/255 whenever power < log(1/(255 o)) by more than the
            // rounding of log/exp/multiply: those pairs skip without the exponential
            s_thr[warp][lane] = r[5] > 0.0 ? log(kAlphaSkipD / r[5]) - 1e-9 : -1e300;
        }
        __syncwarp();
        unsigned bits = 0u;
        for (unsigned cm = cand; cm && live; cm &= cm - 1) {
            const int k = __ffs(cm) - 1;
            const double* e = s_r[warp][k];
            const double dx = __dsub_rn(e[0], px), dy = __dsub_rn(e[1], py);
            const double power =
                __dsub_rn(__dmul_rn(-0.5, __dadd_rn(__dmul_rn(__dmul_rn(e[2], dx), dx), __dmul_rn(__dmul_rn(e[4], dy), dy))),
                          __dmul_rn(__dmul_rn(e[3], dx), dy));
            if (power > 0.0 || power < s_thr[warp][k]) continue;
            double alpha = __dmul_rn(e[5], exp(power));
            if (alpha > kAlphaClampD) alpha = kAlphaClampD;
            if (alpha < kAlphaSkipD) continue;
            const double test_t = __dmul_rn(T, __dsub_rn(1.0, alpha));
            if (test_t < kTFloorD) {
                live = false;  // not blended; the pixel stops
                break;
            }
            const double w = __dmul_rn(alpha, T);
            C0 = __dadd_rn(C0, __dmul_rn(w, static_cast<double>(s_c[warp][k][0])));
            C1 = __dadd_rn(C1, __dmul_rn(w, static_cast<double>(s_c[warp][k][1])));
            C2 = __dadd_rn(C2, __dmul_rn(w, static_cast<double>(s_c[warp][k][2])));
            T = test_t;
            bits |= 1u << k;
        }
        const unsigned un = __reduce_or_sync(0xffffffffu, bits);
        const int rank = __popc(un & ((1u << lane) - 1u));
        const unsigned col = transpose32(bits, lane);  // lane k: pixels blending entry k
        if ((un >> lane) & 1u) {
            glist[run + rank] = g;
            s_col[warp][rank] = col;
        }
        __syncwarp();
        const int nu = __popc(un);
        const unsigned packed = transpose32(lane < nu ? s_col[warp][lane] : 0u, lane);
        buf |= static_cast<unsigned long long>(packed) << nb;
        nb += nu;
        run += nu;
        if (nb >= 32) {
            const unsigned word = static_cast<unsigned>(buf);
            mout[32 * cw + lane] = word;
            rows += __reduce_max_sync(0xffffffffu, __popc(word));
            ++cw;
            buf >>= 32;
            nb -= 32;
        }
        __syncwarp();
    }
    if (nb > 0) {
        const unsigned word = static_cast<unsigned>(buf);
        mout[32 * cw + lane] = word;
        rows += __reduce_max_sync(0xffffffffu, __popc(word));
    }
    if (c.active) {
        A.scol_out[3 * c.s] = static_cast<float>(C0);
        A.scol_out[3 * c.s + 1] = static_cast<float>(C1);
        A.scol_out[3 * c.s + 2] = static_cast<float>(C2);
    }
    if (lane == 0) {
        A.gcount_out[gi] = run;
        A.grows_out[gi] = rows;
    }
}

// An alpha-stream word: the pair's alpha (negated when clamped) rounded to a
// multiple of 32 ulp (<= 16 ulp = 1e-6 relative), its compacted entry index k
// in the low 5 bits, so the product walks need no bit iteration over masks.
__device__ __forceinline__ float alpha_word(float a, int k) {
    return __uint_as_float(((__float_as_uint(a) + 16u) & ~31u) | static_cast<unsigned>(k));
}
__device__ __forceinline__ int word_entry(float w) { return static_cast<int>(__float_as_uint(w) & 31u); }
__device__ __forceinline__ float word_alpha(float w) { return __uint_as_float(__float_as_uint(w) & ~31u); }

// Once per (state, plan), after k_masks: the alpha of every blended pair in
// the order the product passes consume them (SampleArgs::srow_off), so the
// passes never re-evaluate the Gaussian falloff: alpha comes from a TMA-staged
// row, and the geometry enters the derivative passes only through the
// pre-combined tangent polynomial.  Same eval_alpha as k_render / k_masks.
// Also writes each window's record block (SampleArgs::rstream), so the
// products gather no state-only record: it arrives by TMA with the rows.
__global__ void __launch_bounds__(128) k_alpha(SampleArgs A) {
    __shared__ float4 s_rec[4][32][2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gi = blockIdx.x * 4 + warp;
    GroupCtx c;
    if (!setup_group(A.groups, A.n_groups, A.cams, A.spix, nullptr, A.Gp, gi, lane, c)) return;
    const int nun = A.gcount[gi];
    const int* list = A.glist + A.mask_off[gi];
    const unsigned* masks = A.masks + A.mask_off[gi];
    float* out = A.astream_out + 32 * A.srow_off[gi];
    const PixQ pq = pix_q(c.pxc - c.ox, c.pyc - c.oy);
    float* blk = A.rstream_out + static_cast<size_t>(kRecBlock) * A.wbase[gi];
    for (int w = 0, row = 0; 32 * w < nun; ++w, blk += kRecBlock) {
        const int j = 32 * w + lane;
        float4 r0 = make_float4(0.f, 0.f, 0.f, 0.f), r1 = r0;
        float rb = 0.f;
        if (j < nun) {
            const float4* r = A.rec + 3 * (c.vbase + list[j]);
            r0 = r[0];
            r1 = r[1];
            rb = r[2].x;
            const Gate gt = make_gate(r0, r1, c.ox, c.oy);
            s_rec[warp][lane][0] = make_float4(gt.g0, gt.g1, gt.g2, gt.g3);
            s_rec[warp][lane][1] = make_float4(gt.g4, gt.g5, gt.lo, 0.f);
        }
        blk[0 * 32 + lane] = r0.x;
        blk[1 * 32 + lane] = r0.y;
        blk[2 * 32 + lane] = r0.z;
        blk[3 * 32 + lane] = r0.w;
        blk[4 * 32 + lane] = r1.x;
        blk[5 * 32 + lane] = r1.y;
        blk[6 * 32 + lane] = r1.z;
        blk[7 * 32 + lane] = r1.w;
        blk[8 * 32 + lane] = rb;
        unsigned m = c.active ? masks[32 * w + lane] : 0u;
        const int npc = __reduce_max_sync(0xffffffffu, __popc(m));
        A.cols_out[A.mask_off[gi] + 32 * w + lane] = transpose32(m, lane);
        __syncwarp();
        for (int i = 0; m; m &= m - 1, ++i) {
            const int k = __ffs(m) - 1;
            const float4 q0 = s_rec[warp][k][0], q1 = s_rec[warp][k][1];
            const Gate gt{q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z};
            float alpha = 0.0f;
            bool cl = false;
            blended_alpha(gate_q(gt, pq), alpha, cl);  // blended: the mask already decided
            out[32 * (row + i) + lane] = alpha_word(cl ? -alpha : alpha, k);
        }
        row += npc;
        __syncwarp();
    }
}

// ------------------------------------------------------------------ mask statistics
// Diagnostic (tools/mask_stats.py) over the compacted windows:
// st[0] groups, [1] windows, [2] blended pairs, [3] sum_w max_lane popc (the
// per-lane sparse walks' iteration count), [4] compacted entries, [5] sum over
// 64-entry windows of max popc, [6] sum_w max column popc.
__global__ void __launch_bounds__(32) k_mask_stats(SampleArgs A, unsigned long long* st) {
    const int lane = threadIdx.x;
    GroupCtx c;
    if (!setup_group(A.groups, A.n_groups, A.cams, A.spix, nullptr, A.Gp, blockIdx.x, lane, c)) return;
    const int nun = A.gcount[blockIdx.x];
    const int ncw = (nun + 31) >> 5;
    const unsigned* masks = A.masks + A.mask_off[blockIdx.x];
    unsigned long long s[7] = {1ull, (unsigned long long)ncw, 0ull, 0ull, (unsigned long long)nun, 0ull, 0ull};
    int rem = c.active ? __popc(masks[lane]) : 0;
    for (int w = 0; w < ncw; ++w) {
        const unsigned m = c.active ? masks[32 * w + lane] : 0u;
        {   // run-ahead simulation: lanes done with window w continue into w+1
            const int nxt = (c.active && w + 1 < ncw) ? __popc(masks[32 * (w + 1) + lane]) : 0;
            const int steps = __reduce_max_sync(0xffffffffu, rem);
            s[5] += steps;
            rem = nxt - min(steps - rem, nxt);
        }
        s[2] += __popc(m);
        s[3] += __reduce_max_sync(0xffffffffu, __popc(m));
        s[6] += __reduce_max_sync(0xffffffffu, __popc(transpose32(m, lane)));

    }
    for (int o = 16; o; o >>= 1) s[2] += __shfl_xor_sync(0xffffffffu, s[2], o);
    if (lane == 0)
        for (int i = 0; i < 7; ++i)
            if (s[i]) atomicAdd(st + i, s[i]);
    // Balance simulations (pair steps per warp): [13] 64-entry windows (max
    // lane popcount per 64 entries), [14]/[15]/[16] lanes may run ahead of the
    // oldest unfinished window by 1 / 3 / unlimited windows, [17] two-pair
    // iterations of the current walk (sum_w ceil(max popc / 2)).
    unsigned long long x[5] = {0ull, 0ull, 0ull, 0ull, 0ull};
    for (int w = 0; w < ncw; w += 2) {
        int p = c.active ? __popc(masks[32 * w + lane]) : 0;
        if (w + 1 < ncw && c.active) p += __popc(masks[32 * (w + 1) + lane]);
        x[0] += __reduce_max_sync(0xffffffffu, p);
    }
    for (int w = 0; w < ncw; ++w) {
        const int p = c.active ? __popc(masks[32 * w + lane]) : 0;
        x[4] += (__reduce_max_sync(0xffffffffu, p) + 1) >> 1;
    }
    const int look[3] = {1, 3, 1 << 30};
    for (int q = 0; q < 3; ++q) {
        // lane position: the first window it has not finished (ncw = done)
        int wl = 0, rem = (c.active && ncw > 0) ? __popc(masks[lane]) : 0;
        unsigned long long steps = 0;
        while (true) {
            const int wmin = __reduce_min_sync(0xffffffffu, rem > 0 ? wl : wl + 1);
            if (wmin >= ncw) break;
            // advance past exhausted windows (free) within the look-ahead of the oldest
            while (rem == 0 && wl + 1 < ncw && wl + 1 <= wmin + look[q]) {
                ++wl;
                rem = c.active ? __popc(masks[32 * wl + lane]) : 0;
            }
            const bool work = rem > 0;
            if (!__any_sync(0xffffffffu, work)) continue;
            if (work) --rem;
            ++steps;
        }
        x[1 + q] = steps;
    }
    if (lane == 0)
        for (int i = 0; i < 5; ++i)
            if (x[i]) atomicAdd(st + 13 + i, x[i]);
}

void launch_mask_stats(const SampleArgs& a, unsigned long long* st, cudaStream_t stream) {
    if (a.n_groups == 0) return;
    k_mask_stats<<<a.n_groups, 32, 0, stream>>>(a, st); ++g_launches;
}

// ------------------------------------------------------------------ products
__device__ __forceinline__ void red_add_v4(float* dst, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(a), "f"(b), "f"(c),
                 "f"(d)
                 : "memory");
}


// Window prefetch (lane = compacted entry 32w+lane): mask word of the lane's
// pixel and the entry's splat record (and tangent record).
struct Prefetch {
    unsigned m;
    int g;
    float4 r0, r1, r2, t0, t1, t2;
};

struct WinCtx {
    const int* list;
    const unsigned* masks;
    int nun, nwin;
};

template <bool TAN>
__device__ __forceinline__ void prefetch(const GroupCtx& c, const WinCtx& W, const float4* __restrict__ rec,
                                         const float4* __restrict__ tan, int w, int lane, Prefetch& P) {
    P.m = 0u;
    if (w >= W.nwin) return;
    P.m = c.active ? W.masks[w * 32 + lane] : 0u;
    const int j = w * 32 + lane;
    if (j < W.nun) {
        P.g = W.list[j];
        const size_t rg = c.vbase + P.g;
        P.r0 = rec[3 * rg];
        P.r1 = rec[3 * rg + 1];
        P.r2 = rec[3 * rg + 2];
        if (TAN) {
            P.t0 = tan[3 * rg];
            P.t1 = tan[3 * rg + 1];
            P.t2 = tan[3 * rg + 2];
        }
    }
}

// Two-stage window pipeline for the product passes: while window w runs, the
// records of window w+1 and the mask word / list index of window w+2 are in
// flight, so no load result is consumed in the window that issued it.
struct WinPipe {
    unsigned m_cur, m_nxt;  // mask words of windows w, w+1
    int g_cur, g_nxt;       // Gaussian index of this lane's entry in windows w, w+1
    float4 t0, t1, t2;      // tangent record of this lane's entry in window w
};

__device__ __forceinline__ void win_index(const GroupCtx& c, const WinCtx& W, int w, int lane, unsigned& m, int& g) {
    m = 0u;
    g = 0;
    if (w < W.nwin) {
        m = c.active ? W.masks[w * 32 + lane] : 0u;
        if (w * 32 + lane < W.nun) g = W.list[w * 32 + lane];
    }
}

template <bool TAN>
__device__ __forceinline__ void win_records(const GroupCtx& c, const WinCtx& W, const float4* __restrict__ tan, int w,
                                            int g, int lane, WinPipe& P) {
    if (w < W.nwin && w * 32 + lane < W.nun) {
        const size_t rg = c.vbase + g;
        P.t0 = tan[3 * rg];
        P.t1 = tan[3 * rg + 1];
        P.t2 = tan[3 * rg + 2];
    }
}

template <bool TAN>
__device__ __forceinline__ void win_start(const GroupCtx& c, const WinCtx& W, const float4* tan, int lane, WinPipe& P) {
    win_index(c, W, 0, lane, P.m_cur, P.g_cur);
    win_records<TAN>(c, W, tan, 0, P.g_cur, lane, P);
    win_index(c, W, 1, lane, P.m_nxt, P.g_nxt);
}

// After window w's tangents are staged: start window w+1's tangents and w+2's index.
template <bool TAN>
__device__ __forceinline__ void win_advance(const GroupCtx& c, const WinCtx& W, const float4* tan, int w, int lane,
                                            WinPipe& P) {
    win_records<TAN>(c, W, tan, w + 1, P.g_nxt, lane, P);
    P.m_cur = P.m_nxt;
    P.g_cur = P.g_nxt;
    win_index(c, W, w + 2, lane, P.m_nxt, P.g_nxt);
}

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Write a 9-float record (3 float4, first 9 used) as column `lane` of [9][32].
__device__ __forceinline__ void stage_rec(float (*dst)[32], int lane, float4 a, float4 b, float4 c) {
    dst[0][lane] = a.x;
    dst[1][lane] = a.y;
    dst[2][lane] = a.z;
    dst[3][lane] = a.w;
    dst[4][lane] = b.x;
    dst[5][lane] = b.y;
    dst[6][lane] = b.z;
    dst[7][lane] = b.w;
    dst[8][lane] = c.x;
}

// Double-buffered window inputs of one warp: window w's alpha rows and record
// block land in buffer w & 1 (one mbarrier per buffer, one transaction count),
// the copies for window w+1 are in flight while window w runs.
// Rows staged per window by TMA; the rest (windows whose busiest lane blends
// more than 18 entries) are prefetched into L2 with the window and read from
// global.  18 (not the ~98th-percentile 22) so the product CTA fits 7 per SM.
#ifndef SLM_ALPHA_ROWS
#define SLM_ALPHA_ROWS 18
#endif
constexpr int kAlphaRows = SLM_ALPHA_ROWS;

struct AlphaPipe {
    float* buf0;
    float* buf1;
    float* rbuf0;
    float* rbuf1;
    uint64_t* bar;
    const float* src;      // the group's first alpha row
    const float* rsrc;     // the group's first record block
    long long next;        // row of the next window to issue
    long long row0, row1;  // first row of the window held in each buffer
    uint32_t par;          // parity bit per buffer
    __device__ __forceinline__ void issue(int w, int rows, int lane) {
        const int staged = min(rows, kAlphaRows);
        if (lane == 0) {
            uint64_t* b = bar + (w & 1);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                         "r"(128u * staged + 4u * kRecBlock)
                         : "memory");
            if (staged > 0) bulk_copy((w & 1) ? buf1 : buf0, src + 32 * next, 128u * staged, b);
            if (rows > staged)  // the overflow rows, read later from global: warm them into L2
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + 32 * (next + staged)),
                             "r"(128u * (rows - staged))
                             : "memory");
            bulk_copy((w & 1) ? rbuf1 : rbuf0, rsrc + static_cast<size_t>(kRecBlock) * w, 4u * kRecBlock, b);
        }
        if (w & 1) row1 = next;
        else row0 = next;
        next += rows;
    }
    __device__ __forceinline__ const float* wait(int w) {
        mbar_wait(bar + (w & 1), (par >> (w & 1)) & 1u);
        par ^= 1u << (w & 1);
        return (w & 1) ? buf1 : buf0;
    }
    __device__ __forceinline__ const float* block(int w) const { return (w & 1) ? rbuf1 : rbuf0; }
    // rows beyond kAlphaRows are read from global memory (rare)
    __device__ __forceinline__ const float* overflow(int w) const {
        return src + 32 * (((w & 1) ? row1 : row0) + kAlphaRows);
    }
};

__device__ __forceinline__ int max_popc(unsigned m) { return __reduce_max_sync(0xffffffffu, __popc(m)); }

// The sampled-pixel products over the compacted window stream.
//  pass 1 (JVP/GN, lane = pixel): dual blend over the lane's own blended
//    entries of each window (jvp, jacobian.cpp:191-211).  alpha comes from
//    the stream; d alpha = alpha * Q(x, y) with Q the entry's tangent d(power)
//    + do/o re-expanded as a quadratic in the pixel's tile-local coordinates
//    (6 coefficients staged per window), so no per-pair geometry is recomputed;
//  J^T (VJP/GN/RHS), per window:
//    phase A (lane = pixel): front-to-back over the lane's blended entries,
//      keeping T and the colour prefix S; suffix = C_final - S_incl gives
//      dL/dalpha (backward_pixel_vjp :67-94); the pair scalars
//      (dL/dpower, alpha T) go to a smem [pixel][entry] tile;
//    phase B (lane = entry): dense walk over the 32 pixels with broadcast
//      reads of the pixel's local coordinates and u, accumulating six moments
//      sum dL/dpower * {1, x, y, x^2, xy, y^2} and sum alpha T u_c with packed
//      FFMA2; the entry's conic turns the moments into the 9-float
//      intermediate gradient once (dL/do = sum dL/dpower / o), one vector
//      red.global.add per 4 floats.
#ifndef SLM_RASTER_WARPS
#define SLM_RASTER_WARPS 2
#endif
constexpr int kRasterWarps = SLM_RASTER_WARPS;

template <int MODE>
__global__ void __maxnreg__(144) k_sample_raster(SampleArgs A) {  // 144 regs x 64 threads: 7 CTAs per SM
    constexpr int NW = kRasterWarps;
    __shared__ __align__(128) float s_alpha[NW][2][kAlphaRows * 32];
    __shared__ __align__(128) float s_blk[NW][2][kRecBlock];  // record blocks [9][32] (TMA)
    // pass-1 staging, struct-of-arrays so lanes reading different entries hit
    // different banks: tau0..5, dr, dg, db
    // [pixel][entry]: (dL/dpower, alpha T); pass 1's [9][32] staging lives in
    // the same memory (the passes never overlap), which with 18 staged alpha
    // rows keeps a 2-warp CTA at 32 KB: 7 CTAs (14 warps) per SM
    __shared__ __align__(16) float2 s_pair[NW][32][33];
    __shared__ float4 s_phi[NW][32];  // per pixel: (x, y, u0, u1), tile-centre coords
    __shared__ float s_u2[NW][32];
    __shared__ uint64_t s_bar[NW][2];
    if (A.done_flag && *A.done_flag) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gi = blockIdx.x * NW + warp;
    GroupCtx c;
    if (!setup_group(A.groups, A.n_groups, A.cams, A.spix, A.sorig, A.Gp, gi, lane, c)) return;
    WinCtx W;
    W.nun = A.gcount[gi];
    W.nwin = (W.nun + 31) >> 5;
    W.list = A.glist + A.mask_off[gi];
    W.masks = A.masks + A.mask_off[gi];
    float(*sf)[32] = reinterpret_cast<float(*)[32]>(&s_pair[warp][0][0]);
    if (lane == 0) {
        mbar_init(&s_bar[warp][0], 1);
        mbar_init(&s_bar[warp][1], 1);
    }
    __syncwarp();
    AlphaPipe ap{s_alpha[warp][0], s_alpha[warp][1], s_blk[warp][0], s_blk[warp][1], s_bar[warp],
                 A.astream + 32 * A.srow_off[gi], A.rstream + static_cast<size_t>(kRecBlock) * A.wbase[gi], 0, 0, 0, 0u};
    const float lx = c.pxc - c.ox, ly = c.pyc - c.oy;

    float u0 = 0.f, u1 = 0.f, u2 = 0.f;
    if (MODE == kJvp || MODE == kGn) {
        const float lxx = lx * lx, lxy = lx * ly, lyy = ly * ly;
        float T = 1.0f, dT = 0.0f, dC0 = 0.f, dC1 = 0.f, dC2 = 0.f;
        WinPipe P;
        win_start<true>(c, W, A.tan, lane, P);
        int rows = max_popc(P.m_cur);
        if (W.nwin > 0) ap.issue(0, rows, lane);
        for (int w = 0; w < W.nwin; ++w) {
            const unsigned m = P.m_cur;
            const int cur = rows;
            const float* sp = ap.wait(w) + lane;
            const float(*blk)[32] = reinterpret_cast<const float(*)[32]>(ap.block(w));
            if (w * 32 + lane < W.nun) {
                // Q(x, y) = d(power) + do/o about the tile centre: with dx = mx - x,
                // d(power) = A1 dx + A2 dy + A3 dx^2 + A4 dx dy + A5 dy^2
                const float mx = blk[0][lane] - c.ox, my = blk[1][lane] - c.oy;
                const float A1 = P.t0.x, A2 = P.t0.y, A3 = P.t0.z, A4 = P.t0.w, A5 = P.t1.x;
                sf[0][lane] = A1 * mx + A2 * my + mx * (A3 * mx + A4 * my) + A5 * my * my +
                              __fdividef(P.t1.y, blk[5][lane]);
                sf[1][lane] = -A1 - 2.0f * A3 * mx - A4 * my;
                sf[2][lane] = -A2 - A4 * mx - 2.0f * A5 * my;
                sf[3][lane] = A3;
                sf[4][lane] = A4;
                sf[5][lane] = A5;
                sf[6][lane] = P.t1.z;
                sf[7][lane] = P.t1.w;
                sf[8][lane] = P.t2.x;
            }
            __syncwarp();
            rows = max_popc(P.m_nxt);
            if (w + 1 < W.nwin) ap.issue(w + 1, rows, lane);
            win_advance<true>(c, W, A.tan, w, lane, P);
            // two pairs per iteration (the second predicated: alpha = 0 is neutral
            // in the dual blend), so the loads of both overlap
            auto pair = [&](int k, float av) {
                const float alpha = fabsf(av);
                const float Q = sf[0][k] + lx * sf[1][k] + ly * sf[2][k] + lxx * sf[3][k] + lxy * sf[4][k] +
                                lyy * sf[5][k];
                const float dalpha = av < 0.0f ? 0.0f : alpha * Q;
                const float wgt = alpha * T;
                const float dw = fmaf(dalpha, T, alpha * dT);
                dC0 = fmaf(dw, blk[6][k], dC0);
                dC0 = fmaf(wgt, sf[6][k], dC0);
                dC1 = fmaf(dw, blk[7][k], dC1);
                dC1 = fmaf(wgt, sf[7][k], dC1);
                dC2 = fmaf(dw, blk[8][k], dC2);
                dC2 = fmaf(wgt, sf[8][k], dC2);
                const float om = __fsub_rn(1.0f, alpha);
                dT = fmaf(dT, om, -T * dalpha);
                T = __fmul_rn(T, om);
            };
            // n pairs from q (row stride 32): the words carry the entry index;
            // the next iteration's two words are loaded one iteration ahead
            auto walk = [&](int n, const float* q) {
                float nx1 = n > 0 ? q[0] : 0.0f, nx2 = n > 1 ? q[32] : 0.0f;
                for (int i = 0; i < n; i += 2) {
                    const float w1 = nx1, w2 = nx2;
                    q += 64;
                    nx1 = i + 2 < n ? q[0] : 0.0f;
                    nx2 = i + 3 < n ? q[32] : 0.0f;
                    pair(word_entry(w1), word_alpha(w1));
                    pair(word_entry(w2), word_alpha(w2));  // 0 (neutral) past the lane's last pair
                }
            };
            const int npair = __popc(m);
            walk(min(npair, kAlphaRows), sp);
            if (cur > kAlphaRows) walk(npair - min(npair, kAlphaRows), ap.overflow(w) + lane);
            __syncwarp();
        }
        if (MODE == kJvp) {
            if (c.active) {
                A.out_res[3 * c.orig] = dC0;
                A.out_res[3 * c.orig + 1] = dC1;
                A.out_res[3 * c.orig + 2] = dC2;
            }
            return;
        }
        if (c.active) {
            u0 = A.sw[3 * c.s] * dC0;
            u1 = A.sw[3 * c.s + 1] * dC1;
            u2 = A.sw[3 * c.s + 2] * dC2;
        }
        ap.next = 0;
    } else if (MODE == kVjp) {
        if (c.active) {
            u0 = A.in_res[3 * c.orig];
            u1 = A.in_res[3 * c.orig + 1];
            u2 = A.in_res[3 * c.orig + 2];
        }
    } else {  // kRhs: u = -w (rendered - truth)
        if (c.active) {
            const float* gp = A.gt + 3 * c.pix;
            u0 = -A.sw[3 * c.s] * (A.scol[3 * c.s] - gp[0]);
            u1 = -A.sw[3 * c.s + 1] * (A.scol[3 * c.s + 1] - gp[1]);
            u2 = -A.sw[3 * c.s + 2] * (A.scol[3 * c.s + 2] - gp[2]);
        }
    }

    // ---- J^T pass
    const float Cf0 = c.active ? A.scol[3 * c.s] : 0.f;  // C_final of the FP64 blend (k_masks)
    const float Cf1 = c.active ? A.scol[3 * c.s + 1] : 0.f;
    const float Cf2 = c.active ? A.scol[3 * c.s + 2] : 0.f;
    s_phi[warp][lane] = make_float4(lx, ly, u0, u1);
    s_u2[warp][lane] = u2;
    float2(*pt)[33] = s_pair[warp];
    const float uC = u0 * Cf0 + u1 * Cf1 + u2 * Cf2;
    float T = 1.0f, uS = 0.f;
    unsigned m_cur = 0u, m_nxt = 0u;
    int g_cur = 0, g_nxt = 0;
    win_index(c, W, 0, lane, m_cur, g_cur);
    win_index(c, W, 1, lane, m_nxt, g_nxt);
    int rows = max_popc(m_cur);
    if (W.nwin > 0) ap.issue(0, rows, lane);
    const unsigned* cols = A.cols + A.mask_off[gi];
    unsigned col_nxt = W.nwin > 0 ? cols[lane] : 0u;
    const long long slot0 = 32 * A.wbase[gi];  // deterministic mode: first slot of the group
    unsigned dest_nxt = (A.partial && W.nwin > 0 && lane < W.nun) ? A.dest[slot0 + lane] : 0u;
    __syncwarp();
    for (int w = 0; w < W.nwin; ++w) {
        const unsigned m0 = m_cur;
        const int cur = rows;
        const bool ent = w * 32 + lane < W.nun;
        const int e_g = g_cur;
        rows = max_popc(m_nxt);
        if (w + 1 < W.nwin) ap.issue(w + 1, rows, lane);
        m_cur = m_nxt;
        g_cur = g_nxt;
        win_index(c, W, w + 2, lane, m_nxt, g_nxt);
        const unsigned col = col_nxt;  // lane k: pixels that blend entry k
        if (w + 1 < W.nwin) col_nxt = cols[32 * (w + 1) + lane];
        const unsigned dest_w = dest_nxt;  // deterministic mode: this entry's record position
        if (A.partial && w + 1 < W.nwin && (w + 1) * 32 + lane < W.nun) dest_nxt = A.dest[slot0 + 32 * (w + 1) + lane];
        const float* sp = ap.wait(w) + lane;
        const float(*blk)[32] = reinterpret_cast<const float(*)[32]>(ap.block(w));
        // phase A (lane = pixel); with u.S_incl kept as one running scalar:
        // dL/dalpha = sum_c u_c (T c_c - (C_c - S_incl,c) / (1 - alpha))
        auto walk = [&](int n, const float* q) {
            float nx1 = n > 0 ? q[0] : 0.0f, nx2 = n > 1 ? q[32] : 0.0f;
            for (int i = 0; i < n; i += 2) {  // two pairs per iteration, the second predicated
                const bool two = i + 1 < n;
                const int k1 = word_entry(nx1), k2 = word_entry(nx2);
                const float av1 = word_alpha(nx1), av2 = word_alpha(nx2);
                q += 64;
                nx1 = i + 2 < n ? q[0] : 0.0f;
                nx2 = i + 3 < n ? q[32] : 0.0f;
                const float a1 = fabsf(av1), a2 = fabsf(av2);
                const float uc1 = u0 * blk[6][k1] + u1 * blk[7][k1] + u2 * blk[8][k1];
                const float uc2 = u0 * blk[6][k2] + u1 * blk[7][k2] + u2 * blk[8][k2];
                const float w1 = __fmul_rn(a1, T);
                uS = fmaf(w1, uc1, uS);
                const float om1 = __fsub_rn(1.0f, a1);
                const float d1 = fmaf(T, uc1, -(uC - uS) * rcp_approx(om1));
                pt[lane][k1] = make_float2(av1 < 0.0f ? 0.0f : d1 * a1, w1);
                T = __fmul_rn(T, om1);
                const float w2 = __fmul_rn(a2, T);
                uS = fmaf(w2, uc2, uS);
                const float om2 = __fsub_rn(1.0f, a2);
                const float d2 = fmaf(T, uc2, -(uC - uS) * rcp_approx(om2));
                if (two) pt[lane][k2] = make_float2(av2 < 0.0f ? 0.0f : d2 * a2, w2);
                T = __fmul_rn(T, om2);
            }
        };
        const int npair = __popc(m0);
        walk(min(npair, kAlphaRows), sp);
        if (cur > kAlphaRows) walk(npair - min(npair, kAlphaRows), ap.overflow(w) + lane);
        __syncwarp();
        // phase B (lane = entry), dense over the pixels
        float M0 = 0.f;
        float2 M12 = make_float2(0.f, 0.f), M34 = M12, M5G2 = M12, G01 = M12;
#pragma unroll
        for (int p = 0; p < 32; ++p) {
            float2 v = pt[p][lane];
            const bool b = (col >> p) & 1u;
            v.x = b ? v.x : 0.0f;
            v.y = b ? v.y : 0.0f;
            const float4 f0 = s_phi[warp][p];  // (x, y, u0, u1): 2 broadcast wavefronts
            const float fu2 = s_u2[warp][p];
            const float2 sq = fmul2(make_float2(f0.x, f0.x), make_float2(f0.x, f0.y));  // (x^2, xy)
            M12 = ffma2(make_float2(v.x, v.x), make_float2(f0.x, f0.y), M12);
            M34 = ffma2(make_float2(v.x, v.x), sq, M34);
            M5G2 = ffma2(v, make_float2(f0.y * f0.y, fu2), M5G2);
            G01 = ffma2(make_float2(v.y, v.y), make_float2(f0.z, f0.w), G01);
            M0 += v.x;
        }
        if (ent) {
            // moments about the tile centre -> sums over dx = mx - x, dy = my - y
            const float mx = blk[0][lane] - c.ox, my = blk[1][lane] - c.oy;
            const float sx = mx * M0 - M12.x, sy = my * M0 - M12.y;
            const float sxx = mx * (mx * M0 - 2.0f * M12.x) + M34.x;
            const float sxy = mx * (my * M0 - M12.y) - my * M12.x + M34.y;
            const float syy = my * (my * M0 - 2.0f * M12.y) + M5G2.x;
            constexpr float kLn2f = 0.69314718055994530942f;
            const float ca = -2.0f * kLn2f * blk[2][lane], cb = -kLn2f * blk[3][lane], cc = -2.0f * kLn2f * blk[4][lane];
            const float4 o0 = make_float4(-(ca * sx + cb * sy), -(cb * sx + cc * sy), -0.5f * sxx, -sxy);
            const float4 o1 = make_float4(-0.5f * syy, __fdividef(M0, blk[5][lane]), G01.x, G01.y);
            if (A.partial) {  // deterministic: this entry's own record, summed in order by k_chain
                float4* dst = reinterpret_cast<float4*>(A.partial) + (kDetRec / 4) * static_cast<size_t>(dest_w);
                dst[0] = o0;
                dst[1] = o1;
                dst[2] = make_float4(M5G2.y, 0.f, 0.f, 0.f);
                if (kDetRec == 16) dst[3] = make_float4(0.f, 0.f, 0.f, 0.f);  // full sectors
            } else {
                float* dst = A.inter + (c.vbase + e_g) * kRec;
                red_add_v4(dst, o0.x, o0.y, o0.z, o0.w);
                red_add_v4(dst + 4, o1.x, o1.y, o1.z, o1.w);
                atomicAdd(dst + 8, M5G2.y);
            }
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------ K13
// Per blended (pixel, entry), the reference adds for every channel c with
// weight W_c:  W_c (alpha T dcol_c)^2 to the colour rows, and (if not clamped)
// W_c (dp_c gpow . P_j)^2 to the 10 geometry rows, W_c (dalpha_c alpha/o dsig)^2
// to the opacity row.  With s = sum_c W_c dp_c^2 the geometry part is
// P_j^T (s gpow gpow^T) P_j, so we accumulate per entry the 5x5 symmetric
// M = sum_pixels s gpow gpow^T (15 floats), sum W_c dalpha_c^2 (alpha/o)^2 (1),
// and sum W_c (alpha T)^2 per channel (3); k_diag_finalize applies P_j,
// dsig and dcol (chain.cu).  Layout per (view, Gaussian): 20 floats.
// Same compacted window walk as the J^T pass, in half-windows of 16 entries:
// phase A (lane = pixel) writes (alpha^2 s, e^2 s, (alpha T)^2) per pair,
// phase B (lane = entry x pixel half) sums its column as monomials in (dx, dy).
__global__ void __launch_bounds__(128) k_diag_raster(DiagArgs A) {
    __shared__ float s_f[4][9][32];
    __shared__ float s_gate[4][7][32];  // the entries' gate polynomials (make_gate)
    __shared__ float s_io[4][32];        // the entries' 1/o
    __shared__ int s_g[4][32];
    __shared__ float s_t[4][3][32][17];
    __shared__ float4 s_pix[4][32];  // (px+.5, py+.5, W0, W1)
    __shared__ float s_pw2[4][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gi = blockIdx.x * 4 + warp;
    GroupCtx c;
    if (!setup_group(A.groups, A.n_groups, A.cams, A.spix, nullptr, A.Gp, gi, lane, c)) return;
    WinCtx W;
    W.nun = A.gcount[gi];
    W.nwin = (W.nun + 31) >> 5;
    W.list = A.glist + A.mask_off[gi];
    W.masks = A.masks + A.mask_off[gi];
    constexpr float kLn2f = 0.69314718055994530942f;
    float(*sf)[32] = s_f[warp];
    const float W0 = c.active ? A.sw[3 * c.s] : 0.f, W1 = c.active ? A.sw[3 * c.s + 1] : 0.f,
                W2 = c.active ? A.sw[3 * c.s + 2] : 0.f;
    const float Cf0 = c.active ? A.scol[3 * c.s] : 0.f;  // C_final of the FP64 blend (k_masks)
    const float Cf1 = c.active ? A.scol[3 * c.s + 1] : 0.f;
    const float Cf2 = c.active ? A.scol[3 * c.s + 2] : 0.f;
    s_pix[warp][lane] = make_float4(c.pxc, c.pyc, W0, W1);
    s_pw2[warp][lane] = W2;
    const int e16 = lane & 15, ph = lane >> 4;
    const unsigned pmask = ph ? 0xFFFF0000u : 0x0000FFFFu;
    const PixQ pq = pix_q(c.pxc - c.ox, c.pyc - c.oy);
    const long long slot0 = A.partial ? 32 * A.wbase[gi] : 0;  // deterministic mode: first slot of the group
    float T = 1.0f, S0 = 0.f, S1 = 0.f, S2 = 0.f;
    Prefetch P;
    prefetch<false>(c, W, A.rec, nullptr, 0, lane, P);
    __syncwarp();
    for (int w = 0; w < W.nwin; ++w) {
        const unsigned m0 = P.m;
        if (w * 32 + lane < W.nun) {
            stage_rec(sf, lane, P.r0, P.r1, P.r2);
            s_g[warp][lane] = P.g;
            const Gate gt = make_gate(P.r0, P.r1, c.ox, c.oy);
            s_gate[warp][0][lane] = gt.g0;
            s_gate[warp][1][lane] = gt.g1;
            s_gate[warp][2][lane] = gt.g2;
            s_gate[warp][3][lane] = gt.g3;
            s_gate[warp][4][lane] = gt.g4;
            s_gate[warp][5][lane] = gt.g5;
            s_gate[warp][6][lane] = gt.lo;
            s_io[warp][lane] = rcp_approx(P.r1.y);
        }
        __syncwarp();
        prefetch<false>(c, W, A.rec, nullptr, w + 1, lane, P);
        const unsigned col = A.cols[A.mask_off[gi] + 32 * w + lane];
        const int nent = min(32, W.nun - w * 32);
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            if (16 * h >= nent) break;
            for (unsigned m = (m0 >> (16 * h)) & 0xFFFFu; m; m &= m - 1) {
                const int kk = __ffs(m) - 1, k = 16 * h + kk;
                const Gate gt{s_gate[warp][0][k], s_gate[warp][1][k], s_gate[warp][2][k], s_gate[warp][3][k],
                              s_gate[warp][4][k], s_gate[warp][5][k], s_gate[warp][6][k]};
                float alpha = 0.0f;
                bool clamped = false;
                blended_alpha(gate_q(gt, pq), alpha, clamped);  // blended: the mask already decided
                const float e = alpha * s_io[warp][k];  // the falloff before opacity (unclamped)
                const float4 r1 = make_float4(sf[4][k], sf[5][k], sf[6][k], sf[7][k]);
                const float c2 = sf[8][k];
                const float wgt = __fmul_rn(alpha, T);
                const float n0 = __fmaf_rn(wgt, r1.z, S0), n1 = __fmaf_rn(wgt, r1.w, S1),
                            n2 = __fmaf_rn(wgt, c2, S2);
                const float inv1m = rcp_approx(1.0f - alpha);  // 1 - alpha in [0.01, 1): no denormal range
                const float da0 = T * r1.z - (Cf0 - n0) * inv1m;
                const float da1 = T * r1.w - (Cf1 - n1) * inv1m;
                const float da2 = T * c2 - (Cf2 - n2) * inv1m;
                const float sw2 = W0 * da0 * da0 + W1 * da1 * da1 + W2 * da2 * da2;
                s_t[warp][0][lane][kk] = clamped ? 0.0f : alpha * alpha * sw2;
                s_t[warp][1][lane][kk] = clamped ? 0.0f : e * e * sw2;
                s_t[warp][2][lane][kk] = wgt * wgt;
                S0 = n0;
                S1 = n1;
                S2 = n2;
                T = __fmul_rn(T, __fsub_rn(1.0f, alpha));
            }
            const int k = 16 * h + e16;
            const unsigned colk = __shfl_sync(0xffffffffu, col, k) & pmask;
            __syncwarp();
            const float qmx = sf[0][k], qmy = sf[1][k];
            // sdp-weighted monomials in (dx, dy) up to degree 4, opacity, colours
            // packed FFMA2 / FADD2 / FMUL2 pairs; every lane does the scalar code's
            // operations in the same order (so the sums round identically)
            float2 Pa = make_float2(0.f, 0.f), Pb = Pa, Pc = Pa, Pd = Pa, Pe = Pa, Pf = Pa, Pg = Pa, Ph = Pa;
            for (unsigned cc = colk; cc; cc &= cc - 1) {
                const int p = __ffs(cc) - 1;
                const float4 pi = s_pix[warp][p];
                const float pw2 = s_pw2[warp][p];
                const float sdp = s_t[warp][0][p][e16], so = s_t[warp][1][p][e16], w2 = s_t[warp][2][p][e16];
                const float X = qmx - pi.x, Y = qmy - pi.y;
                const float2 XY2 = make_float2(X, Y);
                const float2 xx_xy = fmul2(make_float2(X, X), XY2);  // (XX, XY)
                const float YY = Y * Y;
                const float2 s_xx_xy = fmul2(make_float2(sdp, sdp), xx_xy);  // (sXX, sXY)
                const float sYY = sdp * YY;
                Pa = fadd2(Pa, s_xx_xy);                                              // (m2x, mxy)
                Pb = fadd2(Pb, make_float2(sYY, so));                                 // (m2y, aop)
                Pc = ffma2(make_float2(s_xx_xy.x, s_xx_xy.x), XY2, Pc);             // (m3x, mx2y)
                Pd = ffma2(make_float2(sYY, sYY), XY2, Pd);                           // (mxy2, m3y)
                Pe = ffma2(make_float2(s_xx_xy.x, s_xx_xy.x), xx_xy, Pe);             // (m4x, mx3y)
                Pf = ffma2(make_float2(s_xx_xy.x, sYY), make_float2(YY, YY), Pf);     // (mx2y2, m4y)
                Pg = ffma2(make_float2(s_xx_xy.y, pw2), make_float2(YY, w2), Pg);   // (mxy3, ac2)
                Ph = ffma2(make_float2(pi.z, pi.w), make_float2(w2, w2), Ph);         // (ac0, ac1)
            }
            float m2x = Pa.x, mxy = Pa.y, m2y = Pb.x, aop = Pb.y, m3x = Pc.x, mx2y = Pc.y, mxy2 = Pd.x, m3y = Pd.y;
            float m4x = Pe.x, mx3y = Pe.y, mx2y2 = Pf.x, m4y = Pf.y, mxy3 = Pg.x, ac2 = Pg.y, ac0 = Ph.x, ac1 = Ph.y;
#define HSUM(v) v += __shfl_xor_sync(0xffffffffu, v, 16)
            HSUM(m2x); HSUM(mxy); HSUM(m2y); HSUM(m3x); HSUM(mx2y); HSUM(mxy2); HSUM(m3y);
            HSUM(m4x); HSUM(mx3y); HSUM(mx2y2); HSUM(mxy3); HSUM(m4y); HSUM(aop);
            HSUM(ac0); HSUM(ac1); HSUM(ac2);
#undef HSUM
            if (ph == 0 && k < nent) {
                const float ca = -2.0f * kLn2f * sf[2][k], cb = -kLn2f * sf[3][k], cc = -2.0f * kLn2f * sf[4][k];
                // M_ij = sum sdp gp_i gp_j, gp = (-(ca X + cb Y), -(cb X + cc Y), -X^2/2, -XY, -Y^2/2)
                const float M00 = ca * ca * m2x + 2.0f * ca * cb * mxy + cb * cb * m2y;
                const float M01 = ca * cb * m2x + (ca * cc + cb * cb) * mxy + cb * cc * m2y;
                const float M11 = cb * cb * m2x + 2.0f * cb * cc * mxy + cc * cc * m2y;
                const float M02 = 0.5f * (ca * m3x + cb * mx2y);
                const float M03 = ca * mx2y + cb * mxy2;
                const float M04 = 0.5f * (ca * mxy2 + cb * m3y);
                const float M12 = 0.5f * (cb * m3x + cc * mx2y);
                const float M13 = cb * mx2y + cc * mxy2;
                const float M14 = 0.5f * (cb * mxy2 + cc * m3y);
                const float M22 = 0.25f * m4x, M23 = 0.5f * mx3y, M24 = 0.25f * mx2y2;
                const float M33 = mx2y2, M34 = 0.5f * mxy3, M44 = 0.25f * m4y;
                // upper-triangle order (00,01,02,03,04,11,12,13,14,22,23,24,33,34,44)
                if (A.partial) {  // deterministic: own record, summed in order by k_diag_finalize
                    float4* dst = reinterpret_cast<float4*>(A.partial) +
                                  (kDetDiagRec / 4) * static_cast<size_t>(A.dest[slot0 + 32 * w + k]);
                    dst[0] = make_float4(M00, M01, M02, M03);
                    dst[1] = make_float4(M04, M11, M12, M13);
                    dst[2] = make_float4(M14, M22, M23, M24);
                    dst[3] = make_float4(M33, M34, M44, aop);
                    dst[4] = make_float4(ac0, ac1, ac2, 0.f);
                    dst[5] = make_float4(0.f, 0.f, 0.f, 0.f);  // full sectors
                } else {
                    float* dst = A.diagacc + (c.vbase + s_g[warp][k]) * kDiagRec;
                    red_add_v4(dst, M00, M01, M02, M03);
                    red_add_v4(dst + 4, M04, M11, M12, M13);
                    red_add_v4(dst + 8, M14, M22, M23, M24);
                    red_add_v4(dst + 12, M33, M34, M44, aop);
                    red_add_v4(dst + 16, ac0, ac1, ac2, 0.f);
                }
            }
            __syncwarp();
        }
    }
}

// ------------------------------------------------------------------ exact render
// render_full's drop-in form (rasterizer.cpp:62-104): blend_pixel replayed in
// FP64 per pixel (the reference's operation order, FP64 geometry from
// k_prepare, colours from the record), one thread per pixel.  Slower than
// k_render; used by slm_render_full so the API returns the reference's
// decisions (contrib, T) exactly.
__global__ void __launch_bounds__(128) k_render_exact(const DevCam* __restrict__ cams, const int* __restrict__ tile_view,
                                                      int n_tiles, const int* __restrict__ tile_offsets,
                                                      const int* __restrict__ entries, const double* __restrict__ rec64,
                                                      const float4* __restrict__ rec, int Gp, double* __restrict__ image,
                                                      double* __restrict__ trans, int* __restrict__ contrib) {
    const int tile = static_cast<int>(blockIdx.x >> 1);  // two 128-pixel halves per tile, tiles on x (no 65535 cap)
    if (tile >= n_tiles) return;
    const int v = tile_view[tile];
    const DevCam& cam = cams[v];
    const int lt = tile - cam.tile_base;
    const int tx = lt % cam.tiles_x, ty = lt / cam.tiles_x;
    const int idx = (blockIdx.x & 1) * blockDim.x + threadIdx.x;  // pixel of the 16x16 tile
    if (idx >= kTile * kTile) return;
    const int x = tx * kTile + idx % kTile, y = ty * kTile + idx / kTile;
    if (x >= cam.width || y >= cam.height) return;
    const double px = x + 0.5, py = y + 0.5;
    const int b = tile_offsets[tile], n = tile_offsets[tile + 1] - b;
    const size_t vbase = static_cast<size_t>(v) * Gp;
    double T = 1.0, C0 = 0.0, C1 = 0.0, C2 = 0.0;
    int cnt = 0;
    for (int k = 0; k < n; ++k) {
        const int g = entries[b + k];
        const double* e = rec64 + 6 * (vbase + g);
        const double dx = __dsub_rn(e[0], px), dy = __dsub_rn(e[1], py);
        const double power =
            __dsub_rn(__dmul_rn(-0.5, __dadd_rn(__dmul_rn(__dmul_rn(e[2], dx), dx), __dmul_rn(__dmul_rn(e[4], dy), dy))),
                      __dmul_rn(__dmul_rn(e[3], dx), dy));
        if (power > 0.0) continue;
        double alpha = __dmul_rn(e[5], exp(power));
        if (alpha > kAlphaClampD) alpha = kAlphaClampD;
        if (alpha < kAlphaSkipD) continue;
        const double test_t = __dmul_rn(T, __dsub_rn(1.0, alpha));
        if (test_t < kTFloorD) break;
        const double w = __dmul_rn(alpha, T);
        const float4* r = rec + 3 * (vbase + g);
        const float4 r1 = r[1];
        C0 = __dadd_rn(C0, __dmul_rn(w, static_cast<double>(r1.z)));
        C1 = __dadd_rn(C1, __dmul_rn(w, static_cast<double>(r1.w)));
        C2 = __dadd_rn(C2, __dmul_rn(w, static_cast<double>(r[2].x)));
        T = test_t;
        ++cnt;
    }
    const size_t pix = cam.pix_base + static_cast<size_t>(y) * cam.width + x;
    image[3 * pix] = C0;
    image[3 * pix + 1] = C1;
    image[3 * pix + 2] = C2;
    trans[pix] = T;
    contrib[pix] = cnt;
}

void launch_render_exact(const DevCam* cams, const int* tile_view, int n_tiles, const int* tile_offsets,
                         const int* entries, const double* rec64, const float4* rec, int Gp, double* image,
                         double* trans, int* contrib, cudaStream_t st) {
    if (n_tiles == 0) return;
    k_render_exact<<<2u * static_cast<unsigned>(n_tiles), 128, 0, st>>>(cams, tile_view, n_tiles, tile_offsets, entries, rec64, rec, Gp,
                                                     image, trans, contrib);
    ++g_launches;
}

// ------------------------------------------------------------------ drop-in render_pixel / render_with_context
// The reference's blend over caller-prepared splats (render::SplatD, 10 doubles
// each: mean2d x, y, conic a, b, c, opacity, colour r, g, b, unused): the
// blend_pixel arithmetic of k_render_exact with f64 colours, so the result is
// the reference's bit for bit up to exp's last ulp.
constexpr int kSplatD = 10;

// false: the pixel terminated (this splat not blended)
__device__ __forceinline__ bool blend_splat_f64(const double* e, double px, double py, double& T, double& C0,
                                                double& C1, double& C2, int& cnt) {
    const double dx = __dsub_rn(e[0], px), dy = __dsub_rn(e[1], py);
    const double power = __dsub_rn(
        __dmul_rn(-0.5, __dadd_rn(__dmul_rn(__dmul_rn(e[2], dx), dx), __dmul_rn(__dmul_rn(e[4], dy), dy))),
        __dmul_rn(__dmul_rn(e[3], dx), dy));
    if (power > 0.0) return true;
    double alpha = __dmul_rn(e[5], exp(power));
    if (alpha > kAlphaClampD) alpha = kAlphaClampD;
    if (alpha < kAlphaSkipD) return true;
    const double test_t = __dmul_rn(T, __dsub_rn(1.0, alpha));
    if (test_t < kTFloorD) return false;
    const double w = __dmul_rn(alpha, T);
    C0 = __dadd_rn(C0, __dmul_rn(w, e[6]));
    C1 = __dadd_rn(C1, __dmul_rn(w, e[7]));
    C2 = __dadd_rn(C2, __dmul_rn(w, e[8]));
    T = test_t;
    ++cnt;
    return true;
}

// render_with_context (rasterizer.cpp:62-91): one thread per pixel, two
// 128-pixel halves per tile on blockIdx.x; lists are CSR over the tiles.
__global__ void __launch_bounds__(128) k_render_splats(int width, int height, int tiles_x, int n_tiles,
                                                       const int* __restrict__ offsets, const int* __restrict__ list,
                                                       const double* __restrict__ splats, double* __restrict__ image,
                                                       double* __restrict__ trans, int* __restrict__ contrib) {
    const int tile = static_cast<int>(blockIdx.x >> 1);
    if (tile >= n_tiles) return;
    const int idx = (blockIdx.x & 1) * blockDim.x + threadIdx.x;
    const int x = (tile % tiles_x) * kTile + idx % kTile, y = (tile / tiles_x) * kTile + idx / kTile;
    if (x >= width || y >= height) return;
    const double px = x + 0.5, py = y + 0.5;
    double T = 1.0, C0 = 0.0, C1 = 0.0, C2 = 0.0;
    int cnt = 0;
    for (int k = offsets[tile]; k < offsets[tile + 1]; ++k)
        if (!blend_splat_f64(splats + static_cast<size_t>(kSplatD) * list[k], px, py, T, C0, C1, C2, cnt)) break;
    const size_t pix = static_cast<size_t>(y) * width + x;
    image[3 * pix] = C0;
    image[3 * pix + 1] = C1;
    image[3 * pix + 2] = C2;
    trans[pix] = T;
    contrib[pix] = cnt;
}

// render_pixel (rasterizer.cpp:52-60): the blend of one pixel over all splats in order.
__global__ void k_render_pixel(int n, const double* __restrict__ splats, double px, double py,
                               double* __restrict__ out, int* __restrict__ contrib) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double T = 1.0, C0 = 0.0, C1 = 0.0, C2 = 0.0;
    int cnt = 0;
    for (int k = 0; k < n; ++k)
        if (!blend_splat_f64(splats + static_cast<size_t>(kSplatD) * k, px, py, T, C0, C1, C2, cnt)) break;
    out[0] = C0;
    out[1] = C1;
    out[2] = C2;
    out[3] = T;
    *contrib = cnt;
}

void launch_render_splats(int width, int height, int tiles_x, int n_tiles, const int* offsets, const int* list,
                          const double* splats, double* image, double* trans, int* contrib, cudaStream_t st) {
    if (n_tiles == 0) return;
    k_render_splats<<<2u * static_cast<unsigned>(n_tiles), 128, 0, st>>>(width, height, tiles_x, n_tiles, offsets, list,
                                                                          splats, image, trans, contrib);
    ++g_launches;
}
void launch_render_pixel(int n, const double* splats, double px, double py, double* out, int* contrib,
                         cudaStream_t st) {
    k_render_pixel<<<1, 32, 0, st>>>(n, splats, px, py, out, contrib);
    ++g_launches;
}

// ------------------------------------------------------------------ launchers
void launch_render(const DevCam* cams, const int* tile_view, int n_tiles, const int* tile_offsets,
                   const int* entries, const float4* rec, int Gp, const float* gt, float* image,
                   float* trans, int* contrib, int* last, double* sse_tile, cudaStream_t st,
                   unsigned long long* stats) {
    if (n_tiles == 0) return;
    if (stats)
        k_render<true, true><<<n_tiles, kRenderThreads, 0, st>>>(cams, tile_view, tile_offsets, entries, rec, Gp, gt,
                                                                 image, trans, contrib, last, sse_tile, stats);
    else if (contrib)
        k_render<false, true><<<n_tiles, kRenderThreads, 0, st>>>(cams, tile_view, tile_offsets, entries, rec, Gp, gt,
                                                                  image, trans, contrib, last, sse_tile, nullptr);
    else  // colour + SSE only (the LM step's loss renders)
        k_render<false, false><<<n_tiles, kRenderThreads, 0, st>>>(cams, tile_view, tile_offsets, entries, rec, Gp,
                                                                   gt, image, nullptr, nullptr, nullptr, sse_tile,
                                                                   nullptr);
    ++g_launches;
}

void launch_sse_views(const DevCam* cams, int V, int n_tiles, const double* sse_tile,
                      double* sse_view, cudaStream_t st) {
    if (V == 0) return;
    k_sse_views<<<V, 32, 0, st>>>(cams, V, n_tiles, sse_tile, sse_view); ++g_launches;
}

void launch_masks(const SampleArgs& a, cudaStream_t st) {
    if (a.n_groups == 0) return;
    k_masks<<<(a.n_groups + 3) / 4, 128, 0, st>>>(a); ++g_launches;
}

void launch_alpha(const SampleArgs& a, cudaStream_t st) {
    if (a.n_groups == 0) return;
    k_alpha<<<(a.n_groups + 3) / 4, 128, 0, st>>>(a); ++g_launches;
}

void launch_sample_raster(int mode, const SampleArgs& a, cudaStream_t st) {
    if (a.n_groups == 0) return;
    const int blocks = (a.n_groups + kRasterWarps - 1) / kRasterWarps;
    switch (mode) {
        case kJvp: k_sample_raster<kJvp><<<blocks, 32 * kRasterWarps, 0, st>>>(a); ++g_launches; break;
        case kVjp: k_sample_raster<kVjp><<<blocks, 32 * kRasterWarps, 0, st>>>(a); ++g_launches; break;
        case kGn: k_sample_raster<kGn><<<blocks, 32 * kRasterWarps, 0, st>>>(a); ++g_launches; break;
        default: k_sample_raster<kRhs><<<blocks, 32 * kRasterWarps, 0, st>>>(a); ++g_launches; break;
    }
}

void launch_diag_raster(const DiagArgs& a, cudaStream_t st) {
    if (a.n_groups == 0) return;
    k_diag_raster<<<(a.n_groups + 3) / 4, 128, 0, st>>>(a); ++g_launches;
}

}  // namespace slm
