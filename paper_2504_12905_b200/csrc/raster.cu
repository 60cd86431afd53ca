// raster.cu — FP32 tile rasterizers.
//
//  * k_render          full-image forward (render_with_context, rasterizer.cpp:62-91),
//                      one CTA per 16x16 tile, splat records staged in smem; writes
//                      RGB, final T, contrib count and `last` (the list position
//                      where blend_pixel stopped) and per-tile SSE vs ground truth.
//  * k_sample_raster   the sampled-pixel passes, one warp per group of <=32 samples
//                      of one tile (lanes = samples, all lanes walk the same entry):
//        JVP   Jv      dual blend (jvp, jacobian.cpp:191-211)
//        VJP   J^T u   reverse blend into the 9-float intermediate (vjp :219-247)
//        GN    J^T W J p fused: Jv, *W, J^T in one kernel (gn_apply :339-344)
//        RHS   J^T(-W r) with r read from the forward render (lm.cpp:99-121)
//  * k_diag_raster     diag(J^T W J) accumulators (jtj_diag :272-337), factored as
//                      a per-(tile,Gaussian) 5x5 quadratic form.
//
// The J^T passes sweep front-to-back: the reference's reverse sweep needs
// suffix_c = sum_{j>k} w_j c_j (backward_pixel_vjp :67-94); with the pixel's
// final colour C from the forward render, suffix = C - prefix_incl(k), and
// prefix is accumulated with the very same FP32 operations as the forward
// render, so the gate decisions and sums replay exactly.
#include <cstdint>

#include <atomic>

#include "common.cuh"

namespace slm { extern std::atomic<long long> g_launches; }

namespace slm {

// ------------------------------------------------------------------ K6
__global__ void __launch_bounds__(256) k_render(
    const DevCam* __restrict__ cams, const int* __restrict__ tile_view,
    const int* __restrict__ tile_offsets, const int* __restrict__ entries,
    const float4* __restrict__ rec, int Gp, const float* __restrict__ gt,
    float* __restrict__ image, float* __restrict__ trans, int* __restrict__ contrib,
    int* __restrict__ last_out, double* __restrict__ sse_tile) {
    __shared__ float4 s_rec[256][3];
    __shared__ double s_red[8];
    const int tile = blockIdx.x;
    const int v = tile_view[tile];
    const DevCam& cam = cams[v];
    const int lt = tile - cam.tile_base;
    const int tx = lt % cam.tiles_x, ty = lt / cam.tiles_x;
    const int x = tx * kTile + (threadIdx.x & 15), y = ty * kTile + (threadIdx.x >> 4);
    const bool inside = x < cam.width && y < cam.height;
    const float pxc = (float)x + 0.5f, pyc = (float)y + 0.5f;
    const int b = tile_offsets[tile], n = tile_offsets[tile + 1] - b;
    const size_t vbase = static_cast<size_t>(v) * Gp;

    float T = 1.0f, C0 = 0.0f, C1 = 0.0f, C2 = 0.0f;
    int cnt = 0, last = n;
    bool done = !inside;
    for (int start = 0; start < n; start += 256) {
        if (__syncthreads_count(done) == 256) break;
        const int j = start + threadIdx.x;
        if (j < n) {
            const float4* r = rec + 3 * (vbase + entries[b + j]);
            s_rec[threadIdx.x][0] = r[0];
            s_rec[threadIdx.x][1] = r[1];
            s_rec[threadIdx.x][2] = r[2];
        }
        __syncthreads();
        const int m = min(256, n - start);
        for (int k = 0; k < m && !done; ++k) {
            const float4 r0 = s_rec[k][0], r1 = s_rec[k][1];
            Alpha a;
            if (!eval_alpha(r0, r1, pxc, pyc, a)) continue;
            float tt;
            if (terminates(T, a.alpha, tt)) {
                done = true;
                last = start + k;
                break;
            }
            const float w = __fmul_rn(a.alpha, T);
            const float c2 = s_rec[k][2].x;
            C0 = __fmaf_rn(w, r1.z, C0);
            C1 = __fmaf_rn(w, r1.w, C1);
            C2 = __fmaf_rn(w, c2, C2);
            T = tt;
            ++cnt;
        }
    }
    double sq = 0.0;
    if (inside) {
        const size_t pix = cam.pix_base + static_cast<size_t>(y) * cam.width + x;
        image[3 * pix] = C0;
        image[3 * pix + 1] = C1;
        image[3 * pix + 2] = C2;
        trans[pix] = T;
        contrib[pix] = cnt;
        last_out[pix] = last;
        if (gt) {
            const float* gp = gt + 3 * pix;
            const double d0 = (double)C0 - (double)gp[0], d1 = (double)C1 - (double)gp[1],
                         d2 = (double)C2 - (double)gp[2];
            sq = d0 * d0 + d1 * d1 + d2 * d2;
        }
    }
    if (sse_tile) {
        sq = warp_sum_d(sq);
        if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = sq;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int i = 0; i < 8; ++i) s += s_red[i];
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

// ------------------------------------------------------------------ sampled passes
// Reduce one 9-float intermediate over the warp and add it to global memory.
__device__ __forceinline__ void warp_accumulate9(const float (&gv)[9], unsigned mask, float* dst,
                                                 int lane) {
    if (__popc(mask) == 1) {
        if ((mask >> lane) & 1u) {
#pragma unroll
            for (int i = 0; i < 9; ++i) atomicAdd(dst + i, gv[i]);
        }
        return;
    }
    float mine = 0.0f;
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        const float s = warp_sum(gv[i]);
        if (lane == i) mine = s;
    }
    if (lane < 9) atomicAdd(dst + lane, mine);
}

template <int MODE>
__global__ void __launch_bounds__(128) k_sample_raster(SampleArgs A) {
    __shared__ float4 s_rec[4][32][3];
    __shared__ float4 s_tan[4][32][3];
    __shared__ int s_g[4][32];
    if (A.done_flag && *A.done_flag) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gi = blockIdx.x * 4 + warp;
    if (gi >= A.n_groups) return;
    const Group grp = A.groups[gi];
    const DevCam& cam = A.cams[grp.view];
    const bool active = lane < grp.count;
    const int s = grp.begin + (active ? lane : 0);
    const int packed = A.spix[s];
    const int px = packed & 0xffff, py = packed >> 16;
    const int orig = A.sorig[s];
    const size_t pix = cam.pix_base + static_cast<size_t>(py) * cam.width + px;
    const int mylast = active ? A.last_img[pix] : 0;
    const int maxlast = __reduce_max_sync(0xffffffffu, mylast);
    const int* list = A.entries + A.tile_offsets[cam.tile_base + grp.tile];
    const size_t vbase = static_cast<size_t>(grp.view) * A.Gp;
    const float pxc = (float)px + 0.5f, pyc = (float)py + 0.5f;
    constexpr float kLn2f = 0.69314718055994530942f;

    float u0 = 0.f, u1 = 0.f, u2 = 0.f;
    if (MODE == kJvp || MODE == kGn) {
        float T = 1.0f, dT = 0.0f, dC0 = 0.f, dC1 = 0.f, dC2 = 0.f;
        for (int base = 0; base < maxlast; base += 32) {
            const int j = base + lane;
            if (j < maxlast) {
                const size_t rg = vbase + list[j];
                const float4* r = A.rec + 3 * rg;
                const float4* t = A.tan + 3 * rg;
                s_rec[warp][lane][0] = r[0];
                s_rec[warp][lane][1] = r[1];
                s_rec[warp][lane][2] = r[2];
                s_tan[warp][lane][0] = t[0];
                s_tan[warp][lane][1] = t[1];
                s_tan[warp][lane][2] = t[2];
            }
            __syncwarp();
            const int m = min(32, maxlast - base);
            for (int k = 0; k < m; ++k) {
                if (base + k >= mylast) continue;
                const float4 r0 = s_rec[warp][k][0], r1 = s_rec[warp][k][1];
                Alpha a;
                if (!eval_alpha(r0, r1, pxc, pyc, a)) continue;
                const float4 t0 = s_tan[warp][k][0], t1 = s_tan[warp][k][1];
                const float4 t2 = s_tan[warp][k][2];
                const float alpha = a.alpha, dx = a.dx, dy = a.dy;
                // natural conic from the log2-scaled record
                const float ca = -2.0f * kLn2f * r0.z, cb = -kLn2f * r0.w, cc = -2.0f * kLn2f * r1.x;
                float dalpha = 0.0f;
                if (!a.clamped) {
                    const float dpow = -(ca * dx + cb * dy) * t0.x - (cb * dx + cc * dy) * t0.y -
                                       0.5f * dx * dx * t0.z - dx * dy * t0.w - 0.5f * dy * dy * t1.x;
                    dalpha = alpha * dpow + (alpha / r1.y) * t1.y;
                }
                const float w = alpha * T;
                const float dw = dalpha * T + alpha * dT;
                dC0 += dw * r1.z + w * t1.z;
                dC1 += dw * r1.w + w * t1.w;
                dC2 += dw * s_rec[warp][k][2].x + w * t2.x;
                const float om = 1.0f - alpha;
                dT = dT * om - T * dalpha;
                T = __fmul_rn(T, __fsub_rn(1.0f, alpha));
            }
            __syncwarp();
        }
        if (MODE == kJvp) {
            if (active) {
                A.out_res[3 * orig] = dC0;
                A.out_res[3 * orig + 1] = dC1;
                A.out_res[3 * orig + 2] = dC2;
            }
            return;
        }
        if (active) {
            u0 = A.sw[3 * s] * dC0;
            u1 = A.sw[3 * s + 1] * dC1;
            u2 = A.sw[3 * s + 2] * dC2;
        }
    } else if (MODE == kVjp) {
        if (active) {
            u0 = A.in_res[3 * orig];
            u1 = A.in_res[3 * orig + 1];
            u2 = A.in_res[3 * orig + 2];
        }
    } else {  // kRhs: u = -w (rendered - truth)
        if (active) {
            const float* gp = A.gt + 3 * pix;
            u0 = -A.sw[3 * s] * (A.image[3 * pix] - gp[0]);
            u1 = -A.sw[3 * s + 1] * (A.image[3 * pix + 1] - gp[1]);
            u2 = -A.sw[3 * s + 2] * (A.image[3 * pix + 2] - gp[2]);
        }
    }

    // ---- J^T pass, front to back with suffix = C - inclusive prefix
    const float Cf0 = active ? A.image[3 * pix] : 0.f;
    const float Cf1 = active ? A.image[3 * pix + 1] : 0.f;
    const float Cf2 = active ? A.image[3 * pix + 2] : 0.f;
    float T = 1.0f, S0 = 0.f, S1 = 0.f, S2 = 0.f;
    for (int base = 0; base < maxlast; base += 32) {
        const int j = base + lane;
        if (j < maxlast) {
            const int g = list[j];
            const float4* r = A.rec + 3 * (vbase + g);
            s_rec[warp][lane][0] = r[0];
            s_rec[warp][lane][1] = r[1];
            s_rec[warp][lane][2] = r[2];
            s_g[warp][lane] = g;
        }
        __syncwarp();
        const int m = min(32, maxlast - base);
        for (int k = 0; k < m; ++k) {
            float gv[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            bool blended = false;
            if (base + k < mylast) {
                const float4 r0 = s_rec[warp][k][0], r1 = s_rec[warp][k][1];
                Alpha a;
                if (eval_alpha(r0, r1, pxc, pyc, a)) {
                    blended = true;
                    const float alpha = a.alpha, dx = a.dx, dy = a.dy;
                    const float c2 = s_rec[warp][k][2].x;
                    const float w = __fmul_rn(alpha, T);
                    const float n0 = __fmaf_rn(w, r1.z, S0), n1 = __fmaf_rn(w, r1.w, S1),
                                n2 = __fmaf_rn(w, c2, S2);
                    const float inv1m = 1.0f / (1.0f - alpha);
                    const float dalpha = u0 * (T * r1.z - (Cf0 - n0) * inv1m) +
                                         u1 * (T * r1.w - (Cf1 - n1) * inv1m) +
                                         u2 * (T * c2 - (Cf2 - n2) * inv1m);
                    gv[6] = u0 * w;
                    gv[7] = u1 * w;
                    gv[8] = u2 * w;
                    if (!a.clamped) {
                        const float ca = -2.0f * kLn2f * r0.z, cb = -kLn2f * r0.w,
                                    cc = -2.0f * kLn2f * r1.x;
                        const float dpow = dalpha * alpha;
                        gv[0] = dpow * -(ca * dx + cb * dy);
                        gv[1] = dpow * -(cb * dx + cc * dy);
                        gv[2] = dpow * (-0.5f * dx * dx);
                        gv[3] = dpow * (-dx * dy);
                        gv[4] = dpow * (-0.5f * dy * dy);
                        gv[5] = dalpha * (alpha / r1.y);
                    }
                    S0 = n0;
                    S1 = n1;
                    S2 = n2;
                    T = __fmul_rn(T, __fsub_rn(1.0f, alpha));
                }
            }
            const unsigned mask = __ballot_sync(0xffffffffu, blended);
            if (mask)
                warp_accumulate9(gv, mask, A.inter + (vbase + s_g[warp][k]) * kRec, lane);
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
__global__ void __launch_bounds__(128) k_diag_raster(DiagArgs A) {
    __shared__ float4 s_rec[4][32][3];
    __shared__ int s_g[4][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gi = blockIdx.x * 4 + warp;
    if (gi >= A.n_groups) return;
    const Group grp = A.groups[gi];
    const DevCam& cam = A.cams[grp.view];
    const bool active = lane < grp.count;
    const int s = grp.begin + (active ? lane : 0);
    const int packed = A.spix[s];
    const int px = packed & 0xffff, py = packed >> 16;
    const size_t pix = cam.pix_base + static_cast<size_t>(py) * cam.width + px;
    const int mylast = active ? A.last_img[pix] : 0;
    const int maxlast = __reduce_max_sync(0xffffffffu, mylast);
    const int* list = A.entries + A.tile_offsets[cam.tile_base + grp.tile];
    const size_t vbase = static_cast<size_t>(grp.view) * A.Gp;
    const float pxc = (float)px + 0.5f, pyc = (float)py + 0.5f;
    const float W0 = active ? A.sw[3 * s] : 0.f, W1 = active ? A.sw[3 * s + 1] : 0.f,
                W2 = active ? A.sw[3 * s + 2] : 0.f;
    const float Cf0 = active ? A.image[3 * pix] : 0.f;
    const float Cf1 = active ? A.image[3 * pix + 1] : 0.f;
    const float Cf2 = active ? A.image[3 * pix + 2] : 0.f;
    constexpr float kLn2f = 0.69314718055994530942f;
    float T = 1.0f, S0 = 0.f, S1 = 0.f, S2 = 0.f;
    for (int base = 0; base < maxlast; base += 32) {
        const int j = base + lane;
        if (j < maxlast) {
            const int g = list[j];
            const float4* r = A.rec + 3 * (vbase + g);
            s_rec[warp][lane][0] = r[0];
            s_rec[warp][lane][1] = r[1];
            s_rec[warp][lane][2] = r[2];
            s_g[warp][lane] = g;
        }
        __syncwarp();
        const int m = min(32, maxlast - base);
        for (int k = 0; k < m; ++k) {
            float acc[19];
#pragma unroll
            for (int i = 0; i < 19; ++i) acc[i] = 0.f;
            bool blended = false;
            if (base + k < mylast) {
                const float4 r0 = s_rec[warp][k][0], r1 = s_rec[warp][k][1];
                Alpha a;
                if (eval_alpha(r0, r1, pxc, pyc, a)) {
                    blended = true;
                    const float alpha = a.alpha, dx = a.dx, dy = a.dy;
                    const float c2 = s_rec[warp][k][2].x;
                    const float w = __fmul_rn(alpha, T);
                    const float n0 = __fmaf_rn(w, r1.z, S0), n1 = __fmaf_rn(w, r1.w, S1),
                                n2 = __fmaf_rn(w, c2, S2);
                    const float inv1m = 1.0f / (1.0f - alpha);
                    const float da0 = T * r1.z - (Cf0 - n0) * inv1m;
                    const float da1 = T * r1.w - (Cf1 - n1) * inv1m;
                    const float da2 = T * c2 - (Cf2 - n2) * inv1m;
                    acc[16] = W0 * w * w;
                    acc[17] = W1 * w * w;
                    acc[18] = W2 * w * w;
                    if (!a.clamped) {
                        const float ca = -2.0f * kLn2f * r0.z, cb = -kLn2f * r0.w,
                                    cc = -2.0f * kLn2f * r1.x;
                        const float gp[5] = {-(ca * dx + cb * dy), -(cb * dx + cc * dy),
                                             -0.5f * dx * dx, -dx * dy, -0.5f * dy * dy};
                        const float a2 = alpha * alpha;
                        const float sdp = a2 * (W0 * da0 * da0 + W1 * da1 * da1 + W2 * da2 * da2);
                        int q = 0;
#pragma unroll
                        for (int i = 0; i < 5; ++i)
#pragma unroll
                            for (int jj = i; jj < 5; ++jj) acc[q++] = sdp * gp[i] * gp[jj];
                        const float ao = alpha / r1.y;
                        acc[15] = ao * ao * (W0 * da0 * da0 + W1 * da1 * da1 + W2 * da2 * da2);
                    }
                    S0 = n0;
                    S1 = n1;
                    S2 = n2;
                    T = __fmul_rn(T, __fsub_rn(1.0f, alpha));
                }
            }
            const unsigned mask = __ballot_sync(0xffffffffu, blended);
            if (mask) {
                float* dst = A.diagacc + (vbase + s_g[warp][k]) * kDiagRec;
                if (__popc(mask) == 1) {
                    if ((mask >> lane) & 1u) {
#pragma unroll
                        for (int i = 0; i < 19; ++i) atomicAdd(dst + i, acc[i]);
                    }
                } else {
                    float mine = 0.f;
#pragma unroll
                    for (int i = 0; i < 19; ++i) {
                        const float sum = warp_sum(acc[i]);
                        if (lane == i) mine = sum;
                    }
                    if (lane < 19) atomicAdd(dst + lane, mine);
                }
            }
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------ launchers
void launch_render(const DevCam* cams, const int* tile_view, int n_tiles, const int* tile_offsets,
                   const int* entries, const float4* rec, int Gp, const float* gt, float* image,
                   float* trans, int* contrib, int* last, double* sse_tile, cudaStream_t st) {
    if (n_tiles == 0) return;
    k_render<<<n_tiles, 256, 0, st>>>(cams, tile_view, tile_offsets, entries, rec, Gp, gt, image,
                                      trans, contrib, last, sse_tile); ++g_launches;
}

void launch_sse_views(const DevCam* cams, int V, int n_tiles, const double* sse_tile,
                      double* sse_view, cudaStream_t st) {
    if (V == 0) return;
    k_sse_views<<<V, 32, 0, st>>>(cams, V, n_tiles, sse_tile, sse_view); ++g_launches;
}

void launch_sample_raster(int mode, const SampleArgs& a, cudaStream_t st) {
    if (a.n_groups == 0) return;
    const int blocks = (a.n_groups + 3) / 4;
    switch (mode) {
        case kJvp: k_sample_raster<kJvp><<<blocks, 128, 0, st>>>(a); ++g_launches; break;
        case kVjp: k_sample_raster<kVjp><<<blocks, 128, 0, st>>>(a); ++g_launches; break;
        case kGn: k_sample_raster<kGn><<<blocks, 128, 0, st>>>(a); ++g_launches; break;
        default: k_sample_raster<kRhs><<<blocks, 128, 0, st>>>(a); ++g_launches; break;
    }
}

void launch_diag_raster(const DiagArgs& a, cudaStream_t st) {
    if (a.n_groups == 0) return;
    k_diag_raster<<<(a.n_groups + 3) / 4, 128, 0, st>>>(a); ++g_launches;
}

}  // namespace slm
