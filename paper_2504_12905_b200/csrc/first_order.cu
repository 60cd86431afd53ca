// first_order.cu — the first-order baselines on the device:
// baselines::full_gradient's residual vector and the Adam / RMSprop /
// SGD-momentum steps (baselines/first_order.cpp:11-122).
//
// full_gradient = J^T u over the exhaustive plan (every pixel of every camera,
// :16-44).  k_exhaustive_residual lays the plan out directly in the raster's
// sample order (tile-major, pixels row-major inside the tile, groups of <= 32)
// and writes u = 2/M (r + w s s') there, so the J^T pass is the same
// k_sample_raster<kVjp> + k_chain the LM path uses.
//
// k_first_order_step: one thread per Gaussian over its 14 rows of the f64 SoA
// state, moments in f64 SoA, every operation in the reference's order with
// explicitly rounded f64 ops (its build is -ffp-contract=off) and the
// bias-correction / decay powers computed on the host with the same pow, so a
// step on a given gradient is bitwise the reference's; then
// renormalize_rotations (types.cpp:62-73) and the f32 mirror.
#include <atomic>

#include "common.cuh"

namespace slm { extern std::atomic<long long> g_launches; }

namespace slm {

namespace {

constexpr int kFillWarps = 4;

__global__ void __launch_bounds__(32 * kFillWarps)
k_exhaustive_residual(const DevCam* __restrict__ cams, int n_tiles, const int* __restrict__ tile_view,
                      const int* __restrict__ tile_sbase, const float* __restrict__ image,
                      const float* __restrict__ gt, const float* __restrict__ sres, const float* __restrict__ sdc,
                      float ssim_weight, float scale, int* __restrict__ spix, float* __restrict__ u) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.x * kFillWarps + warp;
    if (t >= n_tiles) return;
    const DevCam& cam = cams[tile_view[t]];
    const int lt = t - cam.tile_base;
    const int x0 = (lt % cam.tiles_x) * kTile, y0 = (lt / cam.tiles_x) * kTile;
    const int rw = min(kTile, cam.width - x0), rh = min(kTile, cam.height - y0);
    const int m = rw * rh, base = tile_sbase[t];
    for (int k = lane; k < m; k += 32) {
        const int px = x0 + k % rw, py = y0 + k / rw;
        spix[base + k] = px | (py << 16);
        const long long e = 3 * (cam.pix_base + static_cast<long long>(py) * cam.width + px);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            float v = image[e + c] - gt[e + c];
            if (sres) v += ssim_weight * sdc[e + c] * sres[e + c];
            u[3 * (base + k) + c] = scale * v;
        }
    }
}

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// kind 0 Adam (:56-69), 1 RMSprop (:71-80), 2 SGD momentum (:82-90).
__global__ void __launch_bounds__(128)
k_first_order_step(double* __restrict__ beta, float* __restrict__ beta32, double* __restrict__ m1,
                   double* __restrict__ m2, const float* __restrict__ grad32, const double* __restrict__ grad64_aos,
                   int G, int Gp, FirstOrderParams fp) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= G) return;
    double p[kP];
#pragma unroll
    for (int k = 0; k < kP; ++k) {
        const size_t i = static_cast<size_t>(k) * Gp + g;
        const double gj = grad64_aos ? grad64_aos[static_cast<size_t>(g) * kP + k] : static_cast<double>(grad32[i]);
        const double lr = fp.lr[k];
        double pj = beta[i];
        if (fp.kind == 0) {
            const double a = dadd(dmul(fp.b1, m1[i]), dmul(dsub(1.0, fp.b1), gj));
            const double b = dadd(dmul(fp.b2, m2[i]), dmul(dmul(dsub(1.0, fp.b2), gj), gj));
            m1[i] = a;
            m2[i] = b;
            const double mhat = __ddiv_rn(a, fp.c1), vhat = __ddiv_rn(b, fp.c2);
            pj = dsub(pj, __ddiv_rn(dmul(lr, mhat), dadd(__dsqrt_rn(vhat), fp.eps)));
        } else if (fp.kind == 1) {
            const double b = dadd(dmul(fp.b2, m2[i]), dmul(dmul(dsub(1.0, fp.b2), gj), gj));
            m2[i] = b;
            pj = dsub(pj, __ddiv_rn(dmul(lr, gj), dadd(__dsqrt_rn(b), fp.eps)));
        } else {
            const double a = dsub(dmul(fp.b1, m1[i]), dmul(lr, gj));
            m1[i] = a;
            pj = dadd(pj, a);
        }
        p[k] = pj;
    }
    // renormalize_rotations (types.cpp:62-73)
    const double n = __dsqrt_rn(dadd(dadd(dadd(dmul(p[6], p[6]), dmul(p[7], p[7])), dmul(p[8], p[8])), dmul(p[9], p[9])));
    if (n == 0.0) {
        p[6] = 1.0;
        p[7] = p[8] = p[9] = 0.0;
    } else {
#pragma unroll
        for (int k = 6; k < 10; ++k) p[k] = __ddiv_rn(p[k], n);
    }
#pragma unroll
    for (int k = 0; k < kP; ++k) {
        const size_t i = static_cast<size_t>(k) * Gp + g;
        beta[i] = p[k];
        beta32[i] = static_cast<float>(p[k]);
    }
}

}  // namespace

void launch_exhaustive_residual(const DevCam* cams, int n_tiles, const int* tile_view, const int* tile_sbase,
                                const float* image, const float* gt, const float* sres, const float* sdc,
                                float ssim_weight, float scale, int* spix, float* u, cudaStream_t st) {
    if (n_tiles == 0) return;
    k_exhaustive_residual<<<(n_tiles + kFillWarps - 1) / kFillWarps, 32 * kFillWarps, 0, st>>>(
        cams, n_tiles, tile_view, tile_sbase, image, gt, sres, sdc, ssim_weight, scale, spix, u);
    ++g_launches;
}

void launch_first_order_step(double* beta, float* beta32, double* m1, double* m2, const float* grad32,
                             const double* grad64_aos, int G, int Gp, const FirstOrderParams& fp, cudaStream_t st) {
    if (G == 0) return;
    k_first_order_step<<<(G + 127) / 128, 128, 0, st>>>(beta, beta32, m1, m2, grad32, grad64_aos, G, Gp, fp);
    ++g_launches;
}

}  // namespace slm
