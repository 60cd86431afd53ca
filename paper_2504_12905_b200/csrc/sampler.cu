// sampler.cu — the weighted residual distributions of build_sample_plan on
// the device (sampling/sample_plan.cpp:127-165).
//
// kResidual: within each tile a softmax of the mean absolute residual
// |render - truth| over the channels; kGaussianCount: 1 + the per-pixel
// contributor count, normalised.  Draws are with replacement from the tile's
// CDF (draw_from_cdf, :53-58): u = U·cdf.back(), first CDF entry > u.
//
// The host keeps the RNG: it draws the batch's uniforms U in the reference's
// order (view, tile, draw) from the caller's std::mt19937_64 — one
// generate_canonical call per draw, exactly what the reference consumes —
// while the GPU renders; this kernel then builds the densities and CDFs from
// the device-resident FP64 render (k_render_exact: the reference's blend
// decisions and colours, so the densities and CDFs are the reference's) and
// picks the pixels, so no image leaves HBM.
// One warp per tile, the tile's density and CDF in shared memory (2 KB each);
// sums and the CDF run sequentially in pixel order like std::partial_sum.
//
// Output is the sample layout of the raster directly (group order = plan
// order: tile-major, min(N, m) draws per tile): spix = px | py << 16 and the
// per-channel weights (1 / max(q, 1e-12)) / N_total (jacobian.cpp:112-116).
#include <atomic>

#include "common.cuh"

namespace slm { extern std::atomic<long long> g_launches; }

namespace slm {

namespace {

constexpr int kDrawWarps = 4;
constexpr int kTilePix = kTile * kTile;
constexpr double kMinDensity = 1e-12;  // sample_plan.cpp:27

__global__ void __launch_bounds__(32 * kDrawWarps)
k_weighted_draw(const DevCam* __restrict__ cams, int n_tiles, const int* __restrict__ tile_view,
                const int* __restrict__ tile_sbase, const double* __restrict__ image, const float* __restrict__ gt,
                const int* __restrict__ contrib, int dist, int spt, const double* __restrict__ U, double n_total,
                double inv_total, int* __restrict__ spix, float* __restrict__ sw) {
    __shared__ double s_den[kDrawWarps][kTilePix];
    __shared__ double s_cdf[kDrawWarps][kTilePix];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.x * kDrawWarps + warp;
    if (t >= n_tiles) return;
    const int v = tile_view[t];
    const DevCam& cam = cams[v];
    const int lt = t - cam.tile_base;
    const int tx = lt % cam.tiles_x, ty = lt / cam.tiles_x;
    const int x0 = tx * kTile, y0 = ty * kTile;
    const int rw = min(kTile, cam.width - x0), rh = min(kTile, cam.height - y0);
    const int m = rw * rh;
    const int n = min(spt, m);
    double* den = s_den[warp];
    double* cdf = s_cdf[warp];

    // densities (unnormalised)
    double vmax = -1.0;
    for (int i = lane; i < m; i += 32) {
        const long long pix = cam.pix_base + static_cast<long long>(y0 + i / rw) * cam.width + x0 + i % rw;
        double d;
        if (dist == 1) {  // kResidual: mean |residual| over the channels
            double a = 0.0;
            for (int c = 0; c < 3; ++c)
                a += fabs(image[3 * pix + c] - static_cast<double>(gt[3 * pix + c]));
            d = a / 3.0;
            vmax = fmax(vmax, d);
        } else {  // kGaussianCount
            d = 1.0 + contrib[pix];
        }
        den[i] = d;
    }
    if (dist == 1) {
        for (int o = 16; o; o >>= 1) vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
        for (int i = lane; i < m; i += 32) den[i] = exp(den[i] - vmax);
    }
    __syncwarp();
    double sum = 0.0;
    if (lane == 0)
        for (int i = 0; i < m; ++i) sum += den[i];
    sum = __shfl_sync(0xffffffffu, sum, 0);
    for (int i = lane; i < m; i += 32) den[i] /= sum;
    __syncwarp();
    if (lane == 0) {  // std::partial_sum
        double acc = 0.0;
        for (int i = 0; i < m; ++i) cdf[i] = (acc += den[i]);
    }
    __syncwarp();

    const double back = cdf[m - 1];
    const int base = tile_sbase[t];
    const double frac = static_cast<double>(n) / n_total;
    for (int k = lane; k < n; k += 32) {
        const double u = U[base + k] * back;
        int lo = 0, hi = m;  // upper_bound: first cdf[i] > u
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (cdf[mid] > u) hi = mid;
            else lo = mid + 1;
        }
        const int local = min(lo, m - 1);
        spix[base + k] = (x0 + local % rw) | ((y0 + local / rw) << 16);
        const double q = frac * den[local];
        const float w = static_cast<float>((1.0 / fmax(q, kMinDensity)) * inv_total);
        sw[3 * (base + k)] = w;
        sw[3 * (base + k) + 1] = w;
        sw[3 * (base + k) + 2] = w;
    }
}

}  // namespace

void launch_weighted_draw(const DevCam* cams, int n_tiles, const int* tile_view, const int* tile_sbase,
                          const double* image, const float* gt, const int* contrib, int dist, int spt,
                          const double* U, double n_total, double inv_total, int* spix, float* sw,
                          cudaStream_t st) {
    if (n_tiles == 0) return;
    k_weighted_draw<<<(n_tiles + kDrawWarps - 1) / kDrawWarps, 32 * kDrawWarps, 0, st>>>(
        cams, n_tiles, tile_view, tile_sbase, image, gt, contrib, dist, spt, U, n_total, inv_total, spix, sw);
    ++g_launches;
}

}  // namespace slm
