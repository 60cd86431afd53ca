// metrics.cu — image metrics on device: metrics::mse / psnr / ssim and the
// per-view parts of evaluate / evaluate_split (metrics/image_metrics.cpp:14-139,
// 180-186; io/run.cpp:77-92).
//
// One CTA per 32x32 output tile of one image (interleaved RGB, f32 device
// renders or f64 caller images), all three channels in turn.  Per channel the
// CTA stages the 42x42 reflect-padded halo of both images as f64 in shared
// memory, runs the horizontal 11-tap pass of the five SSIM moment planes
// (a, b, a², b², ab) into shared memory and the vertical pass straight into
// the per-pixel SSIM term.  Filter taps and the SSIM formula use the
// reference's operation order with explicitly rounded f64 ops (no FMA
// contraction, like its -ffp-contract=off build), so every per-pixel filtered
// moment and local SSIM value equals the reference's bit for bit; only the
// final sum over pixels runs in a different (fixed, deterministic) order.
// Window weights are computed on the host with the reference's formula
// (gaussian_window, :25-35) and passed by value.
//
// The work is tiny next to the LM step (about 250 f64 flops and 2 input reads
// per pixel and channel); it exists so evaluation of a test split needs no
// image download.
#include <atomic>

#include "common.cuh"

namespace slm { extern std::atomic<long long> g_launches; }

namespace slm {

namespace {

constexpr int kHalf = kMetricWin / 2;                  // image_metrics.cpp:14-15
constexpr int kMT = 32;                                // output tile edge
constexpr int kMH = kMT + 2 * kHalf;                   // halo edge (42)
constexpr int kMetricThreads = 256;
constexpr double kC1 = 0.01 * 0.01, kC2 = 0.03 * 0.03;  // image_metrics.cpp:17-18
constexpr size_t kMetricSmem = sizeof(double) * (2 * kMH * kMH + 5 * kMH * kMT);


// image_metrics.cpp:38-42 (single reflection), clamped so images narrower than
// the window stay in bounds (the reference is undefined there).
__device__ __forceinline__ int reflect_idx(int i, int n) {
    if (i < 0) i = -i - 1;
    if (i >= n) i = 2 * n - i - 1;
    return min(max(i, 0), n - 1);
}

__device__ __forceinline__ double fma_free(double acc, double w, double v) {
    return __dadd_rn(acc, __dmul_rn(w, v));
}

template <typename T>
__global__ void __launch_bounds__(kMetricThreads)
k_image_metrics(const T* __restrict__ a, const T* __restrict__ b, const ImgDesc* __restrict__ imgs,
                double2* __restrict__ partial, const MetricWindow win) {
    extern __shared__ double sm[];
    double* sa = sm;                   // [kMH][kMH]
    double* sb = sa + kMH * kMH;       // [kMH][kMH]
    double* hm = sb + kMH * kMH;       // [5][kMH][kMT]
    __shared__ double red[2][kMetricThreads / 32];

    const ImgDesc d = imgs[blockIdx.y];
    if (static_cast<int>(blockIdx.x) >= d.tiles) return;
    const int tx = blockIdx.x % d.tiles_x, ty = blockIdx.x / d.tiles_x;
    const int x0 = tx * kMT, y0 = ty * kMT;
    const T* pa = a + d.off;
    const T* pb = b + d.off;
    double sse = 0.0, ssim = 0.0;

    for (int c = 0; c < 3; ++c) {
        for (int i = threadIdx.x; i < kMH * kMH; i += kMetricThreads) {
            const int r = i / kMH, q = i - r * kMH;
            const long long px = static_cast<long long>(reflect_idx(y0 - kHalf + r, d.h)) * d.w +
                                 reflect_idx(x0 - kHalf + q, d.w);
            sa[i] = static_cast<double>(pa[3 * px + c]);
            sb[i] = static_cast<double>(pb[3 * px + c]);
        }
        __syncthreads();
        // horizontal pass (image_metrics.cpp:51-57): rows of the halo, tile columns
        for (int i = threadIdx.x; i < kMH * kMT; i += kMetricThreads) {
            const int r = i / kMT, q = i - r * kMT;
            const double* ra = sa + r * kMH + q;
            const double* rb = sb + r * kMH + q;
            double m0 = 0.0, m1 = 0.0, m2 = 0.0, m3 = 0.0, m4 = 0.0;
#pragma unroll
            for (int t = 0; t < kMetricWin; ++t) {
                const double w = win.w[t], va = ra[t], vb = rb[t];
                m0 = fma_free(m0, w, va);
                m1 = fma_free(m1, w, vb);
                m2 = fma_free(m2, w, __dmul_rn(va, va));
                m3 = fma_free(m3, w, __dmul_rn(vb, vb));
                m4 = fma_free(m4, w, __dmul_rn(va, vb));
            }
            hm[0 * kMH * kMT + i] = m0;
            hm[1 * kMH * kMT + i] = m1;
            hm[2 * kMH * kMT + i] = m2;
            hm[3 * kMH * kMT + i] = m3;
            hm[4 * kMH * kMT + i] = m4;
        }
        __syncthreads();
        // vertical pass (:58-65) + local SSIM (:127-135) + squared error
        for (int i = threadIdx.x; i < kMT * kMT; i += kMetricThreads) {
            const int r = i / kMT, q = i - r * kMT;
            if (y0 + r >= d.h || x0 + q >= d.w) continue;
            double mu_a = 0.0, mu_b = 0.0, e_aa = 0.0, e_bb = 0.0, e_ab = 0.0;
#pragma unroll
            for (int t = 0; t < kMetricWin; ++t) {
                const int o = (r + t) * kMT + q;
                const double w = win.w[t];
                mu_a = fma_free(mu_a, w, hm[0 * kMH * kMT + o]);
                mu_b = fma_free(mu_b, w, hm[1 * kMH * kMT + o]);
                e_aa = fma_free(e_aa, w, hm[2 * kMH * kMT + o]);
                e_bb = fma_free(e_bb, w, hm[3 * kMH * kMT + o]);
                e_ab = fma_free(e_ab, w, hm[4 * kMH * kMT + o]);
            }
            const double var_a = __dsub_rn(e_aa, __dmul_rn(mu_a, mu_a));
            const double var_b = __dsub_rn(e_bb, __dmul_rn(mu_b, mu_b));
            const double cov = __dsub_rn(e_ab, __dmul_rn(mu_a, mu_b));
            const double num = __dmul_rn(__dadd_rn(__dmul_rn(__dmul_rn(2.0, mu_a), mu_b), kC1),
                                         __dadd_rn(__dmul_rn(2.0, cov), kC2));
            const double den =
                __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(mu_a, mu_a), __dmul_rn(mu_b, mu_b)), kC1),
                          __dadd_rn(__dadd_rn(var_a, var_b), kC2));
            ssim += __ddiv_rn(num, den);
            const int ctr = (r + kHalf) * kMH + q + kHalf;
            const double e = sa[ctr] - sb[ctr];
            sse += e * e;
        }
        __syncthreads();
    }
    sse = warp_sum_d(sse);
    ssim = warp_sum_d(ssim);
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[0][w] = sse;
        red[1][w] = ssim;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s0 = 0.0, s1 = 0.0;
        for (int i = 0; i < kMetricThreads / 32; ++i) {
            s0 += red[0][i];
            s1 += red[1][i];
        }
        partial[d.tile_base + blockIdx.x] = make_double2(s0, s1);
    }
}

// Per image: the tile partials summed in a fixed order -> {sse, sum of local SSIM}.
__global__ void __launch_bounds__(kMetricThreads)
k_metrics_reduce(const ImgDesc* __restrict__ imgs, const double2* __restrict__ partial, double2* __restrict__ out) {
    __shared__ double red[2][kMetricThreads / 32];
    const ImgDesc d = imgs[blockIdx.x];
    double s0 = 0.0, s1 = 0.0;
    for (int t = threadIdx.x; t < d.tiles; t += kMetricThreads) {
        const double2 v = partial[d.tile_base + t];
        s0 += v.x;
        s1 += v.y;
    }
    s0 = warp_sum_d(s0);
    s1 = warp_sum_d(s1);
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[0][w] = s0;
        red[1][w] = s1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t0 = 0.0, t1 = 0.0;
        for (int i = 0; i < kMetricThreads / 32; ++i) {
            t0 += red[0][i];
            t1 += red[1][i];
        }
        out[blockIdx.x] = make_double2(t0, t1);
    }
}

template <typename T>
void launch_metrics_impl(const T* a, const T* b, const ImgDesc* imgs, int n_img, int max_tiles,
                         double2* partial, double2* out, const MetricWindow& win, cudaStream_t st) {
    if (n_img == 0) return;
    if (max_tiles > 0) {
        cudaFuncSetAttribute(k_image_metrics<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kMetricSmem));
        k_image_metrics<T><<<dim3(max_tiles, n_img), kMetricThreads, kMetricSmem, st>>>(a, b, imgs, partial, win);
        ++g_launches;
    }
    k_metrics_reduce<<<n_img, kMetricThreads, 0, st>>>(imgs, partial, out);
    ++g_launches;
}

}  // namespace

int metric_tiles(int w, int h, int* tiles_x) {
    *tiles_x = (w + kMT - 1) / kMT;
    return *tiles_x * ((h + kMT - 1) / kMT);
}

void launch_image_metrics(const float* a, const float* b, const ImgDesc* imgs, int n_img, int max_tiles,
                          double2* partial, double2* out, const MetricWindow& win, cudaStream_t st) {
    launch_metrics_impl(a, b, imgs, n_img, max_tiles, partial, out, win, st);
}

void launch_image_metrics(const double* a, const double* b, const ImgDesc* imgs, int n_img, int max_tiles,
                          double2* partial, double2* out, const MetricWindow& win, cudaStream_t st) {
    launch_metrics_impl(a, b, imgs, n_img, max_tiles, partial, out, win, st);
}

}  // namespace slm
