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
// The same kernel in diag mode is metrics::ssim_diag_residuals (:141-178):
// per pixel and channel s = sqrt(max(0, 1 - local SSIM)) and its derivative
// with respect to the centre pixel (diagonal approximation, effective centre
// weights :69-78), written as planes, with sum(s^2) per image for the
// mse+ssim loss.  k_ssim_fold then folds the diagonal SSIM rows into the
// sampled rhs and per-channel weights of lm_step (lm.cpp:86-119).
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

// effective_center_weights (image_metrics.cpp:69-78): the window weight a
// pixel contributes to its own window, reflect padding included (the
// unclamped reflection: only compared, never dereferenced).
__device__ __forceinline__ double center_weight(int i, int n, const MetricWindow& win) {
    double s = 0.0;
#pragma unroll
    for (int k = -kHalf; k <= kHalf; ++k) {
        int j = i + k;
        if (j < 0) j = -j - 1;
        if (j >= n) j = 2 * n - j - 1;
        if (j == i) s = __dadd_rn(s, win.w[k + kHalf]);
    }
    return s;
}

__device__ __forceinline__ double fma_free(double acc, double w, double v) {
    return __dadd_rn(acc, __dmul_rn(w, v));
}

// DIAG = false: partial = {sse, sum of local SSIM}; DIAG = true: partial =
// {sse, sum of s^2} and, when res/dcen are given, the residual planes.
template <typename T, typename O, bool DIAG>
__global__ void __launch_bounds__(kMetricThreads)
k_image_metrics(const T* __restrict__ a, const T* __restrict__ b, const ImgDesc* __restrict__ imgs,
                double2* __restrict__ partial, const MetricWindow win, O* __restrict__ res,
                O* __restrict__ dcen) {
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
            const double a1 = __dadd_rn(__dmul_rn(__dmul_rn(2.0, mu_a), mu_b), kC1);
            const double a2 = __dadd_rn(__dmul_rn(2.0, cov), kC2);
            const double b1 = __dadd_rn(__dadd_rn(__dmul_rn(mu_a, mu_a), __dmul_rn(mu_b, mu_b)), kC1);
            const double b2 = __dadd_rn(__dadd_rn(var_a, var_b), kC2);
            const double local = __ddiv_rn(__dmul_rn(a1, a2), __dmul_rn(b1, b2));
            const int ctr = (r + kHalf) * kMH + q + kHalf;
            const double av = sa[ctr], bv = sb[ctr];
            const double e = av - bv;
            sse += e * e;
            if (!DIAG) {
                ssim += local;
                continue;
            }
            // ssim_diag_residuals (:158-175)
            const double om = __dsub_rn(1.0, local);
            const double sval = __dsqrt_rn(0.0 < om ? om : 0.0);
            ssim += sval * sval;
            if (res == nullptr) continue;
            double dc = 0.0;
            if (!(sval < 1e-12)) {
                const double wc = __dmul_rn(center_weight(x0 + q, d.w, win), center_weight(y0 + r, d.h, win));
                const double dnum = __dadd_rn(__dmul_rn(mu_b, a2), __dmul_rn(a1, __dsub_rn(bv, mu_b)));
                const double dden = __dadd_rn(__dmul_rn(mu_a, b2), __dmul_rn(b1, __dsub_rn(av, mu_a)));
                const double t = __dsub_rn(__dmul_rn(__dmul_rn(dnum, b1), b2), __dmul_rn(__dmul_rn(a1, a2), dden));
                const double dlocal = __ddiv_rn(__dmul_rn(__dmul_rn(2.0, wc), t),
                                                __dmul_rn(__dmul_rn(__dmul_rn(b1, b2), b1), b2));
                dc = __ddiv_rn(-dlocal, __dmul_rn(2.0, sval));
            }
            const long long o = d.off + 3 * (static_cast<long long>(y0 + r) * d.w + x0 + q) + c;
            res[o] = static_cast<O>(sval);
            dcen[o] = static_cast<O>(dc);
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

template <typename T, typename O, bool DIAG>
void launch_metrics_impl(const T* a, const T* b, const ImgDesc* imgs, int n_img, int max_tiles,
                         double2* partial, double2* out, const MetricWindow& win, O* res, O* dcen,
                         cudaStream_t st) {
    if (n_img == 0) return;
    if (max_tiles > 0) {
        auto* k = k_image_metrics<T, O, DIAG>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kMetricSmem));
        k<<<dim3(max_tiles, n_img), kMetricThreads, kMetricSmem, st>>>(a, b, imgs, partial, win, res, dcen);
        ++g_launches;
    }
    k_metrics_reduce<<<n_img, kMetricThreads, 0, st>>>(imgs, partial, out);
    ++g_launches;
}

// lm.cpp:99-119 on the device, one thread per sample (group order): the rhs
// u = -w (r + ssim_weight sp sv) in plan order for the J^T pass, then the
// per-channel weights w (1 + ssim_weight sp^2) in place for diag / products.
__global__ void k_ssim_fold(const Group* __restrict__ groups, int n_groups, const DevCam* __restrict__ cams,
                            const int* __restrict__ spix, const int* __restrict__ sorig, float* __restrict__ sw,
                            const float* __restrict__ image, const float* __restrict__ gt,
                            const float* __restrict__ sres, const float* __restrict__ sdc, float ssim_weight,
                            float* __restrict__ rhs, const float* __restrict__ scol) {
    const int g = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (g >= n_groups) return;
    const Group gr = groups[g];
    if (lane >= gr.count) return;
    const int k = gr.begin + lane;
    const DevCam& cam = cams[gr.view];
    const int p = spix[k];
    const long long pix = cam.pix_base + static_cast<long long>(p >> 16) * cam.width + (p & 0xffff);
    const int o = sorig[k];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const long long e = 3 * pix + c;
        const float w = sw[3 * k + c], sp = sdc[e];
        const float rendered = scol ? scol[3 * k + c] : image[e];  // C_final of the FP64 blend at the sample
        rhs[3 * o + c] = -w * ((rendered - gt[e]) + ssim_weight * sp * sres[e]);
        sw[3 * k + c] = w * (1.0f + ssim_weight * sp * sp);
    }
}

}  // namespace

int metric_tiles(int w, int h, int* tiles_x) {
    *tiles_x = (w + kMT - 1) / kMT;
    return *tiles_x * ((h + kMT - 1) / kMT);
}

void launch_image_metrics(const float* a, const float* b, const ImgDesc* imgs, int n_img, int max_tiles,
                          double2* partial, double2* out, const MetricWindow& win, cudaStream_t st) {
    launch_metrics_impl<float, float, false>(a, b, imgs, n_img, max_tiles, partial, out, win, nullptr, nullptr, st);
}

void launch_image_metrics(const double* a, const double* b, const ImgDesc* imgs, int n_img, int max_tiles,
                          double2* partial, double2* out, const MetricWindow& win, cudaStream_t st) {
    launch_metrics_impl<double, double, false>(a, b, imgs, n_img, max_tiles, partial, out, win, nullptr, nullptr,
                                               st);
}

void launch_ssim_diag(const float* a, const float* b, const ImgDesc* imgs, int n_img, int max_tiles,
                      double2* partial, double2* out, const MetricWindow& win, float* res, float* dcen,
                      cudaStream_t st) {
    launch_metrics_impl<float, float, true>(a, b, imgs, n_img, max_tiles, partial, out, win, res, dcen, st);
}

void launch_ssim_diag(const double* a, const double* b, const ImgDesc* imgs, int n_img, int max_tiles,
                      double2* partial, double2* out, const MetricWindow& win, double* res, double* dcen,
                      cudaStream_t st) {
    launch_metrics_impl<double, double, true>(a, b, imgs, n_img, max_tiles, partial, out, win, res, dcen, st);
}

void launch_ssim_fold(const Group* groups, int n_groups, const DevCam* cams, const int* spix, const int* sorig,
                      float* sw, const float* image, const float* gt, const float* sres, const float* sdc,
                      float ssim_weight, float* rhs, const float* scol, cudaStream_t st) {
    if (n_groups == 0) return;
    k_ssim_fold<<<(n_groups + 3) / 4, 128, 0, st>>>(groups, n_groups, cams, spix, sorig, sw, image, gt, sres, sdc,
                                                     ssim_weight, rhs, scol);
    ++g_launches;
}

}  // namespace slm
