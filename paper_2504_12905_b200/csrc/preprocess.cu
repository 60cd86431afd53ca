// preprocess.cu — per-(view, Gaussian) FP64 preparation, tile binning and the
// per-tile depth sort (SURVEY §2.2 kernels K1, K3, K4, K5), plus the FP64
// parameter update.
//
// This translation unit is compiled with -fmad=false: every double operation
// below is evaluated in the reference's order without FMA contraction, like
// the reference build's -ffp-contract=off (proj/src/CMakeLists.txt:23-25), so
// depth keys are bit-identical to the reference and tile lists/sort order
// match bit for bit (the north-star "bit-exact" row).
#include <cstdint>

#include <atomic>

#include "common.cuh"

namespace slm { extern std::atomic<long long> g_launches; }

namespace slm {

// ------------------------------------------------------------------ K1
// prepare_splat<double> (rasterizer.hpp:58-94) over covariance_3d /
// quat_to_rotation / project_gaussian (geometry.hpp:21-108), value path only.
struct Prepared {
    double mx, my, ca, cb, cc, o, col[3], cov[3], depth, radius;
    bool valid;
    bool zero_quat;
};

__device__ __forceinline__ double sym2_max_eig(double a, double b, double c) {  // vecmath.hpp:91-96
    const double mid = 0.5 * (a + c);
    const double det = a * c - b * b;
    const double v = mid * mid - det;
    const double disc = sqrt(v > 0.0 ? v : 0.0);
    return mid + disc;
}

// View-independent part (quat_to_rotation, covariance_3d, sigmoid, colour):
// computed once per Gaussian, exactly the operations of the per-view path.
struct GaussCommon {
    double mu[3], sig[9], o, col[3];
    bool zero_quat;
};

__device__ GaussCommon prepare_common(const double* __restrict__ beta, int Gp, int g) {
    GaussCommon gc;
    gc.zero_quat = false;
    for (int k = 0; k < 3; ++k) gc.mu[k] = beta[k * Gp + g];
    const double ls[3] = {beta[3 * Gp + g], beta[4 * Gp + g], beta[5 * Gp + g]};
    const double q[4] = {beta[6 * Gp + g], beta[7 * Gp + g], beta[8 * Gp + g], beta[9 * Gp + g]};
    const double logit = beta[10 * Gp + g];
    gc.o = 1.0 / (1.0 + exp(-logit));  // dual.hpp:74
    for (int k = 0; k < 3; ++k) {
        const double raw = 0.5 + kColorC0 * beta[(11 + k) * Gp + g];
        gc.col[k] = raw > 0.0 ? raw : 0.0;
    }
    // quat_to_rotation (geometry.hpp:21-39)
    const double nsq = q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3];
    if (nsq == 0.0) {
        gc.zero_quat = true;
        return gc;
    }
    const double inv = 1.0 / sqrt(nsq);
    const double w = q[0] * inv, x = q[1] * inv, y = q[2] * inv, z = q[3] * inv;
    double r[9];
    r[0] = 1.0 - 2.0 * (y * y + z * z);
    r[1] = 2.0 * (x * y - w * z);
    r[2] = 2.0 * (x * z + w * y);
    r[3] = 2.0 * (x * y + w * z);
    r[4] = 1.0 - 2.0 * (x * x + z * z);
    r[5] = 2.0 * (y * z - w * x);
    r[6] = 2.0 * (x * z - w * y);
    r[7] = 2.0 * (y * z + w * x);
    r[8] = 1.0 - 2.0 * (x * x + y * y);
    // covariance_3d (geometry.hpp:43-57)
    const double s[3] = {exp(ls[0]), exp(ls[1]), exp(ls[2])};
    double m[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) m[3 * i + j] = r[3 * i + j] * s[j];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            gc.sig[3 * i + j] = m[3 * i] * m[3 * j] + m[3 * i + 1] * m[3 * j + 1] + m[3 * i + 2] * m[3 * j + 2];
    return gc;
}

__device__ Prepared prepare_view(const GaussCommon& gc, const DevCam& cam) {
    Prepared out;
    out.valid = false;
    out.zero_quat = gc.zero_quat;
    out.radius = 0.0;
    out.depth = 0.0;
    if (gc.zero_quat) return out;
    const double* mu = gc.mu;
    const double* sig = gc.sig;
    // project_gaussian (geometry.hpp:71-108)
    const double* W = cam.R;
    const double tx = W[0] * mu[0] + W[1] * mu[1] + W[2] * mu[2] + cam.t[0];
    const double ty = W[3] * mu[0] + W[4] * mu[1] + W[5] * mu[2] + cam.t[1];
    const double tz = W[6] * mu[0] + W[7] * mu[1] + W[8] * mu[2] + cam.t[2];
    out.depth = tz;
    if (tz <= cam.near_clip) return out;
    const double iz = 1.0 / tz;
    out.mx = cam.fx * tx * iz + cam.cx;
    out.my = cam.fy * ty * iz + cam.cy;
    const double iz2 = iz * iz;
    const double j00 = cam.fx * iz, j02 = -cam.fx * tx * iz2;
    const double j11 = cam.fy * iz, j12 = -cam.fy * ty * iz2;
    const double r0[3] = {j00 * W[0] + j02 * W[6], j00 * W[1] + j02 * W[7], j00 * W[2] + j02 * W[8]};
    const double r1[3] = {j11 * W[3] + j12 * W[6], j11 * W[4] + j12 * W[7], j11 * W[5] + j12 * W[8]};
    double s0[3], s1[3];
    for (int i = 0; i < 3; ++i) {
        s0[i] = sig[3 * i] * r0[0] + sig[3 * i + 1] * r0[1] + sig[3 * i + 2] * r0[2];
        s1[i] = sig[3 * i] * r1[0] + sig[3 * i + 1] * r1[1] + sig[3 * i + 2] * r1[2];
    }
    const double a = r0[0] * s0[0] + r0[1] * s0[1] + r0[2] * s0[2] + 0.3;
    const double b = r0[0] * s1[0] + r0[1] * s1[1] + r0[2] * s1[2];
    const double c = r1[0] * s1[0] + r1[1] * s1[1] + r1[2] * s1[2] + 0.3;
    const double cull_r = 3.0 * sqrt(sym2_max_eig(a, b, c));
    if (out.mx + cull_r < 0.0 || out.mx - cull_r > cam.width || out.my + cull_r < 0.0 ||
        out.my - cull_r > cam.height)
        return out;
    out.cov[0] = a;
    out.cov[1] = b;
    out.cov[2] = c;
    // prepare_splat proper (rasterizer.hpp:72-93)
    const double det = a * c - b * b;
    if (!(det > 0.0)) return out;
    const double inv_det = 1.0 / det;
    out.ca = c * inv_det;
    out.cb = -b * inv_det;
    out.cc = a * inv_det;
    out.o = gc.o;
    for (int k = 0; k < 3; ++k) out.col[k] = gc.col[k];
    if (out.o <= kAlphaSkipD) return out;
    const double lam = sym2_max_eig(a, b, c);
    out.radius = sqrt(2.0 * log(255.0 * out.o) * lam) * (1.0 + 1e-6) + 1e-6;
    out.valid = true;
    return out;
}

// Orderable 64-bit key of a double (reference compares depths with < and
// breaks ties by index, rasterizer.cpp:44-47; +0 and -0 compare equal).
__device__ __forceinline__ unsigned long long depth_key(double d) {
    if (d == 0.0) d = 0.0;
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(d));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// One thread per Gaussian, looping over the views: the view-independent FP64
// work (rotation, covariance, sigmoid) is done once per Gaussian.
__global__ void __launch_bounds__(128) k_prepare(const double* __restrict__ beta, int G, int Gp,
                                                 const DevCam* __restrict__ cams, int V, float4* __restrict__ rec,
                                                 unsigned long long* __restrict__ keys, short4* __restrict__ rect,
                                                 unsigned long long* __restrict__ n_entries, int* __restrict__ err,
                                                 double* __restrict__ rec64, float4* __restrict__ conic) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long area = 0ull;  // this Gaussian's tile-list entries over the views
    if (g < G) {
    const GaussCommon gc = prepare_common(beta, Gp, g);
    if (gc.zero_quat) atomicOr(err, 1);
    for (int v = 0; v < V; ++v) {
        const DevCam& cam = cams[v];
        const Prepared p = prepare_view(gc, cam);
        const size_t vg = static_cast<size_t>(v) * Gp + g;
        {  // err[1 + v] = G_v, the valid (view, Gaussian) count (warp-aggregated)
            const unsigned am = __activemask();
            const unsigned vm = __ballot_sync(am, p.valid);
            if (vm && (threadIdx.x & 31) == __ffs(am) - 1) atomicAdd(&err[1 + v], __popc(vm));
        }
        keys[vg] = depth_key(p.depth);
        float4* R = rec + 3 * vg;
        if (rec64) {  // FP64 geometry for the exact blend decisions (k_masks); null: render-only batch
            double* R64 = rec64 + 6 * vg;
            R64[0] = p.valid ? p.mx : 0.0;
            R64[1] = p.valid ? p.my : 0.0;
            R64[2] = p.valid ? p.ca : 0.0;
            R64[3] = p.valid ? p.cb : 0.0;
            R64[4] = p.valid ? p.cc : 0.0;
            R64[5] = p.valid ? p.o : 0.0;
        }
        if (!p.valid) {
            if (conic) conic[vg] = make_float4(0.f, 0.f, 0.f, 0.f);
            R[0] = make_float4(0.f, 0.f, 0.f, 0.f);
            R[1] = make_float4(0.f, 0.f, 0.f, 0.f);
            R[2] = make_float4(0.f, 0.f, 0.f, 0.f);
            rect[vg] = make_short4(1, 0, 1, 0);
            continue;
        }
        R[0] = make_float4((float)p.mx, (float)p.my, (float)(-0.5 * p.ca * kLog2e), (float)(-p.cb * kLog2e));
        R[1] = make_float4((float)(-0.5 * p.cc * kLog2e), (float)p.o, (float)p.col[0], (float)p.col[1]);
        R[2] = make_float4((float)p.col[2], 1.0f, 0.f, 0.f);  // .y = valid marker
        if (conic) conic[vg] = make_float4(R[0].z, R[0].w, R[1].x, R[1].y);  // the linearisation kernels' 16-B view
        // tile rect (rasterizer.cpp:29-36)
        int x0 = (int)floor((p.mx - p.radius) / kTile);
        int x1 = (int)floor((p.mx + p.radius) / kTile);
        int y0 = (int)floor((p.my - p.radius) / kTile);
        int y1 = (int)floor((p.my + p.radius) / kTile);
        x0 = x0 < 0 ? 0 : x0;
        y0 = y0 < 0 ? 0 : y0;
        x1 = x1 > cam.tiles_x - 1 ? cam.tiles_x - 1 : x1;
        y1 = y1 > cam.tiles_y - 1 ? cam.tiles_y - 1 : y1;
        rect[vg] = make_short4((short)x0, (short)x1, (short)y0, (short)y1);
        if (x0 <= x1 && y0 <= y1) area += static_cast<unsigned long long>(x1 - x0 + 1) * (y1 - y0 + 1);
    }
    }
    // n_entries += sum of the block's areas (one atomic per warp)
    for (int o = 16; o; o >>= 1) area += __shfl_xor_sync(0xffffffffu, area, o);
    if ((threadIdx.x & 31) == 0 && area) atomicAdd(n_entries, area);
}

__global__ void k_apply_update(double* __restrict__ beta, const float* __restrict__ delta, int G,
                               int Gp, double eta, float* __restrict__ beta32) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= G) return;
    double b[kP];
    for (int k = 0; k < kP; ++k) b[k] = beta[k * Gp + g] + eta * (double)delta[k * Gp + g];
    const double n = sqrt(b[6] * b[6] + b[7] * b[7] + b[8] * b[8] + b[9] * b[9]);
    if (n == 0.0) {
        b[6] = 1.0;
        b[7] = b[8] = b[9] = 0.0;
    } else {
        for (int k = 6; k < 10; ++k) b[k] /= n;
    }
    for (int k = 0; k < kP; ++k) {
        beta[k * Gp + g] = b[k];
        beta32[k * Gp + g] = (float)b[k];
    }
}

// f64 update from a host-precision (f64) delta, used by the drop-in
// GaussianSet::apply_update entry point.
__global__ void k_apply_update_f64(double* __restrict__ beta, const double* __restrict__ delta_aos,
                                   int G, int Gp, double eta, float* __restrict__ beta32) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= G) return;
    double b[kP];
    for (int k = 0; k < kP; ++k) b[k] = beta[k * Gp + g] + eta * delta_aos[static_cast<size_t>(kP) * g + k];
    const double n = sqrt(b[6] * b[6] + b[7] * b[7] + b[8] * b[8] + b[9] * b[9]);
    if (n == 0.0) {
        b[6] = 1.0;
        b[7] = b[8] = b[9] = 0.0;
    } else {
        for (int k = 6; k < 10; ++k) b[k] /= n;
    }
    for (int k = 0; k < kP; ++k) {
        beta[k * Gp + g] = b[k];
        beta32[k * Gp + g] = (float)b[k];
    }
}

__global__ void k_beta_mirror(const double* __restrict__ beta, float* __restrict__ beta32, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) beta32[i] = (float)beta[i];
}

// ------------------------------------------------------------------ host launchers
void launch_prepare(const double* beta, int G, int Gp, const DevCam* cams, int V, float4* rec,
                    unsigned long long* keys, short4* rect, unsigned long long* n_entries, int* err,
                    double* rec64, float4* conic, cudaStream_t st) {
    if (G == 0 || V == 0) return;
    k_prepare<<<(G + 127) / 128, 128, 0, st>>>(beta, G, Gp, cams, V, rec, keys, rect, n_entries, err, rec64, conic);
    ++g_launches;
}


void launch_apply_update(double* beta, const float* delta, int G, int Gp, double eta,
                         float* beta32, cudaStream_t st) {
    if (G == 0) return;
    k_apply_update<<<(G + 255) / 256, 256, 0, st>>>(beta, delta, G, Gp, eta, beta32); ++g_launches;
}

void launch_apply_update_f64(double* beta, const double* delta_aos, int G, int Gp, double eta,
                             float* beta32, cudaStream_t st) {
    if (G == 0) return;
    k_apply_update_f64<<<(G + 255) / 256, 256, 0, st>>>(beta, delta_aos, G, Gp, eta, beta32); ++g_launches;
}

void launch_beta_mirror(const double* beta, float* beta32, int n, cudaStream_t st) {
    if (n == 0) return;
    k_beta_mirror<<<(n + 255) / 256, 256, 0, st>>>(beta, beta32, n); ++g_launches;
}

}  // namespace slm
