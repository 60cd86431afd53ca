// cg.cu — device-resident Jacobi PCG (pcg_solve, solver/pcg.cpp:10-53) and the
// flat-vector kernels it needs (SURVEY §2.2 K14, K15 lr), plus AoS<->SoA
// conversions at the API edge.
//
// Vectors are f32 SoA [14][Gp] (P = 14*Gp, float4-aligned); every reduction
// accumulates in f64 over a fixed grid and is finished by one CTA summing the
// per-block partials in order, so results are run-to-run deterministic.  The
// CG scalars live in device memory (CgState) and control flow (breakdown,
// early exit) is decided on the device (a `done` flag every later kernel of the
// loop checks), so the loop needs no host round trip.  It is launched as plain
// stream work: at configs[2] one product is ~2 ms against ~3 us per launch, so
// graph capture would buy nothing there.
#include <cstdint>

#include <atomic>

#include "common.cuh"

namespace slm { extern std::atomic<long long> g_launches; }

namespace slm {

__device__ __forceinline__ double block_sum(double v, double* sh) {
    v = warp_sum_d(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sh[i];
    __syncthreads();
    return s;
}

// ---------------------------------------------------------------- conversions
// host ParamVector AoS (f64, stride 14) -> device SoA f32
__global__ void k_aos64_to_soa32(const double* __restrict__ aos, int G, int Gp, float* __restrict__ soa) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= G * kP) return;
    const int g = i / kP, k = i - g * kP;
    soa[k * Gp + g] = (float)aos[i];
}
__global__ void k_soa32_to_aos64(const float* __restrict__ soa, int G, int Gp, double* __restrict__ aos) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= G * kP) return;
    const int g = i / kP, k = i - g * kP;
    aos[i] = (double)soa[k * Gp + g];
}
// f64 AoS (14 per Gaussian, the reference's ParamVector) <-> f32 SoA [14][Gp] over
// Gaussians [g0, g1): the chunked host-vector product (Jacobian::gn_apply)
__global__ void k_aos64_to_soa32_range(const double* __restrict__ aos, int g0, int g1, int Gp, float* __restrict__ soa) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x + static_cast<long long>(g0) * kP;
    if (i >= static_cast<long long>(g1) * kP) return;
    const int g = static_cast<int>(i / kP), k = static_cast<int>(i - static_cast<long long>(g) * kP);
    soa[static_cast<size_t>(k) * Gp + g] = static_cast<float>(aos[i]);
}
__global__ void k_soa32_to_aos64_range(const float* __restrict__ soa, int g0, int g1, int Gp, double* __restrict__ aos) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x + static_cast<long long>(g0) * kP;
    if (i >= static_cast<long long>(g1) * kP) return;
    const int g = static_cast<int>(i / kP), k = static_cast<int>(i - static_cast<long long>(g) * kP);
    aos[i] = static_cast<double>(soa[static_cast<size_t>(k) * Gp + g]);
}
void launch_aos64_to_soa32_range(const double* aos, int g0, int g1, int Gp, float* soa, cudaStream_t st) {
    if (g1 <= g0) return;
    k_aos64_to_soa32_range<<<static_cast<unsigned>((static_cast<long long>(g1 - g0) * kP + 255) / 256), 256, 0, st>>>(
        aos, g0, g1, Gp, soa);
    ++g_launches;
}
void launch_soa32_to_aos64_range(const float* soa, int g0, int g1, int Gp, double* aos, cudaStream_t st) {
    if (g1 <= g0) return;
    k_soa32_to_aos64_range<<<static_cast<unsigned>((static_cast<long long>(g1 - g0) * kP + 255) / 256), 256, 0, st>>>(
        soa, g0, g1, Gp, aos);
    ++g_launches;
}
// GaussianSet SoA (means[3G], ...) f64 <-> device [14][Gp] f64
__global__ void k_set_to_beta(const double* __restrict__ means, const double* __restrict__ ls,
                              const double* __restrict__ rot, const double* __restrict__ logit,
                              const double* __restrict__ col, int G, int Gp, double* __restrict__ beta,
                              float* __restrict__ beta32) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= G) return;
    double b[kP];
    for (int k = 0; k < 3; ++k) {
        b[k] = means[3 * g + k];
        b[3 + k] = ls[3 * g + k];
        b[11 + k] = col[3 * g + k];
    }
    for (int k = 0; k < 4; ++k) b[6 + k] = rot[4 * g + k];
    b[10] = logit[g];
    for (int k = 0; k < kP; ++k) {
        beta[k * Gp + g] = b[k];
        beta32[k * Gp + g] = (float)b[k];
    }
}
__global__ void k_beta_to_set(const double* __restrict__ beta, int G, int Gp, double* __restrict__ means,
                              double* __restrict__ ls, double* __restrict__ rot,
                              double* __restrict__ logit, double* __restrict__ col) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= G) return;
    for (int k = 0; k < 3; ++k) {
        means[3 * g + k] = beta[k * Gp + g];
        ls[3 * g + k] = beta[(3 + k) * Gp + g];
        col[3 * g + k] = beta[(11 + k) * Gp + g];
    }
    for (int k = 0; k < 4; ++k) rot[4 * g + k] = beta[(6 + k) * Gp + g];
    logit[g] = beta[10 * Gp + g];
}

// ---------------------------------------------------------------- reductions
// partial[b] = sum over the block's grid-stride slice of a[i]*b[i] (f64 acc)
__global__ void __launch_bounds__(kRedThreads) k_dot_partial(const float* __restrict__ a,
                                                             const float* __restrict__ b, long long n,
                                                             double* __restrict__ partial,
                                                             const int* __restrict__ done) {
    __shared__ double sh[kRedThreads / 32];
    if (done && *done) return;
    double s = 0.0;
    const long long n4 = n >> 2;
    const float4* a4 = reinterpret_cast<const float4*>(a);
    const float4* b4 = reinterpret_cast<const float4*>(b);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
        const float4 x = a4[i], y = b4[i];
        s += (double)x.x * y.x + (double)x.y * y.y + (double)x.z * y.z + (double)x.w * y.w;
    }
    s = block_sum(s, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__device__ __forceinline__ double sum_partials(const double* __restrict__ partial, double* sh) {
    double s = 0.0;
    for (int i = threadIdx.x; i < kRedBlocks; i += blockDim.x) s += partial[i];
    return block_sum(s, sh);
}

// plain dot -> out[0]
__global__ void k_dot_final(const double* __restrict__ partial, double* __restrict__ out) {
    __shared__ double sh[kRedThreads / 32];
    const double s = sum_partials(partial, sh);
    if (threadIdx.x == 0) *out = s;
}

// max |x| over the colour rows 11..13 (learning_rate, lm.cpp:30-33)
__global__ void k_color_maxabs(const float* __restrict__ x, int G, int Gp, float* __restrict__ out) {
    __shared__ float sh[32];
    float m = 0.0f;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 3 * G; i += gridDim.x * blockDim.x) {
        const int k = i / G, g = i - k * G;
        m = fmaxf(m, fabsf(x[(11 + k) * Gp + g]));
    }
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        float r = 0.0f;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r = fmaxf(r, sh[i]);
        atomicMax(reinterpret_cast<int*>(out), __float_as_int(r));  // non-negative floats order as ints
    }
}

// ---------------------------------------------------------------- PCG steps
// init: x = 0, r = b, z = minv*r, p = z; partial sums of <b,b> and <r,z>
__global__ void __launch_bounds__(kRedThreads) k_cg_init(const float* __restrict__ b,
                                                         const float* __restrict__ minv, long long n,
                                                         float* __restrict__ x, float* __restrict__ r,
                                                         float* __restrict__ z, float* __restrict__ p,
                                                         double* __restrict__ partial) {
    __shared__ double sh[kRedThreads / 32];
    double sbb = 0.0, srz = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const float bi = b[i], zi = minv[i] * bi;
        x[i] = 0.0f;
        r[i] = bi;
        z[i] = zi;
        p[i] = zi;
        sbb += (double)bi * bi;
        srz += (double)bi * zi;
    }
    sbb = block_sum(sbb, sh);
    srz = block_sum(srz, sh);
    if (threadIdx.x == 0) {
        partial[blockIdx.x] = sbb;
        partial[kRedBlocks + blockIdx.x] = srz;
    }
}

__global__ void k_cg_init_final(const double* __restrict__ partial, CgState* __restrict__ st) {
    __shared__ double sh[kRedThreads / 32];
    const double bb = sum_partials(partial, sh);
    const double rz = sum_partials(partial + kRedBlocks, sh);
    if (threadIdx.x == 0) {
        st->bnorm = sqrt(bb);
        st->rz = rz;
        st->iterations = 0;
        st->breakdown = 0;
        st->done = st->bnorm == 0.0 ? 1 : 0;  // pcg.cpp:18-22
        st->rr = bb;
    }
}

// after u = A p: pu = <p,u>; breakdown if pu <= 0 (pcg.cpp:32-36)
__global__ void k_cg_pu_final(const double* __restrict__ partial, CgState* __restrict__ st) {
    __shared__ double sh[kRedThreads / 32];
    if (st->done) return;
    const double pu = sum_partials(partial, sh);
    if (threadIdx.x == 0) {
        st->pu = pu;
        if (pu <= 0.0) {
            st->breakdown = 1;
            st->done = 1;
        } else {
            st->alpha = st->rz / pu;
        }
    }
}

// x += alpha p; r -= alpha u; z = minv*r; partials of <r,r> and <r,z>
__global__ void __launch_bounds__(kRedThreads) k_cg_update(float* __restrict__ x, float* __restrict__ r,
                                                           float* __restrict__ z,
                                                           const float* __restrict__ p,
                                                           const float* __restrict__ u,
                                                           const float* __restrict__ minv, long long n,
                                                           const CgState* __restrict__ st,
                                                           double* __restrict__ partial) {
    __shared__ double sh[kRedThreads / 32];
    if (st->done) return;
    const float alpha = (float)st->alpha;
    double srr = 0.0, srz = 0.0;
    const long long n4 = n >> 2;
    float4* x4 = reinterpret_cast<float4*>(x);
    float4* r4 = reinterpret_cast<float4*>(r);
    float4* z4 = reinterpret_cast<float4*>(z);
    const float4* p4 = reinterpret_cast<const float4*>(p);
    const float4* u4 = reinterpret_cast<const float4*>(u);
    const float4* m4 = reinterpret_cast<const float4*>(minv);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
        float4 xi = x4[i], ri = r4[i];
        const float4 pi = p4[i], ui = u4[i], mi = m4[i];
        xi.x += alpha * pi.x; xi.y += alpha * pi.y; xi.z += alpha * pi.z; xi.w += alpha * pi.w;
        ri.x -= alpha * ui.x; ri.y -= alpha * ui.y; ri.z -= alpha * ui.z; ri.w -= alpha * ui.w;
        const float4 zi = make_float4(mi.x * ri.x, mi.y * ri.y, mi.z * ri.z, mi.w * ri.w);
        x4[i] = xi;
        r4[i] = ri;
        z4[i] = zi;
        srr += (double)ri.x * ri.x + (double)ri.y * ri.y + (double)ri.z * ri.z + (double)ri.w * ri.w;
        srz += (double)ri.x * zi.x + (double)ri.y * zi.y + (double)ri.z * zi.z + (double)ri.w * zi.w;
    }
    srr = block_sum(srr, sh);
    srz = block_sum(srz, sh);
    if (threadIdx.x == 0) {
        partial[blockIdx.x] = srr;
        partial[kRedBlocks + blockIdx.x] = srz;
    }
}

// iterations++, early exit on |r| <= 1e-12 |b| (pcg.cpp:41-42), beta = rz'/rz
__global__ void k_cg_update_final(const double* __restrict__ partial, CgState* __restrict__ st) {
    __shared__ double sh[kRedThreads / 32];
    if (st->done) return;
    const double rr = sum_partials(partial, sh);
    const double rz = sum_partials(partial + kRedBlocks, sh);
    if (threadIdx.x == 0) {
        st->iterations += 1;
        st->rr = rr;
        if (sqrt(rr) <= 1e-12 * st->bnorm) {
            st->done = 1;
        } else {
            st->beta = rz / st->rz;
            st->rz = rz;
        }
    }
}

// p = z + beta p (xpby, pcg.cpp:48)
__global__ void k_cg_p(float* __restrict__ p, const float* __restrict__ z, long long n,
                       const CgState* __restrict__ st) {
    if (st->done) return;
    const float beta = (float)st->beta;
    const long long n4 = n >> 2;
    float4* p4 = reinterpret_cast<float4*>(p);
    const float4* z4 = reinterpret_cast<const float4*>(z);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
        float4 pi = p4[i];
        const float4 zi = z4[i];
        pi.x = zi.x + beta * pi.x; pi.y = zi.y + beta * pi.y;
        pi.z = zi.z + beta * pi.z; pi.w = zi.w + beta * pi.w;
        p4[i] = pi;
    }
}

// minv = 1 / (diag + lambda) (lm.cpp:124-125)
__global__ void k_minv(float* __restrict__ d, long long n, float lambda) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        d[i] = 1.0f / (d[i] + lambda);
}

// out = lambda * p + out   (f32)
__global__ void k_axpy(float* __restrict__ y, const float* __restrict__ x, long long n, float a) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        y[i] += a * x[i];
}

// ---------------------------------------------------------------- launchers
void launch_aos64_to_soa32(const double* aos, int G, int Gp, float* soa, cudaStream_t st) {
    if (G == 0) return;
    k_aos64_to_soa32<<<(G * kP + 255) / 256, 256, 0, st>>>(aos, G, Gp, soa); ++g_launches;
}
void launch_soa32_to_aos64(const float* soa, int G, int Gp, double* aos, cudaStream_t st) {
    if (G == 0) return;
    k_soa32_to_aos64<<<(G * kP + 255) / 256, 256, 0, st>>>(soa, G, Gp, aos); ++g_launches;
}
void launch_set_to_beta(const double* m, const double* ls, const double* rot, const double* logit,
                        const double* col, int G, int Gp, double* beta, float* beta32, cudaStream_t st) {
    if (G == 0) return;
    k_set_to_beta<<<(G + 255) / 256, 256, 0, st>>>(m, ls, rot, logit, col, G, Gp, beta, beta32); ++g_launches;
}
void launch_beta_to_set(const double* beta, int G, int Gp, double* m, double* ls, double* rot,
                        double* logit, double* col, cudaStream_t st) {
    if (G == 0) return;
    k_beta_to_set<<<(G + 255) / 256, 256, 0, st>>>(beta, G, Gp, m, ls, rot, logit, col); ++g_launches;
}
void launch_dot(const float* a, const float* b, long long n, double* partial, double* out, cudaStream_t st) {
    k_dot_partial<<<kRedBlocks, kRedThreads, 0, st>>>(a, b, n, partial, nullptr); ++g_launches;
    k_dot_final<<<1, kRedThreads, 0, st>>>(partial, out); ++g_launches;
}
void launch_color_maxabs(const float* x, int G, int Gp, float* out, cudaStream_t st) {
    cudaMemsetAsync(out, 0, sizeof(float), st);
    if (G == 0) return;
    k_color_maxabs<<<kRedBlocks, 256, 0, st>>>(x, G, Gp, out); ++g_launches;
}
void launch_cg_init(const float* b, const float* minv, long long n, float* x, float* r, float* z,
                    float* p, double* partial, CgState* s, cudaStream_t st) {
    k_cg_init<<<kRedBlocks, kRedThreads, 0, st>>>(b, minv, n, x, r, z, p, partial); ++g_launches;
    k_cg_init_final<<<1, kRedThreads, 0, st>>>(partial, s); ++g_launches;
}
void launch_cg_pu(const float* p, const float* u, long long n, double* partial, CgState* s,
                  cudaStream_t st) {
    k_dot_partial<<<kRedBlocks, kRedThreads, 0, st>>>(p, u, n, partial, &s->done); ++g_launches;
    k_cg_pu_final<<<1, kRedThreads, 0, st>>>(partial, s); ++g_launches;
}
void launch_cg_update(float* x, float* r, float* z, float* p, const float* u, const float* minv,
                      long long n, double* partial, CgState* s, cudaStream_t st) {
    k_cg_update<<<kRedBlocks, kRedThreads, 0, st>>>(x, r, z, p, u, minv, n, s, partial); ++g_launches;
    k_cg_update_final<<<1, kRedThreads, 0, st>>>(partial, s); ++g_launches;
    k_cg_p<<<kRedBlocks, kRedThreads, 0, st>>>(p, z, n, s); ++g_launches;
}
void launch_minv(float* d, long long n, float lambda, cudaStream_t st) {
    k_minv<<<kRedBlocks, 256, 0, st>>>(d, n, lambda); ++g_launches;
}
void launch_axpy(float* y, const float* x, long long n, float a, cudaStream_t st) {
    k_axpy<<<kRedBlocks, 256, 0, st>>>(y, x, n, a); ++g_launches;
}

// LocalComm's reduction: dst[i] = sum over ranks k = 0 .. world-1 (in order) of
// src_k[i] (the staging slots; peers' slots over NVLink when on other GPUs)
struct RankPtrs {
    const void* p[64];
};
template <typename T>
__global__ void k_sum_ranks(RankPtrs s, int world, T* __restrict__ dst, long long n) {
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        T acc = static_cast<const T*>(s.p[0])[i];
        for (int k = 1; k < world; ++k) acc += static_cast<const T*>(s.p[k])[i];
        dst[i] = acc;
    }
}
void launch_sum_ranks(void* const* srcs, int world, void* dst, size_t n, bool f64, cudaStream_t st) {
    if (n == 0) return;
    RankPtrs s{};
    for (int k = 0; k < world && k < 64; ++k) s.p[k] = srcs[k];
    if (f64)
        k_sum_ranks<double><<<kRedBlocks, 256, 0, st>>>(s, world, static_cast<double*>(dst), static_cast<long long>(n));
    else
        k_sum_ranks<float><<<kRedBlocks, 256, 0, st>>>(s, world, static_cast<float*>(dst), static_cast<long long>(n));
    ++g_launches;
}

// f32 <-> f64 element copies (the truth images widened for the FP64 metrics,
// FP64 SSIM planes narrowed for the f32 products)
template <typename A, typename B>
__global__ void k_convert(const A* __restrict__ x, B* __restrict__ y, long long n) {
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        y[i] = static_cast<B>(x[i]);
}
void launch_widen(const float* x, double* y, long long n, cudaStream_t st) {
    if (n <= 0) return;
    k_convert<float, double><<<kRedBlocks, 256, 0, st>>>(x, y, n); ++g_launches;
}
void launch_narrow(const double* x, float* y, long long n, cudaStream_t st) {
    if (n <= 0) return;
    k_convert<double, float><<<kRedBlocks, 256, 0, st>>>(x, y, n); ++g_launches;
}

}  // namespace slm
