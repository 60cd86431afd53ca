// chain.cu — per-Gaussian linearisation kernels.
//
// The reference builds a 5x10 ProjChain per (view, Gaussian) from 10 dual
// probes (jacobian.cpp:127-165) and re-runs the full dual preparation for
// every Jv (dual_splats :167-189).  Here the same derivatives are taken
// analytically and factored through the view-independent 3D covariance:
//
//   (mean, log_scale, quat) --view-independent--> (mu, Sigma)
//   (mu, Sigma) --per view--> t = W mu + t_cam, T = J(t) W, cov2d = T Sigma T^T + 0.3 I,
//                             conic = cov2d^{-1}, mean2d = proj(t)
//
// so one thread per Gaussian computes dSigma (forward) or accumulates
// dL/dSigma over the views (reverse) once, and each view only touches the
// cheap projection part.  Mathematically identical to the reference's dual
// evaluation (same function, exact chain rule); differs only in rounding.
//
// FP32 throughout: the conic derivative is taken in matrix form
// (d conic = -conic d cov2d conic) rather than through the determinant, so
// there is no cancellation to protect, and the conic itself comes from the
// FP64 preparation's record; the parameters come from the f32 mirror of the
// f64 state.  These kernels are HBM-bound (records, probe, intermediates).
//
//  * k_tangents       Jv probe: per (view, Gaussian) tangent record of
//                     (mean2d, conic, opacity, colour) along p            [K8]
//  * k_chain          J^T: 9-float intermediates -> 14 parameter grads, + lambda p,
//                     zeroes the intermediates for the next product         [K11]
//  * k_diag_finalize  diag(J^T W J) from the per-entry quadratic forms     [K13]
#include <cstdint>

#include <atomic>

#include "common.cuh"

namespace slm { extern std::atomic<long long> g_launches; }

namespace slm {

struct Geom {  // view-independent part
    float mu[3];
    float qn[4];   // normalised quaternion
    float qinv;    // 1/|q|
    float R[9], s[3], M[9], Sig[9];
    float o;       // sigmoid(logit)
    float dcol[3]; // C0 if the colour gate is open else 0 (rasterizer.hpp:83-86)
};

__device__ __forceinline__ void load_geom(const float* __restrict__ beta, int Gp, int g, Geom& G) {
    for (int k = 0; k < 3; ++k) G.mu[k] = beta[k * Gp + g];
    const float q[4] = {beta[6 * Gp + g], beta[7 * Gp + g], beta[8 * Gp + g], beta[9 * Gp + g]};
    const float nsq = q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3];
    G.qinv = nsq > 0.0f ? rsqrtf(nsq) : 0.0f;
    for (int k = 0; k < 4; ++k) G.qn[k] = q[k] * G.qinv;
    const float w = G.qn[0], x = G.qn[1], y = G.qn[2], z = G.qn[3];
    G.R[0] = 1.0f - 2.0f * (y * y + z * z);
    G.R[1] = 2.0f * (x * y - w * z);
    G.R[2] = 2.0f * (x * z + w * y);
    G.R[3] = 2.0f * (x * y + w * z);
    G.R[4] = 1.0f - 2.0f * (x * x + z * z);
    G.R[5] = 2.0f * (y * z - w * x);
    G.R[6] = 2.0f * (x * z - w * y);
    G.R[7] = 2.0f * (y * z + w * x);
    G.R[8] = 1.0f - 2.0f * (x * x + y * y);
    for (int k = 0; k < 3; ++k) G.s[k] = expf(beta[(3 + k) * Gp + g]);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) G.M[3 * i + j] = G.R[3 * i + j] * G.s[j];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            G.Sig[3 * i + j] = G.M[3 * i] * G.M[3 * j] + G.M[3 * i + 1] * G.M[3 * j + 1] +
                               G.M[3 * i + 2] * G.M[3 * j + 2];
    G.o = 1.0f / (1.0f + expf(-beta[10 * Gp + g]));
    for (int k = 0; k < 3; ++k) {
        const float raw = 0.5f + (float)kColorC0 * beta[(11 + k) * Gp + g];
        G.dcol[k] = raw > 0.0f ? (float)kColorC0 : 0.0f;
    }
}

struct View {  // per-view projection part
    float tx, ty, iz;
    float r0[3], r1[3], Sr0[3], Sr1[3];
    float ca, cb, cc;
};

// The conic comes from the FP64 preparation (k_prepare's conic view
// {A, B, C, opacity}, scaled by log2(e)), so only t, J, r0, r1 and Sigma r are
// recomputed here.
__device__ __forceinline__ void load_view(const Geom& G, const DevCam& cam, const float4 cn, View& V) {
    const float W[9] = {(float)cam.R[0], (float)cam.R[1], (float)cam.R[2], (float)cam.R[3], (float)cam.R[4],
                        (float)cam.R[5], (float)cam.R[6], (float)cam.R[7], (float)cam.R[8]};
    const float fx = (float)cam.fx, fy = (float)cam.fy;
    V.tx = W[0] * G.mu[0] + W[1] * G.mu[1] + W[2] * G.mu[2] + (float)cam.t[0];
    V.ty = W[3] * G.mu[0] + W[4] * G.mu[1] + W[5] * G.mu[2] + (float)cam.t[1];
    const float tz = W[6] * G.mu[0] + W[7] * G.mu[1] + W[8] * G.mu[2] + (float)cam.t[2];
    V.iz = 1.0f / tz;
    const float iz2 = V.iz * V.iz;
    const float j00 = fx * V.iz, j02 = -fx * V.tx * iz2;
    const float j11 = fy * V.iz, j12 = -fy * V.ty * iz2;
    for (int k = 0; k < 3; ++k) {
        V.r0[k] = j00 * W[k] + j02 * W[6 + k];
        V.r1[k] = j11 * W[3 + k] + j12 * W[6 + k];
    }
    for (int i = 0; i < 3; ++i) {
        V.Sr0[i] = G.Sig[3 * i] * V.r0[0] + G.Sig[3 * i + 1] * V.r0[1] + G.Sig[3 * i + 2] * V.r0[2];
        V.Sr1[i] = G.Sig[3 * i] * V.r1[0] + G.Sig[3 * i + 1] * V.r1[1] + G.Sig[3 * i + 2] * V.r1[2];
    }
    constexpr float kLn2f = 0.69314718055994530942f;
    V.ca = -2.0f * kLn2f * cn.x;
    V.cb = -kLn2f * cn.y;
    V.cc = -2.0f * kLn2f * cn.z;
}

// dSigma (full 3x3) along (dlog_scale, dquat) — forward mode of covariance_3d.
__device__ __forceinline__ void dsigma(const Geom& G, const float dls[3], const float dq[4], float dS[9]) {
    const float proj = G.qn[0] * dq[0] + G.qn[1] * dq[1] + G.qn[2] * dq[2] + G.qn[3] * dq[3];
    float dn[4];
    for (int k = 0; k < 4; ++k) dn[k] = (dq[k] - G.qn[k] * proj) * G.qinv;
    const float w = G.qn[0], x = G.qn[1], y = G.qn[2], z = G.qn[3];
    const float dw = dn[0], dx = dn[1], dy = dn[2], dz = dn[3];
    float dR[9];
    dR[0] = -4.0f * (y * dy + z * dz);
    dR[1] = 2.0f * (dx * y + x * dy - dw * z - w * dz);
    dR[2] = 2.0f * (dx * z + x * dz + dw * y + w * dy);
    dR[3] = 2.0f * (dx * y + x * dy + dw * z + w * dz);
    dR[4] = -4.0f * (x * dx + z * dz);
    dR[5] = 2.0f * (dy * z + y * dz - dw * x - w * dx);
    dR[6] = 2.0f * (dx * z + x * dz - dw * y - w * dy);
    dR[7] = 2.0f * (dy * z + y * dz + dw * x + w * dx);
    dR[8] = -4.0f * (x * dx + y * dy);
    float dM[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) dM[3 * i + j] = dR[3 * i + j] * G.s[j] + G.R[3 * i + j] * G.s[j] * dls[j];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            float acc = 0.0f;
            for (int k = 0; k < 3; ++k) acc += dM[3 * i + k] * G.M[3 * j + k] + G.M[3 * i + k] * dM[3 * j + k];
            dS[3 * i + j] = acc;
        }
}

// Tangent of (mean2d, conic) for one view given (dmu, dSigma).
__device__ __forceinline__ void view_tangent(const View& V, const DevCam& cam, const float dmu[3],
                                             const float dS[9], float out[5]) {
    const float W[9] = {(float)cam.R[0], (float)cam.R[1], (float)cam.R[2], (float)cam.R[3], (float)cam.R[4],
                        (float)cam.R[5], (float)cam.R[6], (float)cam.R[7], (float)cam.R[8]};
    const float fx = (float)cam.fx, fy = (float)cam.fy;
    const float dtx = W[0] * dmu[0] + W[1] * dmu[1] + W[2] * dmu[2];
    const float dty = W[3] * dmu[0] + W[4] * dmu[1] + W[5] * dmu[2];
    const float dtz = W[6] * dmu[0] + W[7] * dmu[1] + W[8] * dmu[2];
    const float diz = -dtz * V.iz * V.iz;
    out[0] = fx * (dtx * V.iz + V.tx * diz);
    out[1] = fy * (dty * V.iz + V.ty * diz);
    const float iz2 = V.iz * V.iz, diz2 = 2.0f * V.iz * diz;
    const float dj00 = fx * diz, dj02 = -fx * (dtx * iz2 + V.tx * diz2);
    const float dj11 = fy * diz, dj12 = -fy * (dty * iz2 + V.ty * diz2);
    float dr0[3], dr1[3];
    for (int k = 0; k < 3; ++k) {
        dr0[k] = dj00 * W[k] + dj02 * W[6 + k];
        dr1[k] = dj11 * W[3 + k] + dj12 * W[6 + k];
    }
    float dSr0[3], dSr1[3];
    for (int i = 0; i < 3; ++i) {
        dSr0[i] = dS[3 * i] * V.r0[0] + dS[3 * i + 1] * V.r0[1] + dS[3 * i + 2] * V.r0[2];
        dSr1[i] = dS[3 * i] * V.r1[0] + dS[3 * i + 1] * V.r1[1] + dS[3 * i + 2] * V.r1[2];
    }
    const float da = 2.0f * (dr0[0] * V.Sr0[0] + dr0[1] * V.Sr0[1] + dr0[2] * V.Sr0[2]) +
                     (V.r0[0] * dSr0[0] + V.r0[1] * dSr0[1] + V.r0[2] * dSr0[2]);
    const float db = (dr0[0] * V.Sr1[0] + dr0[1] * V.Sr1[1] + dr0[2] * V.Sr1[2]) +
                     (dr1[0] * V.Sr0[0] + dr1[1] * V.Sr0[1] + dr1[2] * V.Sr0[2]) +
                     (V.r0[0] * dSr1[0] + V.r0[1] * dSr1[1] + V.r0[2] * dSr1[2]);
    const float dc = 2.0f * (dr1[0] * V.Sr1[0] + dr1[1] * V.Sr1[1] + dr1[2] * V.Sr1[2]) +
                     (V.r1[0] * dSr1[0] + V.r1[1] * dSr1[1] + V.r1[2] * dSr1[2]);
    const float ca = V.ca, cb = V.cb, cc = V.cc;
    out[2] = -(ca * ca * da + 2.0f * ca * cb * db + cb * cb * dc);
    out[3] = -(ca * cb * da + (ca * cc + cb * cb) * db + cb * cc * dc);
    out[4] = -(cb * cb * da + 2.0f * cb * cc * db + cc * cc * dc);
}

// ------------------------------------------------------------------ K8
__global__ void __launch_bounds__(128) k_tangents(const float* __restrict__ beta, const float* __restrict__ p,
                                                  int G, int Gp, const DevCam* __restrict__ cams, int V,
                                                  const float4* __restrict__ conic, float4* __restrict__ tan,
                                                  const int* __restrict__ done_flag, int g0, int g1) {
    if (done_flag && *done_flag) return;
    const int g = g0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= g1) return;
    Geom Gm;
    load_geom(beta, Gp, g, Gm);
    float pv[kP];
    for (int k = 0; k < kP; ++k) pv[k] = p[k * Gp + g];
    float dS[9];
    dsigma(Gm, pv + 3, pv + 6, dS);
    const float dop = Gm.o * (1.0f - Gm.o) * pv[10];
    const float dr = Gm.dcol[0] * pv[11], dg = Gm.dcol[1] * pv[12], db = Gm.dcol[2] * pv[13];
    float4 nc;  // next view's conic view {A, B, C, opacity}, prefetched
    if (V > 0) nc = __ldg(conic + static_cast<size_t>(g));
    for (int v = 0; v < V; ++v) {
        const size_t vg = static_cast<size_t>(v) * Gp + g;
        const float4 cn = nc;
        if (v + 1 < V) nc = __ldg(conic + vg + Gp);
        if (cn.w == 0.0f) continue;  // invalid (view, Gaussian): zero opacity
        const DevCam& cam = cams[v];
        View Vw;
        load_view(Gm, cam, cn, Vw);
        float o5[5];
        view_tangent(Vw, cam, pv, dS, o5);
        // pre-combined so the raster's d(power) is 5 FMAs in (dx, dy):
        // dpow = A1 dx + A2 dy + A3 dx^2 + A4 dx dy + A5 dy^2
        const float A1 = -(Vw.ca * o5[0] + Vw.cb * o5[1]);
        const float A2 = -(Vw.cb * o5[0] + Vw.cc * o5[1]);
        float4* t = tan + 3 * vg;
        t[0] = make_float4(A1, A2, -0.5f * o5[2], -o5[3]);
        t[1] = make_float4(-0.5f * o5[4], dop, dr, dg);
        t[2] = make_float4(db, 0.f, 0.f, 0.f);
    }
}

// ------------------------------------------------------------------ deterministic sums
// A (view, Gaussian)'s partial records -- one per compacted tile-list entry
// that carries it, written by the raster at their position in the per-plan
// (view, Gaussian, slot) order -- are the contiguous range [seg[vg],
// seg[vg + 1]); the thread adds them front to back (two records' loads in
// flight per step).  The order is a function of the plan only, so every
// product rounds identically (the reference's contract: results independent
// of scheduling, jacobian.cpp:19-21,246-247).  The bounds of the next view
// are loaded one view ahead.
struct DetSeg {
    unsigned a, b;  // this thread's records [a, b)
};
__device__ __forceinline__ DetSeg det_seg(const DetOrder& D, size_t vg) {
    return DetSeg{__ldg(D.seg + vg), __ldg(D.seg + vg + 1)};
}

template <int STRIDE4, int NF4>  // record stride and used float4s
__device__ __forceinline__ void det_sum(const DetOrder& D, DetSeg sg, float4 acc[NF4]) {
#pragma unroll
    for (int q = 0; q < NF4; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4* part = reinterpret_cast<const float4*>(D.partial);
    auto add = [&](const float4* v) {
#pragma unroll
        for (int q = 0; q < NF4; ++q) {
            acc[q].x += v[q].x;
            acc[q].y += v[q].y;
            acc[q].z += v[q].z;
            acc[q].w += v[q].w;
        }
    };
    unsigned j = sg.a;
    for (; j + 1 < sg.b; j += 2) {
        float4 r0[NF4], r1[NF4];
        const float4* p0 = part + static_cast<size_t>(j) * STRIDE4;
#pragma unroll
        for (int q = 0; q < NF4; ++q) {
            r0[q] = __ldcs(p0 + q);
            r1[q] = __ldcs(p0 + STRIDE4 + q);
        }
        add(r0);
        add(r1);
    }
    if (j < sg.b) {
        float4 r0[NF4];
        const float4* p0 = part + static_cast<size_t>(j) * STRIDE4;
#pragma unroll
        for (int q = 0; q < NF4; ++q) r0[q] = __ldcs(p0 + q);
        add(r0);
    }
}

// Warp-staged ordered sums (the fused deterministic path): the records of
// the 32 consecutive keys (v, g0 .. g0+31) of a warp are ONE contiguous range
// [seg[v Gp + g0], seg[v Gp + g0 + 32]), so lane 0 brings the next view's
// range into shared memory with one cp.async.bulk while the warp works on the
// current view (double-buffered, one mbarrier per buffer); each lane then
// sums its own records from shared memory in the same order as det_sum
// (bitwise the same result).  A range longer than CAP records is summed from
// global memory instead.
template <int STRIDE4, int CAP>
struct DetStage {
    float4* buf;    // [2][CAP * STRIDE4]
    uint64_t* bar;  // [2]
    unsigned A0, B0, A1, B1;  // the staged range per buffer (no dynamic indexing: registers)
    uint32_t par;
    __device__ __forceinline__ void init(int lane) {
        if (lane == 0) {
            mbar_init(bar, 1);
            mbar_init(bar + 1, 1);
        }
        par = 0u;
        __syncwarp();
    }
    // the warp's range of this key segment set (lane 31 holds the last key)
    __device__ __forceinline__ void issue(const DetOrder& D, DetSeg sg, int slot, int lane) {
        const unsigned a = __shfl_sync(0xffffffffu, sg.a, 0), b = __shfl_sync(0xffffffffu, sg.b, 31);
        if (slot) {
            A1 = a;
            B1 = b;
        } else {
            A0 = a;
            B0 = b;
        }
        if (lane == 0 && b > a && b - a <= CAP)
            bulk_load(buf + slot * CAP * STRIDE4, reinterpret_cast<const float4*>(D.partial) + static_cast<size_t>(a) * STRIDE4,
                      (b - a) * STRIDE4 * 16u, bar + slot);
    }
    template <int NF4>
    __device__ __forceinline__ void sum(const DetOrder& D, DetSeg sg, int slot, float4 acc[NF4]) {
        const unsigned a = slot ? A1 : A0, b = slot ? B1 : B0;
        if (!(b > a && b - a <= CAP)) {
            det_sum<STRIDE4, NF4>(D, sg, acc);
            return;
        }
        mbar_wait(bar + slot, (par >> slot) & 1u);
        par ^= 1u << slot;
#pragma unroll
        for (int q = 0; q < NF4; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        const float4* r = buf + slot * CAP * STRIDE4 + static_cast<size_t>(sg.a - a) * STRIDE4;
        for (unsigned j = sg.a; j < sg.b; ++j, r += STRIDE4) {
#pragma unroll
            for (int q = 0; q < NF4; ++q) {
                const float4 v = r[q];
                acc[q].x += v.x;
                acc[q].y += v.y;
                acc[q].z += v.z;
                acc[q].w += v.w;
            }
        }
    }
};

// Deterministic segmented reduction, parallel over records: one warp per 32
// consecutive keys (view, Gaussian) -- their records are the contiguous range
// [seg[k0], seg[k0 + 32]) -- walked in chunks of 32 records (one per lane,
// coalesced).  Within a chunk a Hillis-Steele segmented inclusive scan (heads
// = the keys' first records, fixed shuffle pattern) gives each key's chunk
// partial at its last record; the key's lane adds the chunk partials in chunk
// order.  Every addition is fixed by the plan, so the sums are bitwise
// reproducible.  Writes all keys (zero for empty segments) with OSTRIDE4
// float4 per key (the inter / diagacc layouts).
template <int NF4, int STRIDE4, int OSTRIDE4>
__global__ void __launch_bounds__(256) k_det_reduce(const unsigned* __restrict__ seg, const float4* __restrict__ part,
                                                    long long n_keys, float4* __restrict__ out) {
    const long long k0 = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) & ~31ll;
    const int lane = threadIdx.x & 31;
    if (k0 >= n_keys) return;
    const long long k = k0 + lane;
    const bool live = k < n_keys;
    const unsigned a = live ? __ldg(seg + k) : __ldg(seg + n_keys), b = live ? __ldg(seg + k + 1) : __ldg(seg + n_keys);
    const unsigned r0 = __shfl_sync(0xffffffffu, a, 0), r1 = __shfl_sync(0xffffffffu, b, 31);
    float4 acc[NF4];
#pragma unroll
    for (int q = 0; q < NF4; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (unsigned base = r0; base < r1; base += 32) {
        const unsigned i = base + lane;
        float4 v[NF4];
#pragma unroll
        for (int q = 0; q < NF4; ++q)
            v[q] = i < r1 ? __ldcs(part + static_cast<size_t>(i) * STRIDE4 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        const bool starts = a < b && a >= base && a < base + 32;
        const unsigned heads = __reduce_or_sync(0xffffffffu, starts ? 1u << (a - base) : 0u) | 1u;
        const int h = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));  // this record's segment head
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
            for (int q = 0; q < NF4; ++q) {
                const float x = __shfl_up_sync(0xffffffffu, v[q].x, d), y = __shfl_up_sync(0xffffffffu, v[q].y, d);
                const float z = __shfl_up_sync(0xffffffffu, v[q].z, d), w = __shfl_up_sync(0xffffffffu, v[q].w, d);
                if (lane - d >= h) {
                    v[q].x += x;
                    v[q].y += y;
                    v[q].z += z;
                    v[q].w += w;
                }
            }
        }
        const bool hit = a < b && a < base + 32 && b > base;  // this key has records in the chunk
        const int e = static_cast<int>((b < base + 32 ? b : base + 32) - 1 - base);
        const int src = hit ? e : lane;
#pragma unroll
        for (int q = 0; q < NF4; ++q) {
            const float x = __shfl_sync(0xffffffffu, v[q].x, src), y = __shfl_sync(0xffffffffu, v[q].y, src);
            const float z = __shfl_sync(0xffffffffu, v[q].z, src), w = __shfl_sync(0xffffffffu, v[q].w, src);
            if (hit) {
                acc[q].x += x;
                acc[q].y += y;
                acc[q].z += z;
                acc[q].w += w;
            }
        }
    }
    if (live) {
        float4* o = out + static_cast<size_t>(k) * OSTRIDE4;
#pragma unroll
        for (int q = 0; q < NF4; ++q) o[q] = acc[q];
#pragma unroll
        for (int q = NF4; q < OSTRIDE4; ++q) o[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

// ------------------------------------------------------------------ K11
// out[k][g] = lambda p[k][g] + sum_v (dconic, dmean2d, ... / dbeta)^T inter_v[g],
// exact reverse mode of the projection.  MODE 0 (atomic): inter holds the
// red.global.add sums and is zeroed after reading.  MODE 1 (deterministic,
// fused): inter_v[g] is the ordered sum of the (view, Gaussian)'s records
// (det_sum).  MODE 2 (deterministic, k_det_reduce first): inter is read as is.
constexpr int kChainThreads = 64;
constexpr int kChainCap = 128;  // staged records per warp and view (6 KB)
template <int MODE>
__global__ void __launch_bounds__(kChainThreads) k_chain(const float* __restrict__ beta, int G, int Gp,
                                               const DevCam* __restrict__ cams, int V,
                                               const float4* __restrict__ conic, float* __restrict__ inter,
                                               DetOrder D, const float* __restrict__ p, float lambda,
                                               float* __restrict__ out, const int* __restrict__ done_flag, int g0,
                                               int g1) {
    if (done_flag && *done_flag) return;
    const int g = g0 + blockIdx.x * blockDim.x + threadIdx.x;
    constexpr bool DET = MODE == 1;
    // the fused deterministic path stages each view's records per warp
    // (DetStage): every lane of a warp with any live Gaussian takes part
    __shared__ __align__(16) float4 s_det[DET ? kChainThreads / 32 : 1][DET ? 2 * kChainCap * (kDetRec / 4) : 1];
    __shared__ uint64_t s_dbar[kChainThreads / 32][2];
    if (g0 + blockIdx.x * blockDim.x + (threadIdx.x & ~31) >= g1) return;  // whole warp past the range
    const bool live = g < g1;
    const int gl = live ? g : g1 - 1;  // dead lanes shadow a live Gaussian (never written)
    DetStage<kDetRec / 4, kChainCap> ds{s_det[threadIdx.x >> 5], s_dbar[threadIdx.x >> 5], 0u, 0u, 0u, 0u, 0u};
    if (DET) ds.init(threadIdx.x & 31);
    Geom Gm;
    load_geom(beta, Gp, gl, Gm);
    float gs00 = 0, gs01 = 0, gs02 = 0, gs11 = 0, gs12 = 0, gs22 = 0;  // gS + gS^T
    float gmu0 = 0, gmu1 = 0, gmu2 = 0, go = 0, gc0 = 0, gc1 = 0, gc2 = 0;
    // Software pipeline: view v+1's record and intermediate are loaded
    // (unconditionally; invalid pairs hold zeros) while view v is processed.
    float4 nc, ni0, ni1, ni2;
    auto fetch = [&](int v) {
        const size_t vg = static_cast<size_t>(v) * Gp + gl;
        nc = __ldg(conic + vg);
        if (!DET) {
            const float4* ip = reinterpret_cast<const float4*>(inter + vg * kRec);
            ni0 = ip[0];
            ni1 = ip[1];
            ni2 = ip[2];
        }
    };
    if (V > 0) fetch(0);
    // segments of views v (cur) and v + 1 (nxt); view v + 1's range is in flight
    // while view v is summed
    DetSeg sc{0u, 0u}, sn{0u, 0u};
    const unsigned lane = threadIdx.x & 31;
    if (DET && V > 0) {
        sc = det_seg(D, g);
        if (!live) sc.b = sc.a;
        ds.issue(D, det_seg(D, g), 0, lane);  // (dead lanes: g < Gp, keys without records)
        if (V > 1) sn = det_seg(D, static_cast<size_t>(Gp) + g);
    }
    for (int v = 0; v < V; ++v) {
        const size_t vg = static_cast<size_t>(v) * Gp + gl;
        float4 i0 = ni0, i1 = ni1, i2 = ni2;
        if (DET) {
            __syncwarp();  // every lane is done with the buffer view v + 1 reuses
            if (v + 1 < V) ds.issue(D, sn, (v + 1) & 1, lane);
            const DetSeg sg = sc;
            sc = sn;
            if (!live) sc.b = sc.a;
            if (v + 2 < V) sn = det_seg(D, static_cast<size_t>(v + 2) * Gp + g);
            float4 acc[3];
            ds.template sum<3>(D, sg, v & 1, acc);
            i0 = acc[0];
            i1 = acc[1];
            i2 = acc[2];
        }
        const float4 cn = nc;
        if (v + 1 < V) fetch(v + 1);
        if (!live || cn.w == 0.0f) continue;  // invalid (view, Gaussian): zero opacity
        if (MODE == 0) {
            float4* ip = reinterpret_cast<float4*>(inter + vg * kRec);
            ip[0] = make_float4(0.f, 0.f, 0.f, 0.f);
            ip[1] = make_float4(0.f, 0.f, 0.f, 0.f);
            ip[2] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        const float gmx = i0.x, gmy = i0.y, gca = i0.z, gcb = i0.w, gcc = i1.x;
        go += i1.y;
        gc0 += i1.z;
        gc1 += i1.w;
        gc2 += i2.x;
        const DevCam& cam = cams[v];
        View Vw;
        load_view(Gm, cam, cn, Vw);
        const float ca = Vw.ca, cb = Vw.cb, cc = Vw.cc;
        // conic -> cov2d (a, b, c): adjoint of d conic = -C dA C
        const float ga = -(gca * ca * ca + gcb * ca * cb + gcc * cb * cb);
        const float gb = -(2.0f * gca * ca * cb + gcb * (ca * cc + cb * cb) + 2.0f * gcc * cc * cb);
        const float gc = -(gca * cb * cb + gcb * cb * cc + gcc * cc * cc);
        float gr0[3], gr1[3];
        for (int k = 0; k < 3; ++k) {
            gr0[k] = 2.0f * ga * Vw.Sr0[k] + gb * Vw.Sr1[k];
            gr1[k] = gb * Vw.Sr0[k] + 2.0f * gc * Vw.Sr1[k];
        }
        const float* r0 = Vw.r0;
        const float* r1 = Vw.r1;
        gs00 += 2.0f * (ga * r0[0] * r0[0] + gb * r0[0] * r1[0] + gc * r1[0] * r1[0]);
        gs11 += 2.0f * (ga * r0[1] * r0[1] + gb * r0[1] * r1[1] + gc * r1[1] * r1[1]);
        gs22 += 2.0f * (ga * r0[2] * r0[2] + gb * r0[2] * r1[2] + gc * r1[2] * r1[2]);
        gs01 += 2.0f * ga * r0[0] * r0[1] + gb * (r0[0] * r1[1] + r1[0] * r0[1]) + 2.0f * gc * r1[0] * r1[1];
        gs02 += 2.0f * ga * r0[0] * r0[2] + gb * (r0[0] * r1[2] + r1[0] * r0[2]) + 2.0f * gc * r1[0] * r1[2];
        gs12 += 2.0f * ga * r0[1] * r0[2] + gb * (r0[1] * r1[2] + r1[1] * r0[2]) + 2.0f * gc * r1[1] * r1[2];
        const float W[9] = {(float)cam.R[0], (float)cam.R[1], (float)cam.R[2], (float)cam.R[3], (float)cam.R[4],
                            (float)cam.R[5], (float)cam.R[6], (float)cam.R[7], (float)cam.R[8]};
        const float fx = (float)cam.fx, fy = (float)cam.fy;
        const float gj00 = gr0[0] * W[0] + gr0[1] * W[1] + gr0[2] * W[2];
        const float gj02 = gr0[0] * W[6] + gr0[1] * W[7] + gr0[2] * W[8];
        const float gj11 = gr1[0] * W[3] + gr1[1] * W[4] + gr1[2] * W[5];
        const float gj12 = gr1[0] * W[6] + gr1[1] * W[7] + gr1[2] * W[8];
        const float iz = Vw.iz, iz2 = iz * iz;
        const float gtx = gmx * fx * iz - gj02 * fx * iz2;
        const float gty = gmy * fy * iz - gj12 * fy * iz2;
        const float giz = gmx * fx * Vw.tx + gmy * fy * Vw.ty + gj00 * fx + gj11 * fy -
                          2.0f * gj02 * fx * Vw.tx * iz - 2.0f * gj12 * fy * Vw.ty * iz;
        const float gtz = -giz * iz2;
        gmu0 += W[0] * gtx + W[3] * gty + W[6] * gtz;
        gmu1 += W[1] * gtx + W[4] * gty + W[7] * gtz;
        gmu2 += W[2] * gtx + W[5] * gty + W[8] * gtz;
    }
    // Sigma = M M^T: gM = (gS + gS^T) M ; M = R diag(s)
    const float gSs[9] = {gs00, gs01, gs02, gs01, gs11, gs12, gs02, gs12, gs22};
    float gM[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            gM[3 * i + j] = gSs[3 * i] * Gm.M[j] + gSs[3 * i + 1] * Gm.M[3 + j] + gSs[3 * i + 2] * Gm.M[6 + j];
    float gR[9], gls[3];
    for (int j = 0; j < 3; ++j) {
        float gsj = 0.0f;
        for (int i = 0; i < 3; ++i) {
            gR[3 * i + j] = gM[3 * i + j] * Gm.s[j];
            gsj += gM[3 * i + j] * Gm.R[3 * i + j];
        }
        gls[j] = gsj * Gm.s[j];
    }
    const float w = Gm.qn[0], x = Gm.qn[1], y = Gm.qn[2], z = Gm.qn[3];
    float gn[4];
    gn[0] = 2.0f * (-z * gR[1] + y * gR[2] + z * gR[3] - x * gR[5] - y * gR[6] + x * gR[7]);
    gn[1] = 2.0f * (y * gR[1] + z * gR[2] + y * gR[3] - 2.0f * x * gR[4] - w * gR[5] + z * gR[6] +
                    w * gR[7] - 2.0f * x * gR[8]);
    gn[2] = 2.0f * (-2.0f * y * gR[0] + x * gR[1] + w * gR[2] + x * gR[3] + z * gR[5] - w * gR[6] +
                    z * gR[7] - 2.0f * y * gR[8]);
    gn[3] = 2.0f * (-2.0f * z * gR[0] - w * gR[1] + x * gR[2] + w * gR[3] - 2.0f * z * gR[4] +
                    y * gR[5] + x * gR[6] + y * gR[7]);
    const float proj = Gm.qn[0] * gn[0] + Gm.qn[1] * gn[1] + Gm.qn[2] * gn[2] + Gm.qn[3] * gn[3];
    float res[kP];
    res[0] = gmu0;
    res[1] = gmu1;
    res[2] = gmu2;
    for (int k = 0; k < 3; ++k) res[3 + k] = gls[k];
    for (int k = 0; k < 4; ++k) res[6 + k] = (gn[k] - Gm.qn[k] * proj) * Gm.qinv;
    res[10] = go * Gm.o * (1.0f - Gm.o);
    res[11] = gc0 * Gm.dcol[0];
    res[12] = gc1 * Gm.dcol[1];
    res[13] = gc2 * Gm.dcol[2];
    if (!live) return;
    for (int k = 0; k < kP; ++k) {
        float val = res[k];
        if (p) val += lambda * p[k * Gp + g];
        out[k * Gp + g] = val;
    }
}

// ------------------------------------------------------------------ K13 finalize
// diag[j] = sum_v P_j^T M_v P_j (j < 10) + opacity / colour rows; the 5x10
// ProjChain columns P_j are the view_tangent of the unit probes e_j.
constexpr int kDiagThreads = 64;
constexpr int kDiagCap = 90;  // staged diag records per warp and view (8.4 KB): 6 CTAs per SM
template <int MODE>
__global__ void __launch_bounds__(kDiagThreads, 6) k_diag_finalize(const float* __restrict__ beta, int G, int Gp,
                                                       const DevCam* __restrict__ cams, int V,
                                                       const float4* __restrict__ conic,
                                                       float* __restrict__ diagacc, DetOrder D,
                                                       float* __restrict__ out) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    constexpr bool DET = MODE == 1;
    __shared__ __align__(16) float4 s_det[DET ? kDiagThreads / 32 : 1][DET ? 2 * kDiagCap * (kDetDiagRec / 4) : 1];
    __shared__ uint64_t s_dbar[kDiagThreads / 32][2];
    if (blockIdx.x * blockDim.x + (threadIdx.x & ~31) >= G) return;  // whole warp past the end
    const bool live = g < G;
    const int gl = live ? g : G - 1;  // dead lanes shadow a live Gaussian (never written)
    DetStage<kDetDiagRec / 4, kDiagCap> ds{s_det[threadIdx.x >> 5], s_dbar[threadIdx.x >> 5], 0u, 0u, 0u, 0u, 0u};
    if (DET) ds.init(threadIdx.x & 31);
    Geom Gm;
    load_geom(beta, Gp, gl, Gm);
    float d[kP];
    for (int k = 0; k < kP; ++k) d[k] = 0.0f;
    const float zero9[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    const float zero3[3] = {0, 0, 0};
    // software pipeline: next view's record and accumulators load during this view
    float4 nc, na[5];
    auto fetch = [&](int v) {
        const size_t vg = static_cast<size_t>(v) * Gp + gl;
        nc = __ldg(conic + vg);
        if (!DET) {
            const float4* a4 = reinterpret_cast<const float4*>(diagacc + vg * kDiagRec);
            for (int q4 = 0; q4 < 5; ++q4) na[q4] = a4[q4];
        }
    };
    if (V > 0) fetch(0);
    // segments of views v (cur) and v + 1 (nxt); view v + 1's records are in
    // flight (DetStage) while view v is summed
    DetSeg sc{0u, 0u}, sn{0u, 0u};
    const unsigned lane = threadIdx.x & 31;
    if (DET && V > 0) {
        sc = det_seg(D, g);
        if (!live) sc.b = sc.a;
        ds.issue(D, det_seg(D, g), 0, lane);
        if (V > 1) sn = det_seg(D, static_cast<size_t>(Gp) + g);
    }
    for (int v = 0; v < V; ++v) {
        const size_t vg = static_cast<size_t>(v) * Gp + gl;
        if (DET) {
            __syncwarp();  // every lane is done with the buffer view v + 1 reuses
            if (v + 1 < V) ds.issue(D, sn, (v + 1) & 1, lane);
            const DetSeg sg = sc;
            sc = sn;
            if (!live) sc.b = sc.a;
            if (v + 2 < V) sn = det_seg(D, static_cast<size_t>(v + 2) * Gp + g);
            ds.template sum<5>(D, sg, v & 1, na);
        }
        const float4 cn = nc;
        float acc[20];
        for (int q4 = 0; q4 < 5; ++q4) {
            acc[4 * q4] = na[q4].x;
            acc[4 * q4 + 1] = na[q4].y;
            acc[4 * q4 + 2] = na[q4].z;
            acc[4 * q4 + 3] = na[q4].w;
        }
        if (v + 1 < V) fetch(v + 1);
        if (!live || cn.w == 0.0f) continue;  // invalid (view, Gaussian)
        if (MODE == 0) {
            float4* acc4 = reinterpret_cast<float4*>(diagacc + vg * kDiagRec);
            for (int q4 = 0; q4 < 5; ++q4) acc4[q4] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        float M[5][5];
        int q = 0;
        for (int i = 0; i < 5; ++i)
            for (int jj = i; jj < 5; ++jj) {
                M[i][jj] = acc[q];
                M[jj][i] = acc[q];
                ++q;
            }
        const DevCam& cam = cams[v];
        View Vw;
        load_view(Gm, cam, cn, Vw);
        // the 10 geometry probes, unrolled so every array index is static (the
        // 3 log-scale + 4 quaternion dSigma are recomputed per view rather than
        // kept as a 63-float array in local memory)
#pragma unroll
        for (int j = 0; j < 10; ++j) {
            float col[5];
            if (j < 3) {
                float dmu[3] = {0, 0, 0};
                dmu[j] = 1.0f;
                view_tangent(Vw, cam, dmu, zero9, col);
            } else {
                float dls[3] = {0, 0, 0}, dq[4] = {0, 0, 0, 0}, dS[9];
                if (j < 6) dls[j - 3] = 1.0f;
                else dq[j - 6] = 1.0f;
                dsigma(Gm, dls, dq, dS);
                view_tangent(Vw, cam, zero3, dS, col);
            }
            float qf = 0.0f;
            for (int a = 0; a < 5; ++a) {
                float r = 0.0f;
                for (int b = 0; b < 5; ++b) r += M[a][b] * col[b];
                qf += col[a] * r;
            }
            d[j] += qf;
        }
        const float ds = Gm.o * (1.0f - Gm.o);
        d[10] += acc[15] * ds * ds;
        d[11] += acc[16] * Gm.dcol[0] * Gm.dcol[0];
        d[12] += acc[17] * Gm.dcol[1] * Gm.dcol[1];
        d[13] += acc[18] * Gm.dcol[2] * Gm.dcol[2];
    }
    // each row is a sum of squares (jtj_diag, jacobian.cpp:272-337); the quadratic
    // form P^T M P of rounded moment sums can dip a few ulp below zero -- clamp
    if (!live) return;
    for (int k = 0; k < kP; ++k) out[k * Gp + g] = fmaxf(d[k], 0.0f);
}

// ------------------------------------------------------------------ launchers
void launch_tangents_range(const float* beta32, const float* p, int G, int Gp, const DevCam* cams, int V,
                           const float4* conic, float4* tan, const int* done, int g0, int g1, cudaStream_t st) {
    g1 = g1 < G ? g1 : G;
    if (g1 <= g0) return;
    k_tangents<<<(g1 - g0 + 127) / 128, 128, 0, st>>>(beta32, p, G, Gp, cams, V, conic, tan, done, g0, g1);
    ++g_launches;
}
void launch_tangents(const float* beta32, const float* p, int G, int Gp, const DevCam* cams, int V,
                     const float4* conic, float4* tan, const int* done, cudaStream_t st) {
    launch_tangents_range(beta32, p, G, Gp, cams, V, conic, tan, done, 0, G, st);
}

// The chain over Gaussians [g0, g1) (the multi-rank path runs it in chunks,
// each chunk's allreduce overlapping the next chunk); `reduce`: run the
// record-parallel k_det_reduce first (deterministic path 0, all keys at once).
void launch_chain_range(const float* beta32, int G, int Gp, const DevCam* cams, int V, const float4* conic,
                        float* inter, const DetOrder& det, const float* p, float lambda, float* out,
                        const int* done, int g0, int g1, bool reduce, cudaStream_t st) {
    g1 = g1 < G ? g1 : G;
    if (g1 <= g0) return;
    const unsigned nb = (g1 - g0 + kChainThreads - 1) / kChainThreads;
    if (!det.partial) {
        k_chain<0><<<nb, kChainThreads, 0, st>>>(beta32, G, Gp, cams, V, conic, inter, det, p, lambda, out, done, g0,
                                                 g1);
    } else if (det.fused) {
        k_chain<1><<<nb, kChainThreads, 0, st>>>(beta32, G, Gp, cams, V, conic, inter, det, p, lambda, out, done, g0,
                                                 g1);
    } else {
        if (reduce) {
            const long long nk = static_cast<long long>(V) * Gp;
            k_det_reduce<kRec / 4, kDetRec / 4, kRec / 4><<<static_cast<unsigned>((nk + 255) / 256), 256, 0, st>>>(
                det.seg, reinterpret_cast<const float4*>(det.partial), nk, reinterpret_cast<float4*>(inter));
            ++g_launches;
        }
        k_chain<2><<<nb, kChainThreads, 0, st>>>(beta32, G, Gp, cams, V, conic, inter, det, p, lambda, out, done, g0,
                                                 g1);
    }
    ++g_launches;
}

void launch_chain(const float* beta32, int G, int Gp, const DevCam* cams, int V, const float4* conic,
                  float* inter, const DetOrder& det, const float* p, float lambda, float* out, const int* done,
                  cudaStream_t st) {
    launch_chain_range(beta32, G, Gp, cams, V, conic, inter, det, p, lambda, out, done, 0, G, true, st);
}

void launch_diag_finalize(const float* beta32, int G, int Gp, const DevCam* cams, int V, const float4* conic,
                          float* diagacc, const DetOrder& det, float* out, cudaStream_t st) {
    if (G == 0) return;
    const unsigned nb = (G + kDiagThreads - 1) / kDiagThreads;
    if (!det.partial) {
        k_diag_finalize<0><<<nb, kDiagThreads, 0, st>>>(beta32, G, Gp, cams, V, conic, diagacc, det, out);
    } else if (det.fused) {
        k_diag_finalize<1><<<nb, kDiagThreads, 0, st>>>(beta32, G, Gp, cams, V, conic, diagacc, det, out);
    } else {
        const long long nk = static_cast<long long>(V) * Gp;
        k_det_reduce<5, kDetDiagRec / 4, kDiagRec / 4><<<static_cast<unsigned>((nk + 255) / 256), 256, 0, st>>>(
            det.seg, reinterpret_cast<const float4*>(det.partial), nk, reinterpret_cast<float4*>(diagacc));
        ++g_launches;
        k_diag_finalize<2><<<nb, kDiagThreads, 0, st>>>(beta32, G, Gp, cams, V, conic, diagacc, det, out);
    }
    ++g_launches;
}

}  // namespace slm
