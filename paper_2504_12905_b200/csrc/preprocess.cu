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

__device__ Prepared prepare_value(const double* __restrict__ beta, int Gp, int g, const DevCam& cam) {
    Prepared out;
    out.valid = false;
    out.zero_quat = false;
    out.radius = 0.0;
    const double mu[3] = {beta[0 * Gp + g], beta[1 * Gp + g], beta[2 * Gp + g]};
    const double ls[3] = {beta[3 * Gp + g], beta[4 * Gp + g], beta[5 * Gp + g]};
    const double q[4] = {beta[6 * Gp + g], beta[7 * Gp + g], beta[8 * Gp + g], beta[9 * Gp + g]};
    const double logit = beta[10 * Gp + g];

    // quat_to_rotation (geometry.hpp:21-39)
    const double nsq = q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3];
    if (nsq == 0.0) {
        out.zero_quat = true;
        return out;
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
    double m[9], sig[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) m[3 * i + j] = r[3 * i + j] * s[j];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            sig[3 * i + j] = m[3 * i] * m[3 * j] + m[3 * i + 1] * m[3 * j + 1] + m[3 * i + 2] * m[3 * j + 2];
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
    out.o = 1.0 / (1.0 + exp(-logit));  // dual.hpp:74
    for (int k = 0; k < 3; ++k) {
        const double raw = 0.5 + kColorC0 * beta[(11 + k) * Gp + g];
        out.col[k] = raw > 0.0 ? raw : 0.0;
    }
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

// grid (ceil(G/256), V): one thread per (view, Gaussian).
__global__ void k_prepare(const double* __restrict__ beta, int G, int Gp,
                          const DevCam* __restrict__ cams, float4* __restrict__ rec,
                          unsigned long long* __restrict__ keys, short4* __restrict__ rect,
                          int* __restrict__ tile_count, int* __restrict__ err) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    const int v = blockIdx.y;
    if (g >= G) return;
    const DevCam cam = cams[v];
    const Prepared p = prepare_value(beta, Gp, g, cam);
    const size_t vg = static_cast<size_t>(v) * Gp + g;
    if (p.zero_quat) atomicOr(err, 1);
    {  // err[1 + v] = G_v, the valid (view, Gaussian) count (warp-aggregated)
        const unsigned am = __activemask();
        const unsigned vm = __ballot_sync(am, p.valid);
        if (vm && (threadIdx.x & 31) == __ffs(am) - 1) atomicAdd(&err[1 + v], __popc(vm));
    }
    keys[vg] = depth_key(p.depth);
    float4* R = rec + 3 * vg;
    if (!p.valid) {
        R[0] = make_float4(0.f, 0.f, 0.f, 0.f);
        R[1] = make_float4(0.f, 0.f, 0.f, 0.f);
        R[2] = make_float4(0.f, 0.f, 0.f, 0.f);
        rect[vg] = make_short4(1, 0, 1, 0);
        return;
    }
    R[0] = make_float4((float)p.mx, (float)p.my, (float)(-0.5 * p.ca * kLog2e), (float)(-p.cb * kLog2e));
    R[1] = make_float4((float)(-0.5 * p.cc * kLog2e), (float)p.o, (float)p.col[0], (float)p.col[1]);
    R[2] = make_float4((float)p.col[2], 1.0f, 0.f, 0.f);  // .y = valid marker
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
    for (int ty = y0; ty <= y1; ++ty)
        for (int tx = x0; tx <= x1; ++tx) atomicAdd(&tile_count[cam.tile_base + ty * cam.tiles_x + tx], 1);
}

// ------------------------------------------------------------------ K3 scan
// Exclusive scan of the batch-concatenated tile counts (single CTA, n is at
// most a few 10^4 tiles).  offsets[n] = total entries.
__global__ void k_scan_tiles(const int* __restrict__ count, int n, int* __restrict__ offsets,
                             int* __restrict__ cursor, long long* __restrict__ total_out) {
    __shared__ long long part[1024];
    const int tid = threadIdx.x, nt = blockDim.x;
    __shared__ int smax;
    const int per = (n + nt - 1) / nt;
    const int lo = tid * per, hi = min(n, lo + per);
    long long s = 0;
    int mx = 0;
    if (tid == 0) smax = 0;
    __syncthreads();
    for (int i = lo; i < hi; ++i) {
        s += count[i];
        mx = max(mx, count[i]);
    }
    atomicMax(&smax, mx);
    part[tid] = s;
    __syncthreads();
    for (int off = 1; off < nt; off <<= 1) {  // Hillis-Steele inclusive scan of partials
        const long long add = tid >= off ? part[tid - off] : 0;
        __syncthreads();
        part[tid] += add;
        __syncthreads();
    }
    long long run = tid == 0 ? 0 : part[tid - 1];
    for (int i = lo; i < hi; ++i) {
        offsets[i] = (int)run;
        cursor[i] = (int)run;
        run += count[i];
    }
    if (tid == nt - 1) {
        offsets[n] = (int)part[nt - 1];
        total_out[0] = part[nt - 1];
        total_out[1] = smax;  // longest tile list: sizes the big-tile sort scratch
    }
}

// ------------------------------------------------------------------ K3 emit
__global__ void k_bin_scatter(int G, int Gp, int V, const DevCam* __restrict__ cams,
                              const short4* __restrict__ rect, int* __restrict__ cursor,
                              int* __restrict__ entries) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    const int v = blockIdx.y;
    if (g >= G) return;
    const short4 r = rect[static_cast<size_t>(v) * Gp + g];
    if (r.x > r.y) return;
    const int base = cams[v].tile_base, tx_n = cams[v].tiles_x;
    for (int ty = r.z; ty <= r.w; ++ty)
        for (int tx = r.x; tx <= r.y; ++tx) {
            const int slot = atomicAdd(&cursor[base + ty * tx_n + tx], 1);
            entries[slot] = g;
        }
}

// ------------------------------------------------------------------ K4 sort
// Per-tile sort by (depth, index) — the reference's std::sort comparator
// (rasterizer.cpp:43-48).  (key, index) pairs are unique, so any correct sort
// reproduces the reference order exactly.
__device__ __forceinline__ bool pair_gt(unsigned long long ka, int va, unsigned long long kb, int vb) {
    return ka > kb || (ka == kb && va > vb);
}

__device__ void bitonic_smem(unsigned long long* key, int* val, int np2) {
    for (int k = 2; k <= np2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < np2; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const bool up = (i & k) == 0;
                    const unsigned long long ka = key[i], kb = key[ixj];
                    const int va = val[i], vb = val[ixj];
                    if (pair_gt(ka, va, kb, vb) == up) {
                        key[i] = kb;
                        key[ixj] = ka;
                        val[i] = vb;
                        val[ixj] = va;
                    }
                }
            }
            __syncthreads();
        }
    }
}

__device__ __forceinline__ int next_pow2(int n) {
    int p = 1;
    while (p < n) p <<= 1;
    return p;
}

template <int CAP>
__global__ void __launch_bounds__(256) k_tile_sort(const int* __restrict__ offsets,
                                                   int* __restrict__ entries,
                                                   const unsigned long long* __restrict__ keys,
                                                   const int* __restrict__ tile_view, int Gp,
                                                   int* __restrict__ overflow,
                                                   int* __restrict__ overflow_count) {
    __shared__ unsigned long long skey[CAP];
    __shared__ int sval[CAP];
    const int tile = blockIdx.x;
    const int b = offsets[tile], n = offsets[tile + 1] - b;
    if (n <= 1) return;
    if (n > CAP) {
        if (threadIdx.x == 0) overflow[atomicAdd(overflow_count, 1)] = tile;
        return;
    }
    const size_t vbase = static_cast<size_t>(tile_view[tile]) * Gp;
    const int np2 = next_pow2(n);
    for (int i = threadIdx.x; i < np2; i += blockDim.x) {
        if (i < n) {
            const int g = entries[b + i];
            skey[i] = keys[vbase + g];
            sval[i] = g;
        } else {
            skey[i] = ~0ull;
            sval[i] = 0x7fffffff;
        }
    }
    __syncthreads();
    bitonic_smem(skey, sval, np2);
    for (int i = threadIdx.x; i < n; i += blockDim.x) entries[b + i] = sval[i];
}

// Overflow tiles (n > 2048): persistent CTAs with up to 16384 entries sorted
// in dynamic shared memory.  Longer lists are sorted in 16384-entry chunks in
// smem and then merged pairwise in global scratch with a merge-path split
// per thread (log2(n/16384) passes), so any list length is handled.
constexpr int kBigCap = 16384;

__device__ __forceinline__ void load_pad(const int* __restrict__ src, int n, int np2,
                                         const unsigned long long* __restrict__ keys, size_t vbase,
                                         unsigned long long* skey, int* sval) {
    for (int i = threadIdx.x; i < np2; i += blockDim.x) {
        if (i < n) {
            const int g = src[i];
            skey[i] = keys[vbase + g];
            sval[i] = g;
        } else {
            skey[i] = ~0ull;
            sval[i] = 0x7fffffff;
        }
    }
    __syncthreads();
}

// Merge sorted runs A=[a0,a1) and B=[a1,b1) of (ka,va) into (kd,vd), whole CTA.
__device__ void merge_runs(const unsigned long long* __restrict__ ka, const int* __restrict__ va,
                           unsigned long long* __restrict__ kd, int* __restrict__ vd, int a0, int a1,
                           int b1) {
    const int la = a1 - a0, lb = b1 - a1, m = la + lb;
    const int T = blockDim.x;
    const int d0 = static_cast<int>(static_cast<long long>(m) * threadIdx.x / T);
    const int d1 = static_cast<int>(static_cast<long long>(m) * (threadIdx.x + 1) / T);
    auto split = [&](int d) {  // number of A elements among the first d merged outputs
        int lo = max(0, d - lb), hi = min(d, la);
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            const int j = d - 1 - mid;
            if (!pair_gt(ka[a0 + mid], va[a0 + mid], ka[a1 + j], va[a1 + j])) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    };
    int i = split(d0), j = d0 - i;
    for (int d = d0; d < d1; ++d) {
        bool take_a;
        if (i >= la) take_a = false;
        else if (j >= lb) take_a = true;
        else take_a = !pair_gt(ka[a0 + i], va[a0 + i], ka[a1 + j], va[a1 + j]);
        if (take_a) {
            kd[a0 + d] = ka[a0 + i];
            vd[a0 + d] = va[a0 + i];
            ++i;
        } else {
            kd[a0 + d] = ka[a1 + j];
            vd[a0 + d] = va[a1 + j];
            ++j;
        }
    }
}

__global__ void __launch_bounds__(1024) k_tile_sort_big(const int* __restrict__ offsets,
                                                        int* __restrict__ entries,
                                                        const unsigned long long* __restrict__ keys,
                                                        const int* __restrict__ tile_view, int Gp,
                                                        const int* __restrict__ overflow,
                                                        const int* __restrict__ overflow_count,
                                                        unsigned long long* __restrict__ scratch_k,
                                                        int* __restrict__ scratch_v, long long max_n) {
    extern __shared__ unsigned char smem_raw[];
    unsigned long long* skey = reinterpret_cast<unsigned long long*>(smem_raw);
    int* sval = reinterpret_cast<int*>(smem_raw + sizeof(unsigned long long) * kBigCap);
    const int cnt = *overflow_count;
    unsigned long long* kA = scratch_k ? scratch_k + 2 * max_n * blockIdx.x : nullptr;
    unsigned long long* kB = kA ? kA + max_n : nullptr;
    int* vA = scratch_v ? scratch_v + 2 * max_n * blockIdx.x : nullptr;
    int* vB = vA ? vA + max_n : nullptr;
    for (int w = blockIdx.x; w < cnt; w += gridDim.x) {
        const int tile = overflow[w];
        const int b = offsets[tile], n = offsets[tile + 1] - b;
        const size_t vbase = static_cast<size_t>(tile_view[tile]) * Gp;
        if (n <= kBigCap) {
            load_pad(entries + b, n, next_pow2(n), keys, vbase, skey, sval);
            bitonic_smem(skey, sval, next_pow2(n));
            for (int i = threadIdx.x; i < n; i += blockDim.x) entries[b + i] = sval[i];
            __syncthreads();
            continue;
        }
        for (int c0 = 0; c0 < n; c0 += kBigCap) {  // sorted chunks -> scratch A
            const int cn = min(kBigCap, n - c0);
            load_pad(entries + b + c0, cn, next_pow2(cn), keys, vbase, skey, sval);
            bitonic_smem(skey, sval, next_pow2(cn));
            for (int i = threadIdx.x; i < cn; i += blockDim.x) {
                kA[c0 + i] = skey[i];
                vA[c0 + i] = sval[i];
            }
            __syncthreads();
        }
        unsigned long long *ks = kA, *kd = kB;
        int *vs = vA, *vd = vB;
        for (int width = kBigCap; width < n; width <<= 1) {
            for (int a0 = 0; a0 < n; a0 += 2 * width) {
                const int a1 = min(a0 + width, n), b1 = min(a0 + 2 * width, n);
                merge_runs(ks, vs, kd, vd, a0, a1, b1);
            }
            __syncthreads();
            unsigned long long* tk = ks; ks = kd; kd = tk;
            int* tv = vs; vs = vd; vd = tv;
        }
        for (int i = threadIdx.x; i < n; i += blockDim.x) entries[b + i] = vs[i];
        __syncthreads();
    }
}

// ------------------------------------------------------------------ K15 update
// GaussianSet::apply_update (types.cpp:48-60) + renormalize_rotations
// (types.cpp:62-73): beta += eta * delta in f64, then q /= |q|.
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
                    unsigned long long* keys, short4* rect, int* tile_count, int* err,
                    cudaStream_t st) {
    if (G == 0 || V == 0) return;
    dim3 grid((G + 255) / 256, V);
    k_prepare<<<grid, 256, 0, st>>>(beta, G, Gp, cams, rec, keys, rect, tile_count, err); ++g_launches;
}

void launch_scan_tiles(const int* count, int n, int* offsets, int* cursor, long long* total,
                       cudaStream_t st) {
    k_scan_tiles<<<1, 1024, 0, st>>>(count, n, offsets, cursor, total); ++g_launches;
}

void launch_bin_scatter(int G, int Gp, int V, const DevCam* cams, const short4* rect, int* cursor,
                        int* entries, cudaStream_t st) {
    if (G == 0 || V == 0) return;
    dim3 grid((G + 255) / 256, V);
    k_bin_scatter<<<grid, 256, 0, st>>>(G, Gp, V, cams, rect, cursor, entries); ++g_launches;
}

void launch_tile_sort(const int* offsets, int* entries, const unsigned long long* keys,
                      const int* tile_view, int n_tiles, int Gp, int* overflow, int* overflow_count,
                      unsigned long long* scratch_k, int* scratch_v, long long max_n, int big_blocks,
                      cudaStream_t st) {
    if (n_tiles == 0) return;
    k_tile_sort<2048><<<n_tiles, 256, 0, st>>>(offsets, entries, keys, tile_view, Gp, overflow,
                                               overflow_count); ++g_launches;
    if (max_n <= 2048) return;  // no overflow tile: skip the persistent big-list kernel
    static bool attr = false;
    const int smem = kBigCap * (sizeof(unsigned long long) + sizeof(int));
    if (!attr) {
        cudaFuncSetAttribute(k_tile_sort_big, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    k_tile_sort_big<<<big_blocks, 1024, smem, st>>>(offsets, entries, keys, tile_view, Gp, overflow,
                                                    overflow_count, scratch_k, scratch_v, max_n); ++g_launches;
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
