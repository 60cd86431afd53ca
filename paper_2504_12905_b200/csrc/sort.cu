// sort.cu — tile-list construction by stable LSD radix sorting.
//
// The reference builds each tile's list by appending Gaussians in index order
// and std::sort-ing it by (depth, index) (rasterizer.cpp:21-50).  Here the
// same order comes out of three device-wide stable passes, with no per-tile
// sort at all:
//   1. depth order: every (view, Gaussian) is sorted by its orderable 64-bit
//      depth key (only the key bytes that vary among the valid Gaussians are
//      sorted), then by view.  Input in index order + stable passes = ties in
//      depth broken by index, exactly the reference comparator;
//   2. emit: in that order, each Gaussian writes its (tile, index) pairs (its
//      tile rect in raster order) at an exclusive-scan offset;
//   3. a stable sort of the pairs by tile id leaves every tile's entries in
//      (depth, index) order at the tile's CSR offset.
// One radix pass = digit histogram per 4096-element block (per-warp smem
// counters), an exclusive scan of the digit-major histogram, and a stable
// scatter that ranks each warp's 512 elements with __match_any_sync (equal
// digits) against per-warp running digit counts, stages the block's elements
// in shared memory in digit order and writes each digit's run out coalesced.
#include <cstdint>

#include <atomic>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace slm { extern std::atomic<long long> g_launches; }

namespace slm {

#ifndef SLM_SCATTER_MINB
#define SLM_SCATTER_MINB 1
#endif
#ifndef SLM_RADIX_MATCH
#define SLM_RADIX_MATCH 0
#endif
constexpr int kRadixThreads = 256;
#ifndef SLM_RADIX_ITEMS
#define SLM_RADIX_ITEMS 8
#endif
constexpr int kRadixItems = SLM_RADIX_ITEMS;
constexpr int kRadixTile = kRadixThreads * kRadixItems;

template <typename K>
__device__ __forceinline__ unsigned digit_of(K k, int shift) {
    return static_cast<unsigned>(k >> shift) & 0xFFu;
}

template <typename K>
__global__ void __launch_bounds__(kRadixThreads) k_radix_hist(const K* __restrict__ keys, long long n, int shift,
                                                              unsigned* __restrict__ hist, int nblocks) {
    __shared__ unsigned hw[kRadixThreads / 32][256];  // per-warp digit counters
#pragma unroll
    for (int w = 0; w < kRadixThreads / 32; ++w) hw[w][threadIdx.x] = 0u;
    const int t = threadIdx.x;
    __syncthreads();
    const long long base = static_cast<long long>(blockIdx.x) * kRadixTile;
    unsigned dig[kRadixItems];
#pragma unroll
    for (int i = 0; i < kRadixItems; ++i) {
        const long long idx = base + i * kRadixThreads + t;
        dig[i] = idx < n ? digit_of(keys[idx], shift) : 256u;
    }
#pragma unroll
    for (int i = 0; i < kRadixItems; ++i)
        if (dig[i] < 256u) atomicAdd(&hw[t >> 5][dig[i]], 1u);
    __syncthreads();
    unsigned sum = 0u;
#pragma unroll
    for (int w = 0; w < kRadixThreads / 32; ++w) sum += hw[w][t];
    hist[static_cast<size_t>(t) * nblocks + blockIdx.x] = sum;
}

// Stable scatter, block-staged, one ranking sweep per block: warp w owns the
// block's elements [512 w, 512 w + 512) (item i, lane l = element 512 w + 32 i
// + l), ranks them with __match_any_sync (the lanes holding the same digit)
// against a per-warp running digit count in shared memory, so the local order
// within a digit is (warp, item, lane) = input order (stable).  The per-warp
// counts are then turned into the block's digit-major local offsets, the
// elements are placed in shared memory in (digit, input) order and written
// out so consecutive threads write consecutive positions of each digit's run
// (coalesced).  `pin`/`pout` (optional) carry a 64-bit payload per element.
template <typename K>
__global__ void __launch_bounds__(kRadixThreads, SLM_SCATTER_MINB) k_radix_scatter(const K* __restrict__ kin,
                                                                  const unsigned* __restrict__ vin,
                                                                  K* __restrict__ kout, unsigned* __restrict__ vout,
                                                                  long long n, int shift,
                                                                  const unsigned* __restrict__ offs, int nblocks,
                                                                  const unsigned long long* __restrict__ pin,
                                                                  unsigned long long* __restrict__ pout) {
    constexpr int NW = kRadixThreads / 32;
    constexpr int WE = kRadixTile / NW;  // elements per warp
    extern __shared__ __align__(16) unsigned char s_raw[];
    unsigned long long* s_pay = reinterpret_cast<unsigned long long*>(s_raw);  // used only with a payload
    K* s_key = reinterpret_cast<K*>(s_raw + (pin ? sizeof(unsigned long long) * kRadixTile : 0));
    unsigned* s_val = reinterpret_cast<unsigned*>(s_key + kRadixTile);
    __shared__ unsigned s_gbase[256], s_lbase[256], s_warp[NW];
    __shared__ unsigned s_wc[NW][257];  // per-warp running digit counts (+ a slot for invalid)
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const long long base = static_cast<long long>(blockIdx.x) * kRadixTile;
    const int cnt = static_cast<int>(n - base < kRadixTile ? n - base : kRadixTile);
    for (int d = lane; d < 257; d += 32) s_wc[warp][d] = 0u;
    __syncwarp();
    const unsigned lt = (1u << lane) - 1u;
    // all of the warp's keys in flight at once (the ranking below is separated
    // by __syncwarp, which the compiler does not move loads across)
    unsigned dig[kRadixItems];
#pragma unroll
    for (int i = 0; i < kRadixItems; ++i) {
        const int li = warp * WE + i * 32 + lane;
        dig[i] = li < cnt ? digit_of(kin[base + li], shift) : 256u;
    }
    unsigned short rank[kRadixItems];
#pragma unroll
    for (int i = 0; i < kRadixItems; ++i) {
        const unsigned d = dig[i];
#if SLM_RADIX_MATCH
        const unsigned peers = __match_any_sync(0xffffffffu, d);
#else
        unsigned peers = 0xffffffffu;  // lanes with the same 9-bit digit (256 = invalid): nine ballots
#pragma unroll
        for (int b = 0; b < 9; ++b) {
            const unsigned bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
            peers &= ((d >> b) & 1u) ? bal : ~bal;
        }
#endif
        const unsigned before = s_wc[warp][d];
        __syncwarp();
        if ((peers & lt) == 0u) s_wc[warp][d] = before + __popc(peers);  // the group's first lane
        __syncwarp();
        rank[i] = static_cast<unsigned short>(before + __popc(peers & lt));
    }
    __syncthreads();
    {   // thread t = digit t: exclusive over warps, then the block's digit starts
        unsigned run = 0u;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const unsigned c = s_wc[w][t];
            s_wc[w][t] = run;
            run += c;
        }
        unsigned incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        unsigned wo = 0u;
        for (int w = 0; w < warp; ++w) wo += s_warp[w];
        s_lbase[t] = wo + incl - run;
        s_gbase[t] = offs[static_cast<size_t>(t) * nblocks + blockIdx.x];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kRadixItems; ++i) {
        const int li = warp * WE + i * 32 + lane;
        if (li < cnt) {
            const K key = kin[base + li];  // L1/L2-resident: read a second time instead of held in registers
            const unsigned d = digit_of(key, shift);
            const unsigned lpos = s_lbase[d] + s_wc[warp][d] + rank[i];
            s_key[lpos] = key;
            s_val[lpos] = vin[base + li];
            if (pin) s_pay[lpos] = pin[base + li];
        }
    }
    __syncthreads();
    for (int i = t; i < cnt; i += kRadixThreads) {
        const K key = s_key[i];
        const unsigned d = digit_of(key, shift);
        const unsigned pos = s_gbase[d] + (static_cast<unsigned>(i) - s_lbase[d]);
        kout[pos] = key;
        vout[pos] = s_val[i];
        if (pin) pout[pos] = s_pay[i];
    }
}

// ---- exclusive scan of u32 (n < 2^31; totals fit u32)
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ unsigned block_exclusive_scan(unsigned v, unsigned* s_warp, unsigned& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        unsigned s = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        s_warp[lane] = s;  // inclusive per-warp totals
    }
    __syncthreads();
    total = s_warp[(blockDim.x >> 5) - 1];
    const unsigned before = warp ? s_warp[warp - 1] : 0u;
    __syncthreads();
    return before + x - v;
}

// Pass 1: per-tile sums.
__global__ void __launch_bounds__(kScanThreads) k_scan_partials(const unsigned* __restrict__ in, long long n,
                                                                unsigned* __restrict__ part) {
    __shared__ unsigned s_warp[32];
    const long long base = static_cast<long long>(blockIdx.x) * kScanTile + static_cast<long long>(threadIdx.x) * kScanItems;
    unsigned s = 0u;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i)
        if (base + i < n) s += in[base + i];
    unsigned total;
    block_exclusive_scan(s, s_warp, total);
    if (threadIdx.x == 0) part[blockIdx.x] = total;
}

// Pass 2: exclusive scan of the partials in one CTA (any count).
__global__ void __launch_bounds__(kScanThreads) k_scan_top(unsigned* __restrict__ part, int m, unsigned* __restrict__ total_out) {
    __shared__ unsigned s_warp[32];
    unsigned carry = 0u;
    for (int b = 0; b < m; b += kScanThreads) {
        const int i = b + threadIdx.x;
        const unsigned v = i < m ? part[i] : 0u;
        unsigned total;
        const unsigned ex = block_exclusive_scan(v, s_warp, total);
        if (i < m) part[i] = carry + ex;
        carry += total;
    }
    if (threadIdx.x == 0 && total_out) *total_out = carry;
}

// Pass 3: per-tile exclusive scan plus the tile's offset.
// (in-place safe: every element is read and written by the same thread)
__global__ void __launch_bounds__(kScanThreads) k_scan_apply(const unsigned* in, long long n,
                                                             const unsigned* __restrict__ part, unsigned* out) {
    __shared__ unsigned s_warp[32];
    const long long base = static_cast<long long>(blockIdx.x) * kScanTile + static_cast<long long>(threadIdx.x) * kScanItems;
    unsigned v[kScanItems];
    unsigned s = 0u;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        v[i] = base + i < n ? in[base + i] : 0u;
        s += v[i];
    }
    unsigned total;
    unsigned run = part[blockIdx.x] + block_exclusive_scan(s, s_warp, total);
#pragma unroll
    for (int i = 0; i < kScanItems; ++i)
        if (base + i < n) {
            out[base + i] = run;
            run += v[i];
        }
}

void launch_exclusive_scan(const unsigned* in, unsigned* out, long long n, unsigned* part, unsigned* total,
                           cudaStream_t st) {
    if (n <= 0) return;
    const int nb = static_cast<int>((n + kScanTile - 1) / kScanTile);
    k_scan_partials<<<nb, kScanThreads, 0, st>>>(in, n, part); ++g_launches;
    k_scan_top<<<1, kScanThreads, 0, st>>>(part, nb, total); ++g_launches;
    k_scan_apply<<<nb, kScanThreads, 0, st>>>(in, n, part, out); ++g_launches;
}

long long scan_scratch(long long n) { return (n + kScanTile - 1) / kScanTile + 1; }

// One stable LSD pass over 8 key bits starting at `shift`.
template <typename K>
void radix_pass(const K* kin, const unsigned* vin, K* kout, unsigned* vout, long long n, int shift,
                unsigned* hist, unsigned* part, cudaStream_t st, const unsigned long long* pin = nullptr,
                unsigned long long* pout = nullptr) {
    const int nb = static_cast<int>((n + kRadixTile - 1) / kRadixTile);
    k_radix_hist<K><<<nb, kRadixThreads, 0, st>>>(kin, n, shift, hist, nb); ++g_launches;
    launch_exclusive_scan(hist, hist, 256ll * nb, part, nullptr, st);
    const size_t smem = (sizeof(K) + sizeof(unsigned) + (pin ? sizeof(unsigned long long) : 0)) * kRadixTile;
    cudaFuncSetAttribute(k_radix_scatter<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>((sizeof(K) + sizeof(unsigned) + sizeof(unsigned long long)) * kRadixTile));
    k_radix_scatter<K><<<nb, kRadixThreads, smem, st>>>(kin, vin, kout, vout, n, shift, hist, nb, pin, pout);
    ++g_launches;
}

// A u32-key pass that also carries a 64-bit payload (the depth keys through the view pass).
void radix_pass_kv(const unsigned* kin, const unsigned* vin, const unsigned long long* pin, unsigned* kout,
                   unsigned* vout, unsigned long long* pout, long long n, int shift, unsigned* hist, unsigned* part,
                   cudaStream_t st) {
    radix_pass<unsigned>(kin, vin, kout, vout, n, shift, hist, part, st, pin, pout);
}

long long radix_hist_size(long long n) { return 256ll * ((n + kRadixTile - 1) / kRadixTile); }

// ---- tile-list construction kernels
// Sort keys for the depth passes: index order, culled / padding Gaussians get
// key 0 and produce no entries (their position is irrelevant).
__global__ void k_depth_init(const unsigned long long* __restrict__ keys, const short4* __restrict__ rect, int G,
                             int Gp, long long n, unsigned long long* __restrict__ kout, unsigned* __restrict__ vout,
                             unsigned long long* __restrict__ and_or) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    bool valid = false;
    unsigned long long k = 0ull;
    if (i < n) {
        const int g = static_cast<int>(i % Gp);
        valid = g < G && rect[i].x <= rect[i].y;
        k = valid ? keys[i] : 0ull;
        kout[i] = k;
        vout[i] = static_cast<unsigned>(i);
    }
    // AND / OR of the valid keys: bytes where they agree need no pass
    __shared__ unsigned long long s_a[32], s_o[32];
    unsigned long long a = valid ? k : ~0ull, o = valid ? k : 0ull;
#pragma unroll
    for (int s = 16; s; s >>= 1) {
        a &= __shfl_xor_sync(0xffffffffu, a, s);
        o |= __shfl_xor_sync(0xffffffffu, o, s);
    }
    if ((threadIdx.x & 31) == 0) {
        s_a[threadIdx.x >> 5] = a;
        s_o[threadIdx.x >> 5] = o;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
            a &= s_a[w];
            o |= s_o[w];
        }
        if (a != ~0ull) atomicAnd(&and_or[0], a);
        if (o != 0ull) atomicOr(&and_or[1], o);
    }
}

void launch_depth_init(const unsigned long long* keys, const short4* rect, int G, int Gp, int V,
                       unsigned long long* kout, unsigned* vout, unsigned long long* and_or, cudaStream_t st) {
    const long long n = static_cast<long long>(V) * Gp;
    if (n == 0) return;
    const unsigned long long init[2] = {~0ull, 0ull};
    cudaMemcpyAsync(and_or, init, sizeof init, cudaMemcpyHostToDevice, st);
    k_depth_init<<<static_cast<unsigned>((n + 1023) / 1024), 1024, 0, st>>>(keys, rect, G, Gp, n, kout, vout, and_or); ++g_launches;
}

// After the passes over the key's upper 32 bits: runs of equal upper halves
// (depths within a relative 2^-20 -- a few per cent of the Gaussians, runs of
// 2-3) are put in (full key, index) order by the thread at each run start:
// insertion sort, heapsort for a (pathological) long run.  Key 0 marks culled
// Gaussians (valid keys have the top bit set); their order is irrelevant.
__device__ __forceinline__ bool kv_less(unsigned long long ka, unsigned va, unsigned long long kb, unsigned vb) {
    return ka < kb || (ka == kb && va < vb);
}

__device__ void heap_sift(unsigned long long* k, unsigned* v, long long root, long long len) {
    while (true) {
        long long c = 2 * root + 1;
        if (c >= len) return;
        if (c + 1 < len && kv_less(k[c], v[c], k[c + 1], v[c + 1])) ++c;
        if (!kv_less(k[root], v[root], k[c], v[c])) return;
        const unsigned long long tk = k[root];
        const unsigned tv = v[root];
        k[root] = k[c];
        v[root] = v[c];
        k[c] = tk;
        v[c] = tv;
        root = c;
    }
}

// Runs are maximal stretches of equal (view, upper key half); after the view
// pass only same-view keys can share a run (ties across views never matter).
// Runs of <= 32 are insertion-sorted by the thread at their start; longer ones
// (near-planar scenes: many depths within 2^-20 of each other) are queued for
// k_sort_long_runs, one CTA per run, so no run is ever sorted by one thread.
constexpr int kShortRun = 32;
__global__ void k_fix_runs(unsigned long long* __restrict__ keys, unsigned* __restrict__ vals, long long n,
                           unsigned Gp, unsigned long long* __restrict__ runs, long long max_runs) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned hi = static_cast<unsigned>(keys[i] >> 32);
    if (hi == 0u) return;  // culled
    const unsigned view = vals[i] / Gp;
    auto same = [&](long long j) { return static_cast<unsigned>(keys[j] >> 32) == hi && vals[j] / Gp == view; };
    if (i > 0 && same(i - 1)) return;  // not a run start
    long long e = i + 1;
    while (e < n && same(e)) ++e;
    const long long len = e - i;
    if (len <= 1) return;
    unsigned long long* k = keys + i;
    unsigned* v = vals + i;
    if (len > kShortRun && runs) {
        const unsigned long long q = atomicAdd(runs, 1ull);
        if (static_cast<long long>(q) < max_runs) {
            runs[1 + 2 * q] = static_cast<unsigned long long>(i);
            runs[2 + 2 * q] = static_cast<unsigned long long>(len);
            return;
        }
    }
    if (len <= kShortRun) {
        for (long long a = 1; a < len; ++a) {  // insertion sort by (key, index)
            const unsigned long long ka = k[a];
            const unsigned va = v[a];
            long long b = a - 1;
            while (b >= 0 && kv_less(ka, va, k[b], v[b])) {
                k[b + 1] = k[b];
                v[b + 1] = v[b];
                --b;
            }
            k[b + 1] = ka;
            v[b + 1] = va;
        }
        return;
    }
    for (long long r = len / 2 - 1; r >= 0; --r) heap_sift(k, v, r, len);
    for (long long end = len - 1; end > 0; --end) {
        const unsigned long long tk = k[0];
        const unsigned tv = v[0];
        k[0] = k[end];
        v[0] = v[end];
        k[end] = tk;
        v[end] = tv;
        heap_sift(k, v, 0, end);
    }
}

// One CTA per long run (grid-stride over the queue): chunks of 2048 (key, index)
// pairs bitonic-sorted in shared memory, then merged pairwise (merge path,
// 256 threads) between the run's slice of the keys/vals and the scratch.
constexpr int kLongChunk = 2048;
constexpr int kLongThreads = 256;

__device__ __forceinline__ bool kv_less2(unsigned long long ka, unsigned va, unsigned long long kb, unsigned vb) {
    return ka < kb || (ka == kb && va < vb);
}

__global__ void __launch_bounds__(kLongThreads) k_sort_long_runs(unsigned long long* __restrict__ keys,
                                                                 unsigned* __restrict__ vals,
                                                                 const unsigned long long* __restrict__ runs,
                                                                 long long max_runs,
                                                                 unsigned long long* __restrict__ tk,
                                                                 unsigned* __restrict__ tv) {
    __shared__ unsigned long long sk[kLongChunk];
    __shared__ unsigned sv[kLongChunk];
    const long long count = min(static_cast<long long>(runs[0]), max_runs);
    const int t = threadIdx.x;
    for (long long r = blockIdx.x; r < count; r += gridDim.x) {
        const long long s = static_cast<long long>(runs[1 + 2 * r]), L = static_cast<long long>(runs[2 + 2 * r]);
        unsigned long long* K = keys + s;
        unsigned* Vv = vals + s;
        // 1. sorted chunks
        for (long long c0 = 0; c0 < L; c0 += kLongChunk) {
            const int m = static_cast<int>(min(static_cast<long long>(kLongChunk), L - c0));
            for (int i = t; i < kLongChunk; i += kLongThreads) {
                sk[i] = i < m ? K[c0 + i] : ~0ull;
                sv[i] = i < m ? Vv[c0 + i] : ~0u;
            }
            __syncthreads();
            for (int k = 2; k <= kLongChunk; k <<= 1)
                for (int j = k >> 1; j > 0; j >>= 1) {
                    for (int i = t; i < kLongChunk; i += kLongThreads) {
                        const int ixj = i ^ j;
                        if (ixj > i) {
                            const bool up = (i & k) == 0;
                            const bool gt = kv_less2(sk[ixj], sv[ixj], sk[i], sv[i]);
                            if (gt == up) {
                                const unsigned long long a = sk[i];
                                const unsigned b = sv[i];
                                sk[i] = sk[ixj];
                                sv[i] = sv[ixj];
                                sk[ixj] = a;
                                sv[ixj] = b;
                            }
                        }
                    }
                    __syncthreads();
                }
            for (int i = t; i < m; i += kLongThreads) {
                K[c0 + i] = sk[i];
                Vv[c0 + i] = sv[i];
            }
            __syncthreads();
        }
        // 2. merge passes, ping-ponging between the run and the scratch
        unsigned long long *srck = K, *dstk = tk + s;
        unsigned *srcv = Vv, *dstv = tv + s;
        for (long long w = kLongChunk; w < L; w <<= 1) {
            for (long long a = 0; a < L; a += 2 * w) {
                const long long na = min(w, L - a), nb = max(0ll, min(w, L - a - w));
                const long long total = na + nb;
                const unsigned long long* Ak = srck + a;
                const unsigned* Av = srcv + a;
                const unsigned long long* Bk = srck + a + na;
                const unsigned* Bv = srcv + a + na;
                // this thread's output range [d0, d1) and its merge-path split points
                const long long d0 = total * t / kLongThreads, d1 = total * (t + 1) / kLongThreads;
                auto split = [&](long long d) {  // A elements among the first d outputs
                    long long lo = max(0ll, d - nb), hi = min(d, na);
                    while (lo < hi) {
                        const long long mid = (lo + hi) >> 1;
                        if (kv_less2(Ak[mid], Av[mid], Bk[d - mid - 1], Bv[d - mid - 1])) lo = mid + 1;
                        else hi = mid;
                    }
                    return lo;
                };
                long long ia = split(d0), ib = d0 - ia;
                for (long long d = d0; d < d1; ++d) {
                    const bool takeA = ib >= nb || (ia < na && kv_less2(Ak[ia], Av[ia], Bk[ib], Bv[ib]));
                    if (takeA) {
                        dstk[a + d] = Ak[ia];
                        dstv[a + d] = Av[ia];
                        ++ia;
                    } else {
                        dstk[a + d] = Bk[ib];
                        dstv[a + d] = Bv[ib];
                        ++ib;
                    }
                }
            }
            __syncthreads();
            unsigned long long* x = srck;
            srck = dstk;
            dstk = x;
            unsigned* y = srcv;
            srcv = dstv;
            dstv = y;
        }
        if (srck != K)
            for (long long i = t; i < L; i += kLongThreads) {
                K[i] = srck[i];
                Vv[i] = srcv[i];
            }
        __syncthreads();
    }
}

__global__ void k_view_key(const unsigned* __restrict__ vals, long long n, int Gp, unsigned* __restrict__ vkey) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) vkey[i] = vals[i] / static_cast<unsigned>(Gp);
}

__global__ void k_emit_count(const unsigned* __restrict__ order, long long n, int G, int Gp,
                             const short4* __restrict__ rect, unsigned* __restrict__ count) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned vg = order[i];
    const int g = static_cast<int>(vg % static_cast<unsigned>(Gp));
    unsigned c = 0u;
    if (g < G) {
        const short4 r = rect[vg];
        if (r.x <= r.y) c = static_cast<unsigned>(r.y - r.x + 1) * static_cast<unsigned>(r.w - r.z + 1);
    }
    count[i] = c;
}

// The block's 256 consecutive (view, Gaussian)s own one contiguous output
// range; their pairs are staged in shared memory and written out coalesced
// (pairs past the staging capacity go straight to global memory).
constexpr int kEmitStage = 4096;

__global__ void __launch_bounds__(256) k_emit(const unsigned* __restrict__ order, long long n, int G, int Gp,
                                              const DevCam* __restrict__ cams, const short4* __restrict__ rect,
                                              const unsigned* __restrict__ start, long long n_entries,
                                              unsigned* __restrict__ tkey, unsigned* __restrict__ tval) {
    __shared__ unsigned s_key[kEmitStage], s_val[kEmitStage];
    __shared__ unsigned s_lo, s_hi;
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long first = static_cast<long long>(blockIdx.x) * blockDim.x;
    const long long lastp1 = first + blockDim.x < n ? first + blockDim.x : n;
    if (threadIdx.x == 0) {
        s_lo = start[first];
        s_hi = lastp1 < n ? start[lastp1] : static_cast<unsigned>(n_entries);
    }
    __syncthreads();
    const unsigned lo = s_lo, hi = s_hi;
    if (i < n) {
        const unsigned vg = order[i];
        const int v = static_cast<int>(vg / static_cast<unsigned>(Gp)), g = static_cast<int>(vg % static_cast<unsigned>(Gp));
        if (g < G) {
            const short4 r = rect[vg];
            if (r.x <= r.y) {
                const int base = cams[v].tile_base, tx_n = cams[v].tiles_x;
                unsigned o = start[i];
                for (int ty = r.z; ty <= r.w; ++ty)
                    for (int tx = r.x; tx <= r.y; ++tx, ++o) {
                        const unsigned key = static_cast<unsigned>(base + ty * tx_n + tx);
                        if (o - lo < static_cast<unsigned>(kEmitStage)) {
                            s_key[o - lo] = key;
                            s_val[o - lo] = static_cast<unsigned>(g);
                        } else {
                            tkey[o] = key;
                            tval[o] = static_cast<unsigned>(g);
                        }
                    }
            }
        }
    }
    __syncthreads();
    const unsigned m = min(hi - lo, static_cast<unsigned>(kEmitStage));
    for (unsigned j = threadIdx.x; j < m; j += blockDim.x) {
        tkey[lo + j] = s_key[j];
        tval[lo + j] = s_val[j];
    }
}

// Host driver (runtime.cpp keeps the buffers).  Returns nothing; `entries`
// receives the per-tile sorted lists; tile_offsets (n_tiles + 1) their CSR offsets.
// CSR offsets from the sorted tile ids: offsets[t] = first entry with tile >= t.
__global__ void k_tile_offsets(const unsigned* __restrict__ tiles, long long n, int n_tiles, int* __restrict__ offsets) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > n_tiles) return;
    long long lo = 0, hi = n;
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (tiles[mid] < static_cast<unsigned>(t)) lo = mid + 1;
        else hi = mid;
    }
    offsets[t] = static_cast<int>(lo);
}

void build_tile_lists(const unsigned long long* keys, const short4* rect, const DevCam* cams, int G, int Gp, int V,
                      int n_tiles, long long n_entries, unsigned long long and_k, unsigned long long or_k,
                      const TileSortBuffers& b, int* entries, int* tile_offsets, cudaStream_t st) {
    const long long n = static_cast<long long>(V) * Gp;
    if (n == 0 || n_entries == 0) {
        cudaMemsetAsync(tile_offsets, 0, sizeof(int) * (n_tiles + 1), st);
        return;
    }
    // 1. depth passes over the varying key bytes, then the view
    const unsigned long long vary = and_k ^ or_k;
    unsigned long long *ka = b.k64a, *kb = b.k64b;
    unsigned *va = b.v32a, *vb = b.v32b;
    // LSD passes over the varying bytes of the upper 32 bits, then a run fix-up
    // for the (rare, short) runs of equal upper halves
    for (int byte = 4; byte < 8; ++byte) {
        if (((vary >> (8 * byte)) & 0xFFull) == 0ull) continue;
        radix_pass<unsigned long long>(ka, va, kb, vb, n, 8 * byte, b.hist, b.part, st);
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    // then by view (not needed for the order -- a tile's entries belong to one
    // view -- but the view-major emit keeps the tile passes' scatter local: measured
    // 0.4 ms faster per batch at configs[2]); the 64-bit keys ride along so the
    // run fix-up below only sees same-view runs
    if (V > 1) {
        k_view_key<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(va, n, Gp, b.k32a); ++g_launches;
        unsigned *k32a = b.k32a, *k32b = b.k32b;
        for (int s = 0; (1ll << s) < V; s += 8) {
            radix_pass_kv(k32a, va, ka, k32b, vb, kb, n, s, b.hist, b.part, st);
            std::swap(k32a, k32b);
            std::swap(va, vb);
            std::swap(ka, kb);
        }
    }
    if (vary & 0xFFFFFFFFull) {
        const long long max_runs = n / (kShortRun + 1) + 1;
        cudaMemsetAsync(b.runs, 0, sizeof(unsigned long long), st);
        k_fix_runs<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(ka, va, n, static_cast<unsigned>(Gp), b.runs,
                                                                           max_runs);
        ++g_launches;
        k_sort_long_runs<<<148, kLongThreads, 0, st>>>(ka, va, b.runs, max_runs, kb, vb);
        ++g_launches;
    }
    // 2. emit (tile, index) pairs in (view, depth, index) order
    k_emit_count<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(va, n, G, Gp, rect, b.count); ++g_launches;
    launch_exclusive_scan(b.count, b.count, n, b.part, nullptr, st);
    unsigned *tka = b.t32a, *tkb = b.t32b, *tva = b.t32va, *tvb = b.t32vb;
    k_emit<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(va, n, G, Gp, cams, rect, b.count, n_entries, tka,
                                                                    tva);
    ++g_launches;
    // 3. stable sort by tile id; the last pass writes the values into `entries`
    int passes = 0;
    for (int s = 0; (1ll << s) < n_tiles; s += 8) ++passes;
    for (int p = 0; p < passes; ++p) {
        const bool last = p == passes - 1;
        radix_pass<unsigned>(tka, tva, tkb, last ? reinterpret_cast<unsigned*>(entries) : tvb, n_entries, 8 * p,
                             b.hist, b.part, st);
        std::swap(tka, tkb);
        std::swap(tva, tvb);
    }
    if (passes == 0)  // a single tile: already in order
        cudaMemcpyAsync(entries, tva, sizeof(unsigned) * n_entries, cudaMemcpyDeviceToDevice, st);
    k_tile_offsets<<<(n_tiles + 1 + 255) / 256, 256, 0, st>>>(tka, n_entries, n_tiles, tile_offsets); ++g_launches;
}

// ---- deterministic accumulation order (DetOrder, layout.hpp)
// Slot keys: slot 32 * wbase[g] + j of group g holds compacted entry j; its key
// is the (view, Gaussian) it accumulates into, the window padding sorts last.
__global__ void __launch_bounds__(128) k_slot_keys(const Group* __restrict__ groups, int n_groups,
                                                   const int* __restrict__ gcount, const int* __restrict__ glist,
                                                   const long long* __restrict__ mask_off,
                                                   const long long* __restrict__ wbase, int Gp, unsigned sentinel,
                                                   unsigned* __restrict__ key, unsigned* __restrict__ val) {
    const int gi = blockIdx.x * 4 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (gi >= n_groups) return;
    const int nun = gcount[gi];
    const int n = 32 * ((nun + 31) >> 5);
    const long long s0 = 32 * wbase[gi], off = mask_off[gi];
    const unsigned vb = static_cast<unsigned>(groups[gi].view) * static_cast<unsigned>(Gp);
    for (int j = lane; j < n; j += 32) {
        key[s0 + j] = j < nun ? vb + static_cast<unsigned>(glist[off + j]) : sentinel;
        val[s0 + j] = static_cast<unsigned>(s0 + j);
    }
}

__global__ void k_count_keys(const unsigned* __restrict__ keys, long long n, long long n_keys,
                             unsigned* __restrict__ count) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n && keys[i] < static_cast<unsigned>(n_keys)) atomicAdd(count + keys[i], 1u);
}

// seg[k] = first sorted slot with key >= k, k in [0, n_keys]
__global__ void k_seg_bounds(const unsigned* __restrict__ keys, long long n, long long n_keys,
                             unsigned* __restrict__ seg) {
    const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k > n_keys) return;
    long long lo = 0, hi = n;
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (keys[mid] < static_cast<unsigned>(k)) lo = mid + 1;
        else hi = mid;
    }
    seg[k] = static_cast<unsigned>(lo);
}

__global__ void k_invert_perm(const unsigned* __restrict__ perm, long long n, unsigned* __restrict__ dest) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) dest[perm[i]] = static_cast<unsigned>(i);
}

// Longest per-key slot count (the counting path's guard).
constexpr unsigned kMaxSortedSegment = 64;
__global__ void k_max_count(const unsigned* __restrict__ count, long long n, unsigned* __restrict__ out) {
    unsigned m = 0u;
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        m = max(m, count[i]);
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

// Counting placement: slot i goes to seg[key] + (an atomic ticket of its key),
// so each key's segment holds its slots in arbitrary order ...
__global__ void k_place_slots(const unsigned* __restrict__ keys, long long n, long long n_keys,
                              const unsigned* __restrict__ seg, unsigned* __restrict__ fill,
                              unsigned* __restrict__ perm, unsigned* __restrict__ dest) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned k = keys[i];
    if (k < static_cast<unsigned>(n_keys)) {
        const unsigned pos = seg[k] + atomicAdd(fill + k, 1u);
        perm[pos] = static_cast<unsigned>(i);
        dest[i] = pos;  // coalesced; rewritten below only where the segment needed sorting
    }
}

// ... which one thread per key then puts in ascending slot order (insertion
// sort: segments hold a few slots -- the number of the plan's groups in which
// some sample blends the (view, Gaussian)) and inverts into dest.  The result
// is exactly the stable sort's: within a key, ascending slot index.
__global__ void k_sort_segments(const unsigned* __restrict__ seg, long long n_keys, unsigned* __restrict__ perm,
                                unsigned* __restrict__ dest) {
    const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n_keys) return;
    const unsigned a = seg[k], b = seg[k + 1];
    bool sorted = true;
    for (unsigned j = a + 1; j < b && sorted; ++j) sorted = perm[j - 1] < perm[j];
    if (sorted) return;  // the placement order already ascends; dest is right
    for (unsigned j = a + 1; j < b; ++j) {
        const unsigned x = perm[j];
        unsigned q = j;
        while (q > a && perm[q - 1] > x) {
            perm[q] = perm[q - 1];
            --q;
        }
        perm[q] = x;
    }
    for (unsigned j = a; j < b; ++j) dest[perm[j]] = j;
}

// dest (n_slots) and seg (V * Gp + 1) of a plan: within each key (view * Gp +
// Gaussian) the slots in ascending order, seg the keys' first positions, dest
// the inverse.  `fill` (n_keys) is scratch.  (Round 2 ran three stable radix
// passes over the keys; the counting placement + segment sort gives the same
// order in three light passes.)
void build_slot_order(const Group* groups, int n_groups, const int* gcount, const int* glist,
                      const long long* mask_off, const long long* wbase, int Gp, int V, long long n_slots,
                      unsigned* ka, unsigned* kb, unsigned* va, unsigned* vb, unsigned* hist, unsigned* part,
                      unsigned* perm, unsigned* seg, unsigned* dest, unsigned* fill, cudaStream_t st) {
    const long long n_keys = static_cast<long long>(V) * Gp;
    if (n_slots == 0) {
        cudaMemsetAsync(seg, 0, sizeof(unsigned) * (n_keys + 1), st);
        return;
    }
    const unsigned sentinel = static_cast<unsigned>(n_keys);
    static const bool prof = std::getenv("SLM_SORT_PROF") && std::getenv("SLM_SORT_PROF")[0] == '1';
    cudaEvent_t pev[12];
    const char* pname[12];
    int np = 0;
    auto pmark = [&](const char* name) {
        if (!prof) return;
        cudaEventCreate(&pev[np]);
        cudaEventRecord(pev[np], st);
        pname[np++] = name;
    };
    auto pdump = [&]() {
        if (!prof) return;
        cudaEventSynchronize(pev[np - 1]);
        std::fprintf(stderr, "[slots] n=%lld keys=%lld:", n_slots, n_keys);
        for (int q = 1; q < np; ++q) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, pev[q - 1], pev[q]);
            std::fprintf(stderr, " %s %.3f", pname[q], ms);
        }
        std::fprintf(stderr, "\n");
        for (int q = 0; q < np; ++q) cudaEventDestroy(pev[q]);
    };
    pmark("start");
    k_slot_keys<<<(n_groups + 3) / 4, 128, 0, st>>>(groups, n_groups, gcount, glist, mask_off, wbase, Gp, sentinel,
                                                    ka, va);
    ++g_launches;
    pmark("keys");
    if (fill) {
        cudaMemsetAsync(seg, 0, sizeof(unsigned) * (n_keys + 1), st);
        cudaMemsetAsync(fill, 0, sizeof(unsigned), st);
        k_count_keys<<<static_cast<unsigned>((n_slots + 255) / 256), 256, 0, st>>>(ka, n_slots, n_keys, seg);
        ++g_launches;
        // the per-key segment sort is serial: a key with many slots (one splat
        // blended in many of the plan's groups) takes the radix passes instead
        k_max_count<<<static_cast<unsigned>(std::min<long long>((n_keys + 255) / 256, 1184)), 256, 0, st>>>(seg, n_keys,
                                                                                                            fill);
        ++g_launches;
        unsigned longest = 0;
        cudaMemcpyAsync(&longest, fill, sizeof(unsigned), cudaMemcpyDeviceToHost, st);
        pmark("count+max");
        cudaStreamSynchronize(st);
        if (longest <= kMaxSortedSegment) {
            cudaMemsetAsync(fill, 0, sizeof(unsigned) * n_keys, st);
            pmark("sync+memset");
            launch_exclusive_scan(seg, seg, n_keys, part, seg + n_keys, st);
            pmark("scan");
        k_place_slots<<<static_cast<unsigned>((n_slots + 255) / 256), 256, 0, st>>>(ka, n_slots, n_keys, seg, fill,
                                                                                     perm, dest);
        ++g_launches;
            pmark("place");
            k_sort_segments<<<static_cast<unsigned>((n_keys + 255) / 256), 256, 0, st>>>(seg, n_keys, perm, dest);
            ++g_launches;
            pmark("sort");
            pdump();
            return;
        }
    }
    int bits = 0;
    while ((1ull << bits) <= sentinel) ++bits;
    const int passes = (bits + 7) / 8;
    for (int p = 0; p < passes; ++p) {
        const bool last = p == passes - 1;
        radix_pass<unsigned>(ka, va, kb, last ? perm : vb, n_slots, 8 * p, hist, part, st);
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    // seg = exclusive scan of the per-key slot counts (integer atomics: exact)
    cudaMemsetAsync(seg, 0, sizeof(unsigned) * (n_keys + 1), st);
    k_count_keys<<<static_cast<unsigned>((n_slots + 255) / 256), 256, 0, st>>>(ka, n_slots, n_keys, seg);
    ++g_launches;
    launch_exclusive_scan(seg, seg, n_keys, part, seg + n_keys, st);
    k_invert_perm<<<static_cast<unsigned>((n_slots + 255) / 256), 256, 0, st>>>(perm, n_slots, dest);
    ++g_launches;
}

}  // namespace slm
