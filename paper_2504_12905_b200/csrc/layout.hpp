// layout.hpp — POD types and constants shared by host (runtime.cpp, g++) and
// device (*.cu, nvcc) code.  See common.cuh for the HBM layout notes.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "slm_types.h"

namespace slm {

constexpr int kTile = 16;               // rasterizer.hpp:14
constexpr int kP = 14;                  // types.hpp:20
constexpr int kRec = 12;                // floats per splat / tangent / inter record
constexpr int kDiagRec = 20;            // floats per diag accumulator record (19 used)
constexpr double kAlphaClampD = 0.99;   // rasterizer.hpp:15
constexpr double kAlphaSkipD = 1.0 / 255.0;
constexpr double kTFloorD = 1e-4;       // rasterizer.hpp:17
constexpr double kColorC0 = 0.28209479177387814;  // types.hpp:24
constexpr double kLog2e = 1.4426950408889634074;
constexpr double kLn2 = 0.69314718055994530942;

// Device-side camera (slm_camera minus nothing): passed by value in kernel
// params or staged in __constant__/smem.
struct DevCam {
    double R[9];
    double t[3];
    double fx, fy, cx, cy, near_clip;
    int width, height;
    int tiles_x, tiles_y;
    int tile_base;   // first tile of this view in the batch-concatenated tile arrays
    int pad0;
    long long pix_base;  // first pixel of this view in the concatenated pixel arrays
};

// A unit of sampled-raster work: up to 32 samples of one tile of one view.
struct Group {
    int view;
    int tile;       // tile index within the view
    int begin;      // first sample (group order) of this group
    int count;      // 1..32
};

struct SampleArgs {
    const Group* groups;
    int n_groups;
    const DevCam* cams;
    const int* tile_offsets;
    const int* entries;
    const float4* rec;
    const float4* tan;
    int Gp;
    const int* spix;   // px | py << 16, group order
    const int* sorig;  // original sample index (plan order)
    const float* sw;   // per-sample per-channel weights, group order [3*s+c]
    const float* image;
    const int* last_img;
    const float* gt;
    const float* in_res;  // VJP: u in plan order [3*orig+c]
    float* out_res;       // JVP: Jv in plan order
    float* inter;         // J^T accumulators [(v*Gp+g)*12 + i]
    const int* done_flag; // optional: skip all work when *done_flag != 0 (PCG converged)
    // Per-group compacted window stream (k_masks, once per state/plan): the
    // group's tile-list entries that at least one of its pixels blends, in
    // list order, and per 32-entry window one blend bitmask per lane.
    const unsigned* masks;      // [mask_off[g] + 32*w + lane], bit k = entry 32w+k blended
    const int* glist;           // [mask_off[g] + j] = Gaussian index of compacted entry j
    const int* gcount;          // [g] = compacted entries of the group
    const long long* mask_off;  // per-group offset into masks / glist (32*ceil(list/32))
    unsigned* masks_out;        // k_masks outputs (same buffers)
    int* glist_out;
    int* gcount_out;
    int* grows_out;             // k_masks: alpha-stream rows of the group (sum_w max_lane popc)
    // Per-pair alpha stream (k_alpha, once per state/plan): window w of group g
    // owns rows [srow_off[g] + r_w, + max_lane popc), row i = the lanes' i-th
    // blended entry of the window, 32 floats (lane order); value = alpha, negated
    // when alpha was clamped at 0.99 (frozen derivative).
    const long long* srow_off;
    const float* astream;
    float* astream_out;
    // Per-window record blocks (k_alpha, once per state/plan): window w of group g
    // holds its 32 entries' state-only splat fields as [9][32] floats
    // (mx, my, A, B, C, o, r, g, b) at rstream[kRecBlock * (wbase[g] + w)].
    const long long* wbase;
    const float* rstream;
    float* rstream_out;
    // Per-window column masks (k_alpha, once per state/plan), same indexing as
    // masks: lane k's word = the pixels that blend compacted entry k.
    const unsigned* cols;
    unsigned* cols_out;
    // Exact blend decisions (k_masks): the FP64 geometry per (view, Gaussian)
    // [mx, my, a, b, c, o] and, per sample (group order), the final colour of
    // the reference's FP64 blend, which the J^T passes use as C_final.
    const double* rec64;
    const float* scol;
    float* scol_out;
    // Deterministic accumulation (the default): instead of red.global.add into
    // `inter`, the J^T pass writes each compacted entry's 9-float contribution
    // (slot = 32 * wbase[g] + j) as one record at position dest[slot] of
    // `partial`; the chain kernel sums a (view, Gaussian)'s records in order
    // (DetOrder).
    const unsigned* dest;
    float* partial;
};

constexpr int kDetRec = 12;      // floats per J^T partial record (9 used)
constexpr int kDetDiagRec = 24;  // floats per diag partial record (19 used): three full sectors

// Per-plan order of the deterministic accumulation (sort.cu build_slot_order):
// the slots sorted by (view * Gp + Gaussian), stable (slot order within a
// key); dest[slot] = the slot's position in that order, so the partial
// records of (view, Gaussian) vg are the contiguous range [seg[vg], seg[vg+1])
// and are summed front to back.  Fixed per plan -> every product rounds the
// same way.
struct DetOrder {
    const unsigned* seg;
    const float* partial;  // kDetRec floats per record (J^T) or kDetDiagRec (diag)
    // 1: the chain kernel's thread sums its (view, Gaussian)'s records itself
    //    (few records per key, many Gaussians: configs[2]);
    // 0: k_det_reduce first sums every key's records with a warp-segmented
    //    reduction (parallel over records: many records per key / few
    //    Gaussians, configs[0]) into inter / diagacc, which the chain reads.
    int fused;
};

constexpr int kRecBlock = 9 * 32;  // floats per window record block (1152 B)

struct DiagArgs {
    const Group* groups;
    int n_groups;
    const DevCam* cams;
    const int* tile_offsets;
    const int* entries;
    const float4* rec;
    int Gp;
    const int* spix;
    const float* sw;
    const float* image;
    const int* last_img;
    float* diagacc;
    const unsigned* masks;
    const int* glist;
    const int* gcount;
    const long long* mask_off;
    const unsigned* cols;  // column masks (SampleArgs::cols)
    const float* scol;     // per-sample final colour (SampleArgs::scol)
    const long long* wbase;  // deterministic mode: slot base per group (SampleArgs::wbase)
    const unsigned* dest;    // deterministic mode: record position per slot (SampleArgs::dest)
    float* partial;          // deterministic mode: kDetDiagRec floats per record
};

// Scratch of the radix tile-list construction (sort.cu), sized by the runtime:
// n = V*Gp (k64*, v32*, k32*, count), E = tile-list entries (t32*),
// hist = 256 * ceil(max(n, E) / 4096), part = scan partials.
struct TileSortBuffers {
    unsigned long long *k64a, *k64b;
    unsigned *v32a, *v32b, *k32a, *k32b, *count;
    unsigned *t32a, *t32b, *t32va, *t32vb;
    unsigned *hist, *part;
    unsigned long long* runs;  // long equal-depth runs queued by k_fix_runs: [count, (start, len) ...]
};

struct CgState {
    double rz, pu, alpha, beta, rr, bnorm;
    int iterations, breakdown, done, pad;
};

enum Mode { kJvp = 0, kVjp = 1, kGn = 2, kRhs = 3 };

// One image of a metrics launch (metrics.cu): interleaved RGB at elements
// [off, off + 3*w*h), its 32x32 output tiles at partial[tile_base, +tiles).
struct ImgDesc {
    long long off;
    int w, h, tiles_x, tiles, tile_base;
};
constexpr int kMetricWin = 11;  // image_metrics.cpp:14
struct MetricWindow {
    double w[kMetricWin];
};

// One first-order step (first_order.cu): per-row learning rates (group rate,
// mean rows already scaled by the decay factor), and the kind's constants:
// Adam b1/b2/eps + bias corrections c1/c2, RMSprop b2 = decay, SGD b1 = momentum.
struct FirstOrderParams {
    int kind;
    double lr[kP];
    double b1, b2, eps, c1, c2;
};

constexpr int kRedBlocks = 592;  // 4 x 148 SMs
constexpr int kRedThreads = 256;

}  // namespace slm
