/*
 * splat_oracle.c — TEST INFRASTRUCTURE ONLY (see splat_oracle.h).
 *
 * Plain-C, single-threaded restatement of the reference LM/PCG hot path.
 * All double arithmetic follows the reference operation order and is
 * compiled with -ffp-contract=off (oracle/Makefile) like the reference
 * (proj/src/CMakeLists.txt:23-25), so value parts reproduce the reference
 * bit for bit; reductions that the reference runs through AVX2 kernels
 * (dot/sum_squares in pcg) use plain left-to-right sums here and agree to
 * rounding only.
 *
 * Every function cites the reference file:line it restates; paths are
 * relative to /root/reference/proj.
 */
#include "splat_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ errors */
static char g_err[512];
static int set_err(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}
enum { E_INVALID = 1, E_DOMAIN = 2, E_RUNTIME = 3 };

const char* orc_last_error(void) { return g_err; }
void orc_set_threads(int n) { (void)n; }
int orc_threads(void) { return 1; }

/* ------------------------------------------- std::mt19937_64 (C++11 26.5.3.2) */
typedef struct {
    uint64_t mt[312];
    int idx;
} rng64;

static void rng_seed(rng64* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = 312;
}

static uint64_t rng_next(rng64* r) {
    if (r->idx >= 312) {
        const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
        for (int i = 0; i < 312; ++i) {
            const uint64_t y = (r->mt[i] & upper) | (r->mt[(i + 1) % 312] & lower);
            r->mt[i] = r->mt[(i + 156) % 312] ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
        }
        r->idx = 0;
    }
    uint64_t z = r->mt[r->idx++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}

void* orc_rng_new(uint64_t seed) {
    rng64* r = (rng64*)malloc(sizeof(rng64));
    rng_seed(r, seed);
    return r;
}
void orc_rng_free(void* r) { free(r); }
uint64_t orc_rng_next(void* r) { return rng_next((rng64*)r); }

/* libstdc++-13 uniform_int_distribution with a 64-bit engine: Lemire's
 * nearly divisionless downscaling over unsigned __int128
 * (/usr/include/c++/13/bits/uniform_int_dist.h:256-281,305-319). */
static uint64_t uniform_u64(rng64* r, uint64_t a, uint64_t b) {
    const uint64_t urange = b - a;
    if (urange == UINT64_MAX) return rng_next(r) + a;
    const uint64_t range = urange + 1;
    unsigned __int128 product = (unsigned __int128)rng_next(r) * range;
    uint64_t low = (uint64_t)product;
    if (low < range) {
        const uint64_t threshold = (0 - range) % range;
        while (low < threshold) {
            product = (unsigned __int128)rng_next(r) * range;
            low = (uint64_t)product;
        }
    }
    return (uint64_t)(product >> 64) + a;
}
static int uniform_int(rng64* r, int a, int b) {
    return (int)uniform_u64(r, (uint64_t)(int64_t)a, (uint64_t)(int64_t)b);
}

/* generate_canonical<double,53> with one 64-bit draw (random.tcc:3349-3381)
 * and uniform_real_distribution: canonical * (b - a) + a (random.h). */
static double canonical(rng64* r) {
    const double sum = (double)rng_next(r);
    const double tmp = 18446744073709551616.0; /* 2^64 */
    double ret = sum / tmp;
    if (ret >= 1.0) ret = nextafter(1.0, 0.0);
    return ret;
}
static double uniform_real(rng64* r, double a, double b) { return canonical(r) * (b - a) + a; }

/* --------------------------------------------- dual numbers (autodiff/dual.hpp) */
/* Dual (dual.hpp:11-41): every mixed double/Dual operation promotes the
 * double to Dual(x, 0) (dual.hpp:48-56), reproduced literally here. */
typedef struct {
    double re, pr;
} dual;

static inline dual D(double re) { dual d = {re, 0.0}; return d; }
static inline dual DP(double re, double pr) { dual d = {re, pr}; return d; }
static inline dual dadd(dual a, dual b) { return DP(a.re + b.re, a.pr + b.pr); }
static inline dual dsub(dual a, dual b) { return DP(a.re - b.re, a.pr - b.pr); }
static inline dual dmul(dual a, dual b) { return DP(a.re * b.re, a.pr * b.re + a.re * b.pr); }
static inline dual ddiv(dual a, dual b) {
    return DP(a.re / b.re, (a.pr * b.re - a.re * b.pr) / (b.re * b.re));
}
static inline dual dneg(dual a) { return DP(-a.re, -a.pr); }
static inline dual dexp(dual x) { const double e = exp(x.re); return DP(e, x.pr * e); }      /* :58-61 */
static inline dual dsqrt(dual x) { const double s = sqrt(x.re); return DP(s, x.pr / (2.0 * s)); } /* :63-66 */
static inline dual dsigmoid(dual x) {                                                         /* :69-72 */
    const double s = 1.0 / (1.0 + exp(-x.re));
    return DP(s, x.pr * s * (1.0 - s));
}

/* ------------------------------------------------- geometry (core/geometry.hpp) */
#define COV_DILATION 0.3      /* geometry.hpp:12 */
#define SCREEN_CULL_SIGMA 3.0 /* geometry.hpp:15 */
#define ALPHA_CLAMP 0.99      /* rasterizer.hpp:15 */
#define ALPHA_SKIP (1.0 / 255.0)
#define T_FLOOR 1e-4
#define COLOR_C0 0.28209479177387814 /* types.hpp:24 */
#define NP 14

/* sym2_max_eigenvalue (vecmath.hpp:91-96) */
static double sym2_max_eig(double a, double b, double c) {
    const double mid = 0.5 * (a + c);
    const double det = a * c - b * b;
    const double v = mid * mid - det;
    const double disc = sqrt(v > 0.0 ? v : 0.0);
    return mid + disc;
}

/* quat_to_rotation (geometry.hpp:21-39); returns -1 on a zero quaternion */
static int quat_to_rotation(const dual q[4], dual r[9]) {
    const dual nsq = dadd(dadd(dadd(dmul(q[0], q[0]), dmul(q[1], q[1])), dmul(q[2], q[2])),
                          dmul(q[3], q[3]));
    if (nsq.re == 0.0) return -1;
    const dual inv = ddiv(D(1.0), dsqrt(nsq));
    const dual w = dmul(q[0], inv), x = dmul(q[1], inv), y = dmul(q[2], inv), z = dmul(q[3], inv);
    r[0] = dsub(D(1.0), dmul(D(2.0), dadd(dmul(y, y), dmul(z, z))));
    r[1] = dmul(D(2.0), dsub(dmul(x, y), dmul(w, z)));
    r[2] = dmul(D(2.0), dadd(dmul(x, z), dmul(w, y)));
    r[3] = dmul(D(2.0), dadd(dmul(x, y), dmul(w, z)));
    r[4] = dsub(D(1.0), dmul(D(2.0), dadd(dmul(x, x), dmul(z, z))));
    r[5] = dmul(D(2.0), dsub(dmul(y, z), dmul(w, x)));
    r[6] = dmul(D(2.0), dsub(dmul(x, z), dmul(w, y)));
    r[7] = dmul(D(2.0), dadd(dmul(y, z), dmul(w, x)));
    r[8] = dsub(D(1.0), dmul(D(2.0), dadd(dmul(x, x), dmul(y, y))));
    return 0;
}

/* covariance_3d (geometry.hpp:43-57): Sigma = (R S)(R S)^T */
static int covariance_3d(const dual ls[3], const dual q[4], dual sigma[9]) {
    dual r[9], m[9];
    if (quat_to_rotation(q, r)) return -1;
    const dual s[3] = {dexp(ls[0]), dexp(ls[1]), dexp(ls[2])};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) m[3 * i + j] = dmul(r[3 * i + j], s[j]);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            sigma[3 * i + j] = dadd(dadd(dmul(m[3 * i], m[3 * j]), dmul(m[3 * i + 1], m[3 * j + 1])),
                                    dmul(m[3 * i + 2], m[3 * j + 2]));
    return 0;
}

typedef struct {
    dual mx, my, ca, cb, cc; /* mean2d, conic */
    dual opacity;
    dual color[3];
    double cov[3];
    double depth, radius;
    int valid;
} splat;

typedef struct {
    double mean[3], log_scale[3], rot[4], logit, color[3];
} gparams;

static gparams params_of(const slm_gaussians* g, int i) {
    gparams p;
    for (int k = 0; k < 3; ++k) {
        p.mean[k] = g->means[3 * i + k];
        p.log_scale[k] = g->log_scales[3 * i + k];
        p.color[k] = g->colors[3 * i + k];
    }
    for (int k = 0; k < 4; ++k) p.rot[k] = g->rotations[4 * i + k];
    p.logit = g->opacity_logits[i];
    return p;
}

/* prepare_splat (rasterizer.hpp:58-94) over project_gaussian (geometry.hpp:71-108).
 * tangent: 14 raw-parameter tangent components (NULL = zero); returns -1 on a
 * zero quaternion (std::domain_error in the reference). */
static int prepare_splat(const gparams* gp, const double* tangent, const slm_camera* cam,
                         splat* out) {
    memset(out, 0, sizeof *out);
    dual mean[3], ls[3], q[4], logit, col[3];
#define TG(k) (tangent ? tangent[k] : 0.0)
    for (int k = 0; k < 3; ++k) {
        mean[k] = DP(gp->mean[k], TG(k));
        ls[k] = DP(gp->log_scale[k], TG(3 + k));
        col[k] = DP(gp->color[k], TG(11 + k));
    }
    for (int k = 0; k < 4; ++k) q[k] = DP(gp->rot[k], TG(6 + k));
    logit = DP(gp->logit, TG(10));
#undef TG

    dual sigma[9];
    if (covariance_3d(ls, q, sigma)) return -1;

    /* project_gaussian */
    const double* r = cam->world_to_cam;
    dual t[3];
    for (int k = 0; k < 3; ++k)
        t[k] = dadd(dadd(dadd(dmul(D(r[3 * k]), mean[0]), dmul(D(r[3 * k + 1]), mean[1])),
                         dmul(D(r[3 * k + 2]), mean[2])),
                    D(cam->translation[k]));
    out->depth = t[2].re;
    if (t[2].re <= cam->near_clip) return 0;

    const dual iz = ddiv(D(1.0), t[2]);
    const dual mx = dadd(dmul(dmul(D(cam->fx), t[0]), iz), D(cam->cx));
    const dual my = dadd(dmul(dmul(D(cam->fy), t[1]), iz), D(cam->cy));
    const dual iz2 = dmul(iz, iz);
    const dual j00 = dmul(D(cam->fx), iz), j02 = dmul(dmul(D(-cam->fx), t[0]), iz2);
    const dual j11 = dmul(D(cam->fy), iz), j12 = dmul(dmul(D(-cam->fy), t[1]), iz2);
    dual row0[3], row1[3], s0[3], s1[3];
    for (int k = 0; k < 3; ++k) {
        row0[k] = dadd(dmul(j00, D(r[k])), dmul(j02, D(r[6 + k])));
        row1[k] = dadd(dmul(j11, D(r[3 + k])), dmul(j12, D(r[6 + k])));
    }
    for (int i = 0; i < 3; ++i) {
        s0[i] = dadd(dadd(dmul(sigma[3 * i], row0[0]), dmul(sigma[3 * i + 1], row0[1])),
                     dmul(sigma[3 * i + 2], row0[2]));
        s1[i] = dadd(dadd(dmul(sigma[3 * i], row1[0]), dmul(sigma[3 * i + 1], row1[1])),
                     dmul(sigma[3 * i + 2], row1[2]));
    }
#define DOT3(u, v) dadd(dadd(dmul(u[0], v[0]), dmul(u[1], v[1])), dmul(u[2], v[2]))
    const dual ca = dadd(DOT3(row0, s0), D(COV_DILATION));
    const dual cb = DOT3(row0, s1);
    const dual cc = dadd(DOT3(row1, s1), D(COV_DILATION));
#undef DOT3
    const double cull_r = SCREEN_CULL_SIGMA * sqrt(sym2_max_eig(ca.re, cb.re, cc.re));
    if (mx.re + cull_r < 0.0 || mx.re - cull_r > cam->width || my.re + cull_r < 0.0 ||
        my.re - cull_r > cam->height)
        return 0;

    /* prepare_splat proper */
    out->mx = mx;
    out->my = my;
    out->cov[0] = ca.re;
    out->cov[1] = cb.re;
    out->cov[2] = cc.re;
    const dual det = dsub(dmul(ca, cc), dmul(cb, cb));
    if (!(det.re > 0.0)) return 0;
    const dual inv_det = ddiv(D(1.0), det);
    out->ca = dmul(cc, inv_det);
    out->cb = dmul(dneg(cb), inv_det);
    out->cc = dmul(ca, inv_det);
    out->opacity = dsigmoid(logit);
    for (int c = 0; c < 3; ++c) {
        const dual raw = dadd(D(0.5), dmul(D(COLOR_C0), col[c]));
        out->color[c] = raw.re > 0.0 ? raw : D(0.0);
    }
    const double o = out->opacity.re;
    if (o <= ALPHA_SKIP) return 0;
    const double lam = sym2_max_eig(out->cov[0], out->cov[1], out->cov[2]);
    out->radius = sqrt(2.0 * log(255.0 * o) * lam) * (1.0 + 1e-6) + 1e-6;
    out->valid = 1;
    return 0;
}

/* blend_pixel (rasterizer.hpp:100-130); last = list position where the loop
 * stopped (== n when it ran to the end). */
static void blend_pixel(const splat* sp, const int* order, int n, double px, double py,
                        dual rgb[3], dual* trans_out, int* contrib) {
    rgb[0] = rgb[1] = rgb[2] = D(0.0);
    dual T = D(1.0);
    *contrib = 0;
    for (int k = 0; k < n; ++k) {
        const splat* s = &sp[order[k]];
        const dual dx = dsub(s->mx, D(px)), dy = dsub(s->my, D(py));
        const dual power =
            dsub(dmul(D(-0.5), dadd(dmul(dmul(s->ca, dx), dx), dmul(dmul(s->cc, dy), dy))),
                 dmul(dmul(s->cb, dx), dy));
        if (power.re > 0.0) continue;
        dual alpha = dmul(s->opacity, dexp(power));
        if (alpha.re > ALPHA_CLAMP) alpha = D(ALPHA_CLAMP);
        if (alpha.re < ALPHA_SKIP) continue;
        const dual test_t = dmul(T, dsub(D(1.0), alpha));
        if (test_t.re < T_FLOOR) break;
        const dual w = dmul(alpha, T);
        for (int c = 0; c < 3; ++c) rgb[c] = dadd(rgb[c], dmul(w, s->color[c]));
        T = test_t;
        ++*contrib;
    }
    *trans_out = T;
}

/* ------------------------------------------------ tile grid (rasterizer.cpp:21-50) */
typedef struct {
    int tiles_x, tiles_y;
    int* offsets; /* tiles+1, CSR */
    int* idx;
} tilegrid;

static const splat* g_sort_splats;
static int cmp_depth_index(const void* pa, const void* pb) {
    const int a = *(const int*)pa, b = *(const int*)pb;
    const double da = g_sort_splats[a].depth, db = g_sort_splats[b].depth;
    if (da != db) return da < db ? -1 : 1;
    return (a > b) - (a < b);
}

static void build_tile_grid(const splat* sp, int count, const slm_camera* cam, tilegrid* grid) {
    grid->tiles_x = (cam->width + SLM_TILE - 1) / SLM_TILE;
    grid->tiles_y = (cam->height + SLM_TILE - 1) / SLM_TILE;
    const int nt = grid->tiles_x * grid->tiles_y;
    int* cnt = (int*)calloc(nt + 1, sizeof(int));
    int(*rect)[4] = malloc(sizeof(int[4]) * (count > 0 ? count : 1));
    for (int g = 0; g < count; ++g) {
        rect[g][0] = 1;
        rect[g][1] = 0;
        if (!sp[g].valid) continue;
        const double r = sp[g].radius;
        int x0 = (int)floor((sp[g].mx.re - r) / SLM_TILE);
        int x1 = (int)floor((sp[g].mx.re + r) / SLM_TILE);
        int y0 = (int)floor((sp[g].my.re - r) / SLM_TILE);
        int y1 = (int)floor((sp[g].my.re + r) / SLM_TILE);
        if (x0 < 0) x0 = 0;
        if (y0 < 0) y0 = 0;
        if (x1 > grid->tiles_x - 1) x1 = grid->tiles_x - 1;
        if (y1 > grid->tiles_y - 1) y1 = grid->tiles_y - 1;
        rect[g][0] = x0;
        rect[g][1] = x1;
        rect[g][2] = y0;
        rect[g][3] = y1;
        for (int ty = y0; ty <= y1; ++ty)
            for (int tx = x0; tx <= x1; ++tx) ++cnt[ty * grid->tiles_x + tx + 1];
    }
    grid->offsets = (int*)malloc(sizeof(int) * (nt + 1));
    grid->offsets[0] = 0;
    for (int t = 0; t < nt; ++t) grid->offsets[t + 1] = grid->offsets[t] + cnt[t + 1];
    grid->idx = (int*)malloc(sizeof(int) * (grid->offsets[nt] > 0 ? grid->offsets[nt] : 1));
    memset(cnt, 0, sizeof(int) * (nt + 1));
    for (int g = 0; g < count; ++g) { /* push in Gaussian order */
        if (!sp[g].valid) continue;
        for (int ty = rect[g][2]; ty <= rect[g][3]; ++ty)
            for (int tx = rect[g][0]; tx <= rect[g][1]; ++tx) {
                const int t = ty * grid->tiles_x + tx;
                grid->idx[grid->offsets[t] + cnt[t]++] = g;
            }
    }
    g_sort_splats = sp; /* per-tile (depth, index) order: rasterizer.cpp:43-48 */
    for (int t = 0; t < nt; ++t)
        qsort(grid->idx + grid->offsets[t], grid->offsets[t + 1] - grid->offsets[t], sizeof(int),
              cmp_depth_index);
    free(cnt);
    free(rect);
}

static void free_grid(tilegrid* g) {
    free(g->offsets);
    free(g->idx);
}

/* prepare_camera (rasterizer.cpp:10-19) */
typedef struct {
    slm_camera cam;
    splat* splats;
    tilegrid grid;
} camctx;

static int prepare_camera(const slm_gaussians* g, const slm_camera* cam, camctx* ctx) {
    ctx->cam = *cam;
    ctx->splats = (splat*)malloc(sizeof(splat) * (g->count > 0 ? g->count : 1));
    for (int i = 0; i < g->count; ++i) {
        const gparams p = params_of(g, i);
        if (prepare_splat(&p, NULL, cam, &ctx->splats[i])) {
            free(ctx->splats);
            ctx->splats = NULL;
            return set_err(E_DOMAIN, "zero-norm quaternion");
        }
    }
    build_tile_grid(ctx->splats, g->count, cam, &ctx->grid);
    return 0;
}

static void free_ctx(camctx* c) {
    free(c->splats);
    free_grid(&c->grid);
}

/* render_with_context (rasterizer.cpp:62-91) */
static void render_ctx(const camctx* ctx, double* image, double* trans, int32_t* contrib) {
    const slm_camera* cam = &ctx->cam;
    for (int ty = 0; ty < ctx->grid.tiles_y; ++ty)
        for (int tx = 0; tx < ctx->grid.tiles_x; ++tx) {
            const int t = ty * ctx->grid.tiles_x + tx;
            const int* list = ctx->grid.idx + ctx->grid.offsets[t];
            const int n = ctx->grid.offsets[t + 1] - ctx->grid.offsets[t];
            const int x1 = tx * SLM_TILE + SLM_TILE < cam->width ? tx * SLM_TILE + SLM_TILE : cam->width;
            const int y1 = ty * SLM_TILE + SLM_TILE < cam->height ? ty * SLM_TILE + SLM_TILE : cam->height;
            for (int y = ty * SLM_TILE; y < y1; ++y)
                for (int x = tx * SLM_TILE; x < x1; ++x) {
                    dual rgb[3], T;
                    int cn;
                    blend_pixel(ctx->splats, list, n, x + 0.5, y + 0.5, rgb, &T, &cn);
                    const size_t pix = (size_t)y * cam->width + x;
                    for (int c = 0; c < 3; ++c) image[3 * pix + c] = rgb[c].re;
                    if (trans) trans[pix] = T.re;
                    if (contrib) contrib[pix] = cn;
                }
        }
}

int orc_prepare(const slm_gaussians* g, const slm_camera* cam, double* mean2d, double* conic,
                double* opacity, double* color, double* depth, double* radius, int32_t* valid) {
    for (int i = 0; i < g->count; ++i) {
        const gparams p = params_of(g, i);
        splat s;
        if (prepare_splat(&p, NULL, cam, &s)) return set_err(E_DOMAIN, "zero-norm quaternion");
        mean2d[2 * i] = s.mx.re;
        mean2d[2 * i + 1] = s.my.re;
        conic[3 * i] = s.ca.re;
        conic[3 * i + 1] = s.cb.re;
        conic[3 * i + 2] = s.cc.re;
        opacity[i] = s.opacity.re;
        for (int c = 0; c < 3; ++c) color[3 * i + c] = s.color[c].re;
        depth[i] = s.depth;
        radius[i] = s.radius;
        valid[i] = s.valid;
    }
    return 0;
}

int orc_bin_and_sort(const slm_gaussians* g, const slm_camera* cam, int32_t* offsets,
                     int32_t* indices, int64_t capacity, int64_t* n_entries) {
    camctx ctx;
    const int rc = prepare_camera(g, cam, &ctx);
    if (rc) return rc;
    const int nt = ctx.grid.tiles_x * ctx.grid.tiles_y;
    for (int t = 0; t <= nt; ++t) offsets[t] = ctx.grid.offsets[t];
    const int64_t n = ctx.grid.offsets[nt];
    for (int64_t k = 0; k < n && k < capacity; ++k) indices[k] = ctx.grid.idx[k];
    *n_entries = n;
    free_ctx(&ctx);
    return 0;
}

int orc_render_full(const slm_gaussians* g, const slm_camera* cam, double* image,
                    double* transmittance, int32_t* contrib) {
    camctx ctx;
    const int rc = prepare_camera(g, cam, &ctx);
    if (rc) return rc;
    render_ctx(&ctx, image, transmittance, contrib);
    free_ctx(&ctx);
    return 0;
}

/* -------------------------------------------------- io helpers (harness) */
/* ring_camera (io/scene_gen.cpp:11-36) */
int orc_ring_camera(double angle, double radius, double height, int size, slm_camera* out) {
    const double pos[3] = {radius * cos(angle), height, radius * sin(angle)};
    double fwd[3] = {0.0 - pos[0], 0.0 - pos[1], 0.0 - pos[2]};
    const double fn = sqrt(fwd[0] * fwd[0] + fwd[1] * fwd[1] + fwd[2] * fwd[2]);
    for (int k = 0; k < 3; ++k) fwd[k] /= fn;
    const double up[3] = {0.0, 1.0, 0.0};
    double right[3] = {fwd[1] * up[2] - fwd[2] * up[1], fwd[2] * up[0] - fwd[0] * up[2],
                       fwd[0] * up[1] - fwd[1] * up[0]};
    const double rn = sqrt(right[0] * right[0] + right[1] * right[1] + right[2] * right[2]);
    for (int k = 0; k < 3; ++k) right[k] /= rn;
    const double down[3] = {fwd[1] * right[2] - fwd[2] * right[1],
                            fwd[2] * right[0] - fwd[0] * right[2],
                            fwd[0] * right[1] - fwd[1] * right[0]};
    memset(out, 0, sizeof *out);
    for (int k = 0; k < 3; ++k) {
        out->world_to_cam[k] = right[k];
        out->world_to_cam[3 + k] = down[k];
        out->world_to_cam[6 + k] = fwd[k];
    }
    for (int r = 0; r < 3; ++r) {
        const double* row = out->world_to_cam + 3 * r;
        out->translation[r] = -(row[0] * pos[0] + row[1] * pos[1] + row[2] * pos[2]);
    }
    out->width = out->height = size;
    const double fov_x = 50.0 * 3.14159265358979323846 / 180.0;
    out->fx = out->fy = 0.5 * size / tan(0.5 * fov_x);
    out->cx = out->cy = 0.5 * size;
    out->near_clip = 0.2;
    return 0;
}

static void alloc_set(slm_gaussians* g, int count) {
    g->count = count;
    g->means = (double*)calloc(3 * (size_t)count + 1, sizeof(double));
    g->log_scales = (double*)calloc(3 * (size_t)count + 1, sizeof(double));
    g->rotations = (double*)calloc(4 * (size_t)count + 1, sizeof(double));
    g->opacity_logits = (double*)calloc((size_t)count + 1, sizeof(double));
    g->colors = (double*)calloc(3 * (size_t)count + 1, sizeof(double));
    for (int i = 0; i < count; ++i) g->rotations[4 * i] = 1.0;
}
static void copy_set(const slm_gaussians* s, slm_gaussians* d) {
    const size_t n = (size_t)s->count;
    memcpy(d->means, s->means, 3 * n * sizeof(double));
    memcpy(d->log_scales, s->log_scales, 3 * n * sizeof(double));
    memcpy(d->rotations, s->rotations, 4 * n * sizeof(double));
    memcpy(d->opacity_logits, s->opacity_logits, n * sizeof(double));
    memcpy(d->colors, s->colors, 3 * n * sizeof(double));
}
static void free_set(slm_gaussians* g) {
    free(g->means);
    free(g->log_scales);
    free(g->rotations);
    free(g->opacity_logits);
    free(g->colors);
}

/* GaussianSet::renormalize_rotations (types.cpp:62-73) */
static void renormalize(slm_gaussians* g) {
    for (int i = 0; i < g->count; ++i) {
        double* q = g->rotations + 4 * i;
        const double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
        if (n == 0.0) {
            q[0] = 1.0;
            q[1] = q[2] = q[3] = 0.0;
            continue;
        }
        for (int k = 0; k < 4; ++k) q[k] /= n;
    }
}

/* random_init (io/dataset.cpp:138-166) */
int orc_random_init(int count, const double* lo, const double* hi, void* rngp,
                    slm_gaussians* out) {
    if (count < 1) return set_err(E_INVALID, "random_init: count must be at least 1");
    rng64* rng = (rng64*)rngp;
    const double coeff_max = 0.5 / COLOR_C0;
    double edge = hi[0] - lo[0];
    if (hi[1] - lo[1] > edge) edge = hi[1] - lo[1];
    if (hi[2] - lo[2] > edge) edge = hi[2] - lo[2];
    const double scale = log(0.5 * edge * pow((double)count, -1.0 / 3.0));
    const double logit = log(0.1 / 0.9);
    for (int i = 0; i < count; ++i) {
        out->means[3 * i] = uniform_real(rng, lo[0], hi[0]);
        out->means[3 * i + 1] = uniform_real(rng, lo[1], hi[1]);
        out->means[3 * i + 2] = uniform_real(rng, lo[2], hi[2]);
        for (int c = 0; c < 3; ++c) {
            out->log_scales[3 * i + c] = scale;
            out->colors[3 * i + c] = uniform_real(rng, -coeff_max, coeff_max);
        }
        out->rotations[4 * i] = 1.0;
        out->rotations[4 * i + 1] = out->rotations[4 * i + 2] = out->rotations[4 * i + 3] = 0.0;
        out->opacity_logits[i] = logit;
    }
    return 0;
}

/* generate_toy_scene (io/scene_gen.cpp:38-86) */
int orc_toy_scene(int gaussians, int train_cams, int test_cams, int image_size, uint64_t seed,
                  slm_gaussians* gt, slm_camera* cams_out, float* images_out) {
    if (gaussians < 1) return set_err(E_INVALID, "toy scene needs at least one Gaussian");
    rng64 rng;
    rng_seed(&rng, seed);
    const double PI = 3.14159265358979323846;
    for (int i = 0; i < gaussians; ++i) {
        for (int c = 0; c < 3; ++c) {
            gt->means[3 * i + c] = uniform_real(&rng, -0.8, 0.8);
            gt->log_scales[3 * i + c] = uniform_real(&rng, log(0.12), log(0.35));
            gt->colors[3 * i + c] = uniform_real(&rng, -1.2, 1.2);
        }
        double q[4], norm;
        do {
            norm = 0.0;
            for (int k = 0; k < 4; ++k) {
                q[k] = uniform_real(&rng, -1.0, 1.0);
                norm += q[k] * q[k];
            }
        } while (norm < 1e-4);
        for (int k = 0; k < 4; ++k) gt->rotations[4 * i + k] = q[k];
        const double o = uniform_real(&rng, 0.4, 0.9);
        gt->opacity_logits[i] = log(o / (1.0 - o));
    }
    gt->count = gaussians;
    renormalize(gt);
    float* dst = images_out;
    const int counts[2] = {train_cams, test_cams};
    const double phase[2] = {0.0, 0.37}, height[2] = {1.1, 1.6};
    int k = 0;
    double* img = (double*)malloc(sizeof(double) * 3 * (size_t)image_size * image_size);
    for (int split = 0; split < 2; ++split)
        for (int i = 0; i < counts[split]; ++i) {
            const double angle = phase[split] + 2.0 * PI * i / counts[split];
            orc_ring_camera(angle, 3.2, height[split], image_size, &cams_out[k]);
            const int rc = orc_render_full(gt, &cams_out[k], img, NULL, NULL);
            if (rc) {
                free(img);
                return rc;
            }
            for (size_t e = 0; e < 3 * (size_t)image_size * image_size; ++e) dst[e] = (float)img[e];
            dst += 3 * (size_t)image_size * image_size;
            ++k;
        }
    free(img);
    return 0;
}

/* --------------------------------------------------------- sample plans */
typedef struct {
    int n_views, samples_per_tile, dist;
    int* view_camera;
    int64_t* view_offset;
    int *px, *py, *tile;
    double* weight;
    int64_t cap;
} plan_t;

static void plan_push(plan_t* p, int x, int y, int t, double w) {
    const int64_t n = p->view_offset[p->n_views];
    if (n >= p->cap) {
        p->cap = p->cap ? 2 * p->cap : 1024;
        p->px = realloc(p->px, sizeof(int) * p->cap);
        p->py = realloc(p->py, sizeof(int) * p->cap);
        p->tile = realloc(p->tile, sizeof(int) * p->cap);
        p->weight = realloc(p->weight, sizeof(double) * p->cap);
    }
    p->px[n] = x;
    p->py[n] = y;
    p->tile[n] = t;
    p->weight[n] = w;
    p->view_offset[p->n_views] = n + 1;
}

static plan_t* plan_new(int n_cams) {
    plan_t* p = (plan_t*)calloc(1, sizeof(plan_t));
    p->view_camera = (int*)calloc(n_cams + 1, sizeof(int));
    p->view_offset = (int64_t*)calloc(n_cams + 2, sizeof(int64_t));
    return p;
}

void orc_plan_free(void* pp) {
    plan_t* p = (plan_t*)pp;
    if (!p) return;
    free(p->view_camera);
    free(p->view_offset);
    free(p->px);
    free(p->py);
    free(p->tile);
    free(p->weight);
    free(p);
}
int orc_plan_views(void* p) { return ((plan_t*)p)->n_views; }
int64_t orc_plan_total(void* p) { return ((plan_t*)p)->view_offset[((plan_t*)p)->n_views]; }
void orc_plan_export(void* pp, int32_t* view_camera, int64_t* view_offset, int32_t* px,
                     int32_t* py, int32_t* tile, double* weight) {
    const plan_t* p = (const plan_t*)pp;
    for (int v = 0; v < p->n_views; ++v) view_camera[v] = p->view_camera[v];
    for (int v = 0; v <= p->n_views; ++v) view_offset[v] = p->view_offset[v];
    const int64_t n = p->view_offset[p->n_views];
    for (int64_t k = 0; k < n; ++k) {
        px[k] = p->px[k];
        py[k] = p->py[k];
        tile[k] = p->tile[k];
        weight[k] = p->weight[k];
    }
}

static int imin(int a, int b) { return a < b ? a : b; }

/* build_sample_plan (sampling/sample_plan.cpp:62-171) */
void* orc_build_sample_plan(const slm_camera* cams, int n_cams, int spt, int dist, int lane,
                            void* rngp, const double* const* aux_image,
                            const int32_t* const* aux_contrib, const double* const* aux_gt) {
    rng64* rng = (rng64*)rngp;
    if (spt < 1) {
        set_err(E_INVALID, "samples_per_tile must be positive");
        return NULL;
    }
    if (spt > SLM_TILE * SLM_TILE) {
        set_err(E_INVALID, "samples_per_tile exceeds the pixels in a tile");
        return NULL;
    }
    if (lane < 1 || spt % lane != 0) {
        set_err(E_INVALID, "samples_per_tile must be a multiple of the lane width");
        return NULL;
    }
    if (dist != SLM_DIST_UNIFORM) {
        if (!aux_image || !aux_contrib) {
            set_err(E_INVALID, "weighted distributions need per-camera aux data");
            return NULL;
        }
        if (dist == SLM_DIST_RESIDUAL && !aux_gt) {
            set_err(E_INVALID, "residual distribution needs ground-truth images");
            return NULL;
        }
    }
    /* batch-wide total, known before drawing (:86-94) */
    size_t total = 0;
    for (int ci = 0; ci < n_cams; ++ci) {
        const int tx_n = (cams[ci].width + SLM_TILE - 1) / SLM_TILE;
        const int ty_n = (cams[ci].height + SLM_TILE - 1) / SLM_TILE;
        for (int ty = 0; ty < ty_n; ++ty)
            for (int tx = 0; tx < tx_n; ++tx) {
                const int w = imin(cams[ci].width - tx * SLM_TILE, SLM_TILE);
                const int h = imin(cams[ci].height - ty * SLM_TILE, SLM_TILE);
                total += (size_t)imin(spt, w * h);
            }
    }
    const double n_total = (double)total;
    plan_t* plan = plan_new(n_cams);
    plan->samples_per_tile = spt;
    plan->dist = dist;
    int* pool = (int*)malloc(sizeof(int) * 256);
    double density[256], cdf[256];
    for (int ci = 0; ci < n_cams; ++ci) {
        const slm_camera* cam = &cams[ci];
        const int tx_n = (cam->width + SLM_TILE - 1) / SLM_TILE;
        const int ty_n = (cam->height + SLM_TILE - 1) / SLM_TILE;
        plan->view_camera[ci] = ci;
        plan->view_offset[ci + 1] = plan->view_offset[ci];
        plan->n_views = ci + 1;
        for (int ty = 0; ty < ty_n; ++ty)
            for (int tx = 0; tx < tx_n; ++tx) {
                const int x0 = tx * SLM_TILE, y0 = ty * SLM_TILE;
                const int rw = imin(cam->width - x0, SLM_TILE), rh = imin(cam->height - y0, SLM_TILE);
                const int m = rw * rh, n = imin(spt, m), tile = ty * tx_n + tx;
#define EMIT(local, q_tile)                                                     \
    do {                                                                        \
        const double q = (n / n_total) * (q_tile);                              \
        plan_push(plan, x0 + (local) % rw, y0 + (local) / rw, tile,             \
                  1.0 / (q > 1e-12 ? q : 1e-12));                               \
    } while (0)
                if (dist == SLM_DIST_UNIFORM) {
                    /* draw_without_replacement: partial Fisher-Yates (:42-51) */
                    for (int i = 0; i < m; ++i) pool[i] = i;
                    for (int i = 0; i < n; ++i) {
                        const int j = uniform_int(rng, i, m - 1);
                        const int t = pool[i];
                        pool[i] = pool[j];
                        pool[j] = t;
                    }
                    for (int i = 0; i < n; ++i) EMIT(pool[i], 1.0 / m);
                    continue;
                }
                if (dist == SLM_DIST_RESIDUAL) { /* softmax of |residual| (:129-145) */
                    double vmax = -1.0;
                    for (int l = 0; l < m; ++l) {
                        const int x = x0 + l % rw, y = y0 + l / rw;
                        const size_t pix = (size_t)y * cam->width + x;
                        double v = 0.0;
                        for (int c = 0; c < 3; ++c)
                            v += fabs(aux_image[ci][3 * pix + c] - aux_gt[ci][3 * pix + c]);
                        density[l] = v / 3.0;
                        if (density[l] > vmax) vmax = density[l];
                    }
                    double sum = 0.0;
                    for (int l = 0; l < m; ++l) sum += (density[l] = exp(density[l] - vmax));
                    for (int l = 0; l < m; ++l) density[l] /= sum;
                } else { /* contributor counts + 1 (:146-158) */
                    double sum = 0.0;
                    for (int l = 0; l < m; ++l) {
                        const int x = x0 + l % rw, y = y0 + l / rw;
                        sum += (density[l] = 1.0 + aux_contrib[ci][(size_t)y * cam->width + x]);
                    }
                    for (int l = 0; l < m; ++l) density[l] /= sum;
                }
                /* with replacement through the CDF (:160-165, draw_from_cdf :53-58) */
                double acc = 0.0;
                for (int l = 0; l < m; ++l) cdf[l] = (acc += density[l]);
                for (int k = 0; k < n; ++k) {
                    const double u = uniform_real(rng, 0.0, 1.0) * cdf[m - 1];
                    int lo = 0, hi = m; /* upper_bound */
                    while (lo < hi) {
                        const int mid = (lo + hi) / 2;
                        if (u < cdf[mid]) hi = mid; else lo = mid + 1;
                    }
                    const int local = lo < m - 1 ? lo : m - 1;
                    EMIT(local, density[local]);
                }
#undef EMIT
            }
    }
    free(pool);
    return plan;
}

/* exhaustive_plan (sample_plan.cpp:173-197) */
void* orc_exhaustive_plan(const slm_camera* cams, int n_cams) {
    double n_total = 0;
    for (int i = 0; i < n_cams; ++i) n_total += (double)cams[i].width * cams[i].height;
    plan_t* plan = plan_new(n_cams);
    plan->samples_per_tile = SLM_TILE * SLM_TILE;
    for (int ci = 0; ci < n_cams; ++ci) {
        const int tx_n = (cams[ci].width + SLM_TILE - 1) / SLM_TILE;
        plan->view_camera[ci] = ci;
        plan->view_offset[ci + 1] = plan->view_offset[ci];
        plan->n_views = ci + 1;
        for (int y = 0; y < cams[ci].height; ++y)
            for (int x = 0; x < cams[ci].width; ++x)
                plan_push(plan, x, y, (y / SLM_TILE) * tx_n + x / SLM_TILE, n_total);
    }
    return plan;
}

/* estimate_loss (sample_plan.cpp:199-222) */
int orc_estimate_loss(const slm_camera* cams, const slm_plan* plan,
                      const double* const* fields, double* out) {
    const int64_t n_total = plan->view_offset[plan->n_views];
    if (n_total == 0) {
        *out = 0.0;
        return 0;
    }
    double pixels = 0.0;
    for (int v = 0; v < plan->n_views; ++v)
        pixels += (double)cams[plan->view_camera[v]].width * cams[plan->view_camera[v]].height;
    double acc = 0.0;
    for (int v = 0; v < plan->n_views; ++v) {
        const int w = cams[plan->view_camera[v]].width;
        for (int64_t s = plan->view_offset[v]; s < plan->view_offset[v + 1]; ++s) {
            double sq = 0.0;
            for (int c = 0; c < 3; ++c) {
                const double r = fields[v][((size_t)plan->py[s] * w + plan->px[s]) * 3 + c];
                sq += r * r;
            }
            acc += plan->weight[s] * sq;
        }
    }
    *out = acc / ((double)n_total * pixels * 3.0);
    return 0;
}

/* ------------------------------------------ view sampler (sampling/view_sampler.cpp) */
/* camera_features (:10-40); position = -R^T t (types.cpp:75-81), direction = R row 2 */
int orc_camera_features(const slm_camera* cams, int n, double* f) {
    double lo[3] = {1.79769313486231570815e308, 1.79769313486231570815e308, 1.79769313486231570815e308};
    double hi[3] = {-1.79769313486231570815e308, -1.79769313486231570815e308, -1.79769313486231570815e308};
    double* pos = (double*)malloc(sizeof(double) * 3 * (n + 1));
    for (int c = 0; c < n; ++c) {
        const double* r = cams[c].world_to_cam;
        const double* t = cams[c].translation;
        pos[3 * c] = -(r[0] * t[0] + r[3] * t[1] + r[6] * t[2]);
        pos[3 * c + 1] = -(r[1] * t[0] + r[4] * t[1] + r[7] * t[2]);
        pos[3 * c + 2] = -(r[2] * t[0] + r[5] * t[1] + r[8] * t[2]);
        for (int i = 0; i < 3; ++i) {
            if (pos[3 * c + i] < lo[i]) lo[i] = pos[3 * c + i];
            if (pos[3 * c + i] > hi[i]) hi[i] = pos[3 * c + i];
        }
    }
    for (int c = 0; c < n; ++c) {
        for (int i = 0; i < 3; ++i) {
            const double ext = hi[i] - lo[i];
            f[6 * c + i] = ext > 1e-12 ? (pos[3 * c + i] - lo[i]) / ext : 0.5;
        }
        for (int i = 0; i < 3; ++i) f[6 * c + 3 + i] = cams[c].world_to_cam[6 + i];
    }
    free(pos);
    return 0;
}

static double dist_sq6(const double* a, const double* b) {
    double acc = 0.0;
    for (int i = 0; i < 6; ++i) {
        const double d = a[i] - b[i];
        acc += d * d;
    }
    return acc;
}

/* kmeans_cameras (:101-171) with seed_centroids (:55-97) */
static int kmeans(const double* feats, int n, int k, uint64_t seed, int* assign) {
    if (k < 1) return set_err(E_INVALID, "cluster count must be at least 1");
    if (k > n) return set_err(E_INVALID, "cluster count exceeds camera count");
    rng64 rng;
    rng_seed(&rng, seed);
    double* cen = (double*)malloc(sizeof(double) * 6 * k);
    char* chosen = (char*)calloc(n, 1);
    double* d2 = (double*)malloc(sizeof(double) * n);
    int nc = 0;
    int idx = uniform_int(&rng, 0, n - 1);
    memcpy(cen, feats + 6 * idx, 6 * sizeof(double));
    chosen[idx] = 1;
    nc = 1;
    while (nc < k) {
        double total = 0.0;
        for (int i = 0; i < n; ++i) {
            d2[i] = 1.79769313486231570815e308;
            for (int c = 0; c < nc; ++c) {
                const double d = dist_sq6(feats + 6 * i, cen + 6 * c);
                if (d < d2[i]) d2[i] = d;
            }
            if (chosen[i]) d2[i] = 0.0;
            total += d2[i];
        }
        int pick = -1;
        if (total > 0.0) {
            double u = uniform_real(&rng, 0.0, total);
            for (int i = 0; i < n; ++i) {
                u -= d2[i];
                if (u <= 0.0) {
                    pick = i;
                    break;
                }
            }
            if (pick < 0) pick = n - 1;
        }
        if (pick < 0 || chosen[pick]) {
            pick = 0;
            while (pick < n && chosen[pick]) ++pick;
        }
        memcpy(cen + 6 * nc, feats + 6 * pick, 6 * sizeof(double));
        chosen[pick] = 1;
        ++nc;
    }
    for (int i = 0; i < n; ++i) assign[i] = -1;
    int* sizes = (int*)malloc(sizeof(int) * k);
    for (int iter = 0; iter < 100; ++iter) {
        int changed = 0;
        for (int i = 0; i < n; ++i) {
            int best = 0;
            double bd = dist_sq6(feats + 6 * i, cen);
            for (int c = 1; c < k; ++c) {
                const double d = dist_sq6(feats + 6 * i, cen + 6 * c);
                if (d < bd) {
                    bd = d;
                    best = c;
                }
            }
            if (assign[i] != best) {
                assign[i] = best;
                changed = 1;
            }
        }
        memset(sizes, 0, sizeof(int) * k);
        for (int i = 0; i < n; ++i) ++sizes[assign[i]];
        for (int c = 0; c < k; ++c) {
            if (sizes[c] > 0) continue;
            int far = -1;
            double far_d = -1.0;
            for (int i = 0; i < n; ++i) {
                if (sizes[assign[i]] <= 1) continue;
                const double d = dist_sq6(feats + 6 * i, cen + 6 * assign[i]);
                if (d > far_d) {
                    far_d = d;
                    far = i;
                }
            }
            if (far < 0) continue;
            --sizes[assign[far]];
            assign[far] = c;
            ++sizes[c];
            memcpy(cen + 6 * c, feats + 6 * far, 6 * sizeof(double));
            changed = 1;
        }
        for (int c = 0; c < k; ++c) {
            double mean[6] = {0, 0, 0, 0, 0, 0};
            int count = 0;
            for (int i = 0; i < n; ++i) {
                if (assign[i] != c) continue;
                for (int d = 0; d < 6; ++d) mean[d] += feats[6 * i + d];
                ++count;
            }
            if (count > 0)
                for (int d = 0; d < 6; ++d) cen[6 * c + d] = mean[d] / count;
        }
        if (!changed) break;
    }
    free(sizes);
    free(cen);
    free(chosen);
    free(d2);
    return 0;
}

int orc_kmeans_cameras(const slm_camera* cams, int n, int k, uint64_t seed, int32_t* assign) {
    double* f = (double*)malloc(sizeof(double) * 6 * (n + 1));
    orc_camera_features(cams, n, f);
    int* a = (int*)malloc(sizeof(int) * (n + 1));
    const int rc = kmeans(f, n, k, seed, a);
    if (!rc)
        for (int i = 0; i < n; ++i) assign[i] = a[i];
    free(f);
    free(a);
    return rc;
}

/* -------------------------------------------------- SampledJacobian (autodiff/jacobian.cpp) */
#define ACCUM_CHUNKS 16 /* jacobian.cpp:21 */
static void vaxpy(double alpha, const double* x, double* y, size_t n);
#define INTER 9         /* jacobian.cpp:65 */

typedef struct {
    double p[5][10];
    double dop, dcol[3];
    int valid;
} projchain;

typedef struct {
    slm_gaussians g;
    slm_camera* cams;
    int n_cams;
    plan_t* plan;
    camctx* ctx;
    projchain** chains;
    int64_t* view_off;
    double* weights;
    int64_t rdim, pdim;
} jac_t;

typedef struct {
    int idx;
    double alpha, trans;
    int clamped;
} blendrec;

/* replay_forward (jacobian.cpp:34-61) */
static int replay_forward(const splat* sp, const int* order, int n, double px, double py,
                          blendrec* rec) {
    int nr = 0;
    double T = 1.0;
    for (int k = 0; k < n; ++k) {
        const splat* s = &sp[order[k]];
        const double dx = s->mx.re - px, dy = s->my.re - py;
        const double power = -0.5 * (s->ca.re * dx * dx + s->cc.re * dy * dy) - s->cb.re * dx * dy;
        if (power > 0.0) continue;
        double alpha = s->opacity.re * exp(power);
        int clamped = 0;
        if (alpha > ALPHA_CLAMP) {
            alpha = ALPHA_CLAMP;
            clamped = 1;
        }
        if (alpha < ALPHA_SKIP) continue;
        const double test_t = T * (1.0 - alpha);
        if (test_t < T_FLOOR) break;
        rec[nr].idx = order[k];
        rec[nr].alpha = alpha;
        rec[nr].trans = T;
        rec[nr].clamped = clamped;
        ++nr;
        T = test_t;
    }
    return nr;
}

/* backward_pixel_vjp (jacobian.cpp:67-94) */
static void backward_pixel(const splat* sp, const blendrec* rec, int nr, double px, double py,
                           const double u[3], double* inter) {
    double suffix[3] = {0.0, 0.0, 0.0};
    for (int k = nr - 1; k >= 0; --k) {
        const blendrec* r = &rec[k];
        const splat* s = &sp[r->idx];
        double* gi = inter + (size_t)INTER * r->idx;
        const double w = r->alpha * r->trans;
        double dalpha = 0.0;
        for (int c = 0; c < 3; ++c) {
            gi[6 + c] += u[c] * w;
            dalpha += u[c] * (r->trans * s->color[c].re - suffix[c] / (1.0 - r->alpha));
            suffix[c] += w * s->color[c].re;
        }
        if (r->clamped) continue;
        const double dpower = dalpha * r->alpha;
        const double dx = s->mx.re - px, dy = s->my.re - py;
        gi[0] += dpower * -(s->ca.re * dx + s->cb.re * dy);
        gi[1] += dpower * -(s->cb.re * dx + s->cc.re * dy);
        gi[2] += dpower * (-0.5 * dx * dx);
        gi[3] += dpower * (-dx * dy);
        gi[4] += dpower * (-0.5 * dy * dy);
        gi[5] += dalpha * (r->alpha / s->opacity.re);
    }
}

static plan_t* plan_from_c(const slm_plan* p) {
    plan_t* q = plan_new(p->n_views);
    q->n_views = p->n_views;
    q->samples_per_tile = p->samples_per_tile;
    q->dist = p->dist;
    const int64_t n = p->view_offset[p->n_views];
    q->cap = n > 0 ? n : 1;
    q->px = malloc(sizeof(int) * q->cap);
    q->py = malloc(sizeof(int) * q->cap);
    q->tile = malloc(sizeof(int) * q->cap);
    q->weight = malloc(sizeof(double) * q->cap);
    for (int v = 0; v < p->n_views; ++v) q->view_camera[v] = p->view_camera[v];
    for (int v = 0; v <= p->n_views; ++v) q->view_offset[v] = p->view_offset[v];
    for (int64_t k = 0; k < n; ++k) {
        q->px[k] = p->px[k];
        q->py[k] = p->py[k];
        q->tile[k] = p->tile[k];
        q->weight[k] = p->weight[k];
    }
    return q;
}

/* SampledJacobian ctor (jacobian.cpp:98-119) + build_chains (:127-165) */
void* orc_jac_new(const slm_gaussians* g, const slm_camera* cams, int n_cams,
                  const slm_plan* plan) {
    for (int v = 0; v < plan->n_views; ++v)
        if (plan->view_camera[v] < 0 || plan->view_camera[v] >= n_cams) {
            set_err(E_INVALID, "sample plan references a camera outside the batch");
            return NULL;
        }
    jac_t* j = (jac_t*)calloc(1, sizeof(jac_t));
    alloc_set(&j->g, g->count);
    copy_set(g, &j->g);
    j->n_cams = n_cams;
    j->cams = (slm_camera*)malloc(sizeof(slm_camera) * (n_cams + 1));
    memcpy(j->cams, cams, sizeof(slm_camera) * n_cams);
    j->plan = plan_from_c(plan);
    const int nv = plan->n_views;
    j->ctx = (camctx*)calloc(nv + 1, sizeof(camctx));
    j->view_off = (int64_t*)malloc(sizeof(int64_t) * (nv + 1));
    for (int v = 0; v < nv; ++v) {
        if (prepare_camera(&j->g, &cams[plan->view_camera[v]], &j->ctx[v])) {
            for (int u = 0; u < v; ++u) free_ctx(&j->ctx[u]);
            return NULL; /* error already set */
        }
        j->view_off[v] = plan->view_offset[v];
    }
    const int64_t total = plan->view_offset[nv];
    j->rdim = 3 * total;
    j->pdim = (int64_t)NP * g->count;
    j->weights = (double*)malloc(sizeof(double) * (j->rdim + 1));
    const double inv_total = total > 0 ? 1.0 / (double)total : 0.0;
    for (int64_t s = 0; s < total; ++s)
        for (int c = 0; c < 3; ++c) j->weights[3 * s + c] = plan->weight[s] * inv_total;

    j->chains = (projchain**)calloc(nv + 1, sizeof(projchain*));
    for (int v = 0; v < nv; ++v) {
        projchain* ch = (projchain*)calloc(g->count + 1, sizeof(projchain));
        const slm_camera* cam = &cams[plan->view_camera[v]];
        for (int i = 0; i < g->count; ++i) {
            const splat* s = &j->ctx[v].splats[i];
            ch[i].valid = s->valid;
            if (!s->valid) continue;
            const gparams base = params_of(&j->g, i);
            for (int k = 0; k < 10; ++k) {
                double tg[NP] = {0};
                tg[k] = 1.0;
                splat ds;
                prepare_splat(&base, tg, cam, &ds);
                ch[i].p[0][k] = ds.mx.pr;
                ch[i].p[1][k] = ds.my.pr;
                ch[i].p[2][k] = ds.ca.pr;
                ch[i].p[3][k] = ds.cb.pr;
                ch[i].p[4][k] = ds.cc.pr;
            }
            const double o = s->opacity.re;
            ch[i].dop = o * (1.0 - o);
            for (int c = 0; c < 3; ++c) ch[i].dcol[c] = s->color[c].re > 0.0 ? COLOR_C0 : 0.0;
        }
        j->chains[v] = ch;
    }
    return j;
}

void orc_jac_free(void* jp) {
    jac_t* j = (jac_t*)jp;
    if (!j) return;
    for (int v = 0; v < j->plan->n_views; ++v) {
        free_ctx(&j->ctx[v]);
        free(j->chains[v]);
    }
    free(j->ctx);
    free(j->chains);
    free(j->view_off);
    free(j->weights);
    free(j->cams);
    orc_plan_free(j->plan);
    free_set(&j->g);
    free(j);
}
int64_t orc_jac_residual_dim(void* j) { return ((jac_t*)j)->rdim; }
int64_t orc_jac_param_dim(void* j) { return ((jac_t*)j)->pdim; }

/* jvp (jacobian.cpp:191-211) with dual_splats (:167-189) */
int orc_jac_jvp(void* jp, const double* v, double* out) {
    jac_t* j = (jac_t*)jp;
    splat* duals = (splat*)malloc(sizeof(splat) * (j->g.count + 1));
    for (int vi = 0; vi < j->plan->n_views; ++vi) {
        const slm_camera* cam = &j->cams[j->plan->view_camera[vi]];
        for (int i = 0; i < j->g.count; ++i) {
            const gparams base = params_of(&j->g, i);
            prepare_splat(&base, v + (size_t)NP * i, cam, &duals[i]);
        }
        const camctx* ctx = &j->ctx[vi];
        for (int64_t s = j->plan->view_offset[vi]; s < j->plan->view_offset[vi + 1]; ++s) {
            const int t = j->plan->tile[s];
            dual rgb[3], T;
            int cn;
            blend_pixel(duals, ctx->grid.idx + ctx->grid.offsets[t],
                        ctx->grid.offsets[t + 1] - ctx->grid.offsets[t], j->plan->px[s] + 0.5,
                        j->plan->py[s] + 0.5, rgb, &T, &cn);
            for (int c = 0; c < 3; ++c) out[3 * s + c] = rgb[c].pr;
        }
    }
    free(duals);
    return 0;
}

static blendrec* rec_buf(const camctx* ctx) {
    int maxn = 1;
    const int nt = ctx->grid.tiles_x * ctx->grid.tiles_y;
    for (int t = 0; t < nt; ++t)
        if (ctx->grid.offsets[t + 1] - ctx->grid.offsets[t] > maxn)
            maxn = ctx->grid.offsets[t + 1] - ctx->grid.offsets[t];
    return (blendrec*)malloc(sizeof(blendrec) * maxn);
}

/* vjp (jacobian.cpp:219-264): 16 fixed chunks merged in order, then the chain */
int orc_jac_vjp(void* jp, const double* u, double* out) {
    jac_t* j = (jac_t*)jp;
    const size_t G = (size_t)j->g.count, isz = G * INTER;
    for (int64_t k = 0; k < j->pdim; ++k) out[k] = 0.0;
    double* inter = (double*)malloc(sizeof(double) * (isz + 1));
    double* chunk = (double*)malloc(sizeof(double) * (isz * ACCUM_CHUNKS + 1));
    for (int vi = 0; vi < j->plan->n_views; ++vi) {
        const camctx* ctx = &j->ctx[vi];
        const int64_t off = j->plan->view_offset[vi];
        const int64_t n = j->plan->view_offset[vi + 1] - off;
        memset(inter, 0, sizeof(double) * isz);
        memset(chunk, 0, sizeof(double) * isz * ACCUM_CHUNKS);
        blendrec* rec = rec_buf(ctx);
        if (n > 0) {
            const int chunks = n < ACCUM_CHUNKS ? (int)n : ACCUM_CHUNKS;
            for (int c = 0; c < chunks; ++c) {
                const int64_t lo = n * c / chunks, hi = n * (c + 1) / chunks;
                for (int64_t s = off + lo; s < off + hi; ++s) {
                    const int t = j->plan->tile[s];
                    const double px = j->plan->px[s] + 0.5, py = j->plan->py[s] + 0.5;
                    const int nr = replay_forward(ctx->splats, ctx->grid.idx + ctx->grid.offsets[t],
                                                  ctx->grid.offsets[t + 1] - ctx->grid.offsets[t],
                                                  px, py, rec);
                    backward_pixel(ctx->splats, rec, nr, px, py, u + 3 * s, chunk + isz * c);
                }
            }
        }
        free(rec);
        for (int c = 0; c < ACCUM_CHUNKS; ++c)
            for (size_t k = 0; k < isz; ++k) inter[k] += 1.0 * chunk[isz * c + k];
        const projchain* ch = j->chains[vi];
        for (size_t g = 0; g < G; ++g) {
            if (!ch[g].valid) continue;
            const double* gi = inter + INTER * g;
            double* ob = out + NP * g;
            for (int k = 0; k < 10; ++k) {
                double acc = 0.0;
                for (int i = 0; i < 5; ++i) acc += ch[g].p[i][k] * gi[i];
                ob[k] += acc;
            }
            ob[10] += gi[5] * ch[g].dop;
            for (int c = 0; c < 3; ++c) ob[11 + c] += gi[6 + c] * ch[g].dcol[c];
        }
    }
    free(inter);
    free(chunk);
    return 0;
}

/* jtj_diag (jacobian.cpp:272-337) */
int orc_jac_jtj_diag(void* jp, double* diag) {
    jac_t* j = (jac_t*)jp;
    const size_t p = (size_t)j->pdim;
    for (size_t k = 0; k < p; ++k) diag[k] = 0.0;
    double* chunk = (double*)malloc(sizeof(double) * (p * ACCUM_CHUNKS + 1));
    for (int vi = 0; vi < j->plan->n_views; ++vi) {
        const camctx* ctx = &j->ctx[vi];
        const projchain* ch = j->chains[vi];
        const int64_t off = j->plan->view_offset[vi];
        const int64_t n = j->plan->view_offset[vi + 1] - off;
        memset(chunk, 0, sizeof(double) * p * ACCUM_CHUNKS);
        blendrec* rec = rec_buf(ctx);
        const int chunks = n < ACCUM_CHUNKS ? (int)n : ACCUM_CHUNKS;
        for (int c = 0; c < chunks && n > 0; ++c) {
            double* local = chunk + p * c;
            const int64_t lo = n * c / chunks, hi = n * (c + 1) / chunks;
            for (int64_t s = off + lo; s < off + hi; ++s) {
                const int t = j->plan->tile[s];
                const double px = j->plan->px[s] + 0.5, py = j->plan->py[s] + 0.5;
                const int nr = replay_forward(ctx->splats, ctx->grid.idx + ctx->grid.offsets[t],
                                              ctx->grid.offsets[t + 1] - ctx->grid.offsets[t], px,
                                              py, rec);
                const double* we = j->weights + 3 * s;
                double suffix[3] = {0.0, 0.0, 0.0};
                for (int k = nr - 1; k >= 0; --k) {
                    const blendrec* r = &rec[k];
                    const splat* sp = &ctx->splats[r->idx];
                    const projchain* pc = &ch[r->idx];
                    double* d = local + (size_t)NP * r->idx;
                    const double w = r->alpha * r->trans;
                    double dac[3];
                    for (int cc = 0; cc < 3; ++cc) {
                        dac[cc] = r->trans * sp->color[cc].re - suffix[cc] / (1.0 - r->alpha);
                        suffix[cc] += w * sp->color[cc].re;
                        const double e = w * pc->dcol[cc];
                        d[11 + cc] += we[cc] * e * e;
                    }
                    if (r->clamped) continue;
                    const double dx = sp->mx.re - px, dy = sp->my.re - py;
                    const double gp[5] = {-(sp->ca.re * dx + sp->cb.re * dy),
                                          -(sp->cb.re * dx + sp->cc.re * dy), -0.5 * dx * dx,
                                          -dx * dy, -0.5 * dy * dy};
                    for (int cc = 0; cc < 3; ++cc) {
                        if (we[cc] == 0.0) continue;
                        const double dp = dac[cc] * r->alpha;
                        double q[5];
                        for (int i = 0; i < 5; ++i) q[i] = dp * gp[i];
                        for (int k2 = 0; k2 < 10; ++k2) {
                            double row = 0.0;
                            for (int i = 0; i < 5; ++i) row += q[i] * pc->p[i][k2];
                            d[k2] += we[cc] * row * row;
                        }
                        const double eo = dac[cc] * (r->alpha / sp->opacity.re) * pc->dop;
                        d[10] += we[cc] * eo * eo;
                    }
                }
            }
        }
        free(rec);
        for (int c = 0; c < ACCUM_CHUNKS; ++c)
            for (size_t k = 0; k < p; ++k) diag[k] += 1.0 * chunk[p * c + k];
    }
    free(chunk);
    return 0;
}

/* gn_apply (jacobian.cpp:339-344) */
int orc_jac_gn_apply(void* jp, double lambda, const double* p, double* out) {
    jac_t* j = (jac_t*)jp;
    double* tmp = (double*)malloc(sizeof(double) * (j->rdim + 1));
    orc_jac_jvp(j, p, tmp);
    for (int64_t k = 0; k < j->rdim; ++k) tmp[k] = tmp[k] * j->weights[k];
    orc_jac_vjp(j, tmp, out);
    vaxpy(lambda, p, out, (size_t)j->pdim);
    free(tmp);
    return 0;
}

int orc_jac_weights(void* jp, double* out) {
    jac_t* j = (jac_t*)jp;
    memcpy(out, j->weights, sizeof(double) * j->rdim);
    return 0;
}
int orc_jac_set_weights(void* jp, const double* w) {
    jac_t* j = (jac_t*)jp;
    memcpy(j->weights, w, sizeof(double) * j->rdim);
    return 0;
}

/* ---------------------------------------------------------- PCG (solver/pcg.cpp:10-53) */
typedef void (*apply_fn)(void* user, const double* p, double* out);

/* The reference dispatches its flat-vector kernels to the AVX2/FMA variants
 * on x86 hosts with AVX2+FMA (kernels/vec_kernels.cpp:72-90); these restate
 * their exact association order (kernels/vec_kernels_avx2.cpp:14-96): two
 * 4-lane fused accumulators, hsum = (l0+l2)+(l1+l3), scalar tails. */
static double hsum4(const double v[4]) { return (v[0] + v[2]) + (v[1] + v[3]); }

static double vdot(const double* a, const double* b, size_t n) { /* dot_avx2 :24-37 */
    double acc0[4] = {0, 0, 0, 0}, acc1[4] = {0, 0, 0, 0};
    size_t i = 0;
    for (; i + 8 <= n; i += 8)
        for (int l = 0; l < 4; ++l) {
            acc0[l] = fma(a[i + l], b[i + l], acc0[l]);
            acc1[l] = fma(a[i + 4 + l], b[i + 4 + l], acc1[l]);
        }
    for (; i + 4 <= n; i += 4)
        for (int l = 0; l < 4; ++l) acc0[l] = fma(a[i + l], b[i + l], acc0[l]);
    double s[4];
    for (int l = 0; l < 4; ++l) s[l] = acc0[l] + acc1[l];
    double acc = hsum4(s);
    for (; i < n; ++i) acc += a[i] * b[i];
    return acc;
}

static double vssd(const double* a, const double* b, size_t n) { /* sum_squared_diff_avx2 :41-61 */
    double acc0[4] = {0, 0, 0, 0}, acc1[4] = {0, 0, 0, 0};
    size_t i = 0;
    for (; i + 8 <= n; i += 8)
        for (int l = 0; l < 4; ++l) {
            const double d0 = a[i + l] - b[i + l], d1 = a[i + 4 + l] - b[i + 4 + l];
            acc0[l] = fma(d0, d0, acc0[l]);
            acc1[l] = fma(d1, d1, acc1[l]);
        }
    for (; i + 4 <= n; i += 4)
        for (int l = 0; l < 4; ++l) {
            const double d = a[i + l] - b[i + l];
            acc0[l] = fma(d, d, acc0[l]);
        }
    double s[4];
    for (int l = 0; l < 4; ++l) s[l] = acc0[l] + acc1[l];
    double acc = hsum4(s);
    for (; i < n; ++i) {
        const double d = a[i] - b[i];
        acc += d * d;
    }
    return acc;
}

static void vaxpy(double alpha, const double* x, double* y, size_t n) { /* axpy_avx2 :63-71 */
    size_t i = 0;
    for (; i + 4 <= n; i += 4)
        for (int l = 0; l < 4; ++l) y[i + l] = fma(alpha, x[i + l], y[i + l]);
    for (; i < n; ++i) y[i] += alpha * x[i];
}

static void vxpby(const double* x, double beta, double* y, size_t n) { /* xpby_avx2 :73-81 */
    size_t i = 0;
    for (; i + 4 <= n; i += 4)
        for (int l = 0; l < 4; ++l) y[i + l] = fma(beta, y[i + l], x[i + l]);
    for (; i < n; ++i) y[i] = x[i] + beta * y[i];
}

static void pcg(apply_fn apply, void* user, const double* b, const double* minv, size_t n,
                int max_iters, double* x, slm_pcg_result* res) {
    for (size_t i = 0; i < n; ++i) x[i] = 0.0;
    res->iterations = 0;
    res->breakdown = 0;
    res->rel_residual = 1.0;
    const double b_norm = sqrt(vdot(b, b, n));
    if (b_norm == 0.0) {
        res->rel_residual = 0.0;
        return;
    }
    double* r = (double*)malloc(sizeof(double) * (n + 1));
    double* z = (double*)malloc(sizeof(double) * (n + 1));
    double* p = (double*)malloc(sizeof(double) * (n + 1));
    double* u = (double*)malloc(sizeof(double) * (n + 1));
    memcpy(r, b, sizeof(double) * n);
    for (size_t i = 0; i < n; ++i) z[i] = minv[i] * r[i];
    memcpy(p, z, sizeof(double) * n);
    double rz = vdot(r, z, n);
    for (int it = 0; it < max_iters; ++it) {
        apply(user, p, u);
        const double pu = vdot(p, u, n);
        if (pu <= 0.0) {
            res->breakdown = 1;
            break;
        }
        const double alpha = rz / pu;
        vaxpy(alpha, p, x, n);
        vaxpy(-alpha, u, r, n);
        ++res->iterations;
        if (sqrt(vdot(r, r, n)) <= 1e-12 * b_norm) break;
        for (size_t i = 0; i < n; ++i) z[i] = minv[i] * r[i];
        const double rz_next = vdot(r, z, n);
        const double beta = rz_next / rz;
        rz = rz_next;
        vxpby(z, beta, p, n);
    }
    res->rel_residual = sqrt(vdot(r, r, n)) / b_norm;
    free(r);
    free(z);
    free(p);
    free(u);
}

typedef struct {
    jac_t* j;
    double lambda;
} gn_user;
static void gn_apply_cb(void* user, const double* p, double* out) {
    gn_user* g = (gn_user*)user;
    orc_jac_gn_apply(g->j, g->lambda, p, out);
}
int orc_jac_pcg(void* jp, double lambda, const double* b, const double* minv, int iters, double* x,
                slm_pcg_result* res) {
    gn_user u = {(jac_t*)jp, lambda};
    pcg(gn_apply_cb, &u, b, minv, (size_t)((jac_t*)jp)->pdim, iters, x, res);
    return 0;
}

typedef struct {
    const double* a;
    int n;
} dense_user;
static void dense_cb(void* user, const double* p, double* out) {
    const dense_user* d = (const dense_user*)user;
    for (int i = 0; i < d->n; ++i) {
        double acc = 0.0;
        for (int k = 0; k < d->n; ++k) acc += d->a[(size_t)i * d->n + k] * p[k];
        out[i] = acc;
    }
}
int orc_pcg_dense(const double* a, int n, const double* b, const double* minv, int iters,
                  double* x, slm_pcg_result* res) {
    dense_user u = {a, n};
    pcg(dense_cb, &u, b, minv, (size_t)n, iters, x, res);
    return 0;
}

/* ------------------------------------------------------------- LM (solver/lm.cpp) */
/* learning_rate (lm.cpp:26-37) */
double orc_learning_rate(const double* delta, int64_t n, int iteration, const slm_lm_config* cfg) {
    if (n % NP != 0) {
        set_err(E_INVALID, "learning_rate: bad update length");
        return 0.0;
    }
    if (iteration < cfg->warmup_iterations) return cfg->warmup_lr;
    double m = 0.0;
    for (int64_t base = 0; base < n; base += NP)
        for (int c = 0; c < 3; ++c) {
            const double a = fabs(delta[base + 11 + c]);
            if (a > m) m = a;
        }
    if (m > 1.0) return cfg->lr_cap < 1.0 / m ? cfg->lr_cap : 1.0 / m;
    return cfg->lr_cap < 1.0 ? cfg->lr_cap : 1.0;
}

/* GaussianSet::apply_update (types.cpp:48-60) */
int orc_apply_update(slm_gaussians* g, const double* delta, double eta) {
    for (int i = 0; i < g->count; ++i) {
        const double* b = delta + (size_t)NP * i;
        for (int k = 0; k < 3; ++k) g->means[3 * i + k] += eta * b[k];
        for (int k = 0; k < 3; ++k) g->log_scales[3 * i + k] += eta * b[3 + k];
        for (int k = 0; k < 4; ++k) g->rotations[4 * i + k] += eta * b[6 + k];
        g->opacity_logits[i] += eta * b[10];
        for (int k = 0; k < 3; ++k) g->colors[3 * i + k] += eta * b[11 + k];
    }
    renormalize(g);
    return 0;
}

typedef struct {
    slm_camera* cams;
    int n;
    double** images;
    int* assign;
    int k;
} train_t;

void* orc_train_new(const slm_camera* cams, int n, const float* images) {
    train_t* t = (train_t*)calloc(1, sizeof(train_t));
    t->n = n;
    t->cams = (slm_camera*)malloc(sizeof(slm_camera) * (n + 1));
    memcpy(t->cams, cams, sizeof(slm_camera) * n);
    t->images = (double**)calloc(n + 1, sizeof(double*));
    t->assign = (int*)calloc(n + 1, sizeof(int));
    const float* src = images;
    for (int i = 0; i < n; ++i) {
        const size_t sz = 3 * (size_t)cams[i].width * cams[i].height;
        t->images[i] = (double*)malloc(sizeof(double) * sz);
        for (size_t e = 0; e < sz; ++e) t->images[i][e] = (double)src[e];
        src += sz;
    }
    return t;
}
void* orc_train_new_f64(const slm_camera* cams, int n, const double* images) {
    train_t* t = (train_t*)calloc(1, sizeof(train_t));
    t->n = n;
    t->cams = (slm_camera*)malloc(sizeof(slm_camera) * (n + 1));
    memcpy(t->cams, cams, sizeof(slm_camera) * n);
    t->images = (double**)calloc(n + 1, sizeof(double*));
    t->assign = (int*)calloc(n + 1, sizeof(int));
    const double* src = images;
    for (int i = 0; i < n; ++i) {
        const size_t sz = 3 * (size_t)cams[i].width * cams[i].height;
        t->images[i] = (double*)malloc(sizeof(double) * sz);
        memcpy(t->images[i], src, sizeof(double) * sz);
        src += sz;
    }
    return t;
}
void orc_train_free(void* tp) {
    train_t* t = (train_t*)tp;
    if (!t) return;
    for (int i = 0; i < t->n; ++i) free(t->images[i]);
    free(t->images);
    free(t->cams);
    free(t->assign);
    free(t);
}
/* TrainData::rebuild_clusters (lm.cpp:21-24) */
int orc_train_rebuild_clusters(void* tp, int k, uint64_t seed) {
    train_t* t = (train_t*)tp;
    const int rc = orc_kmeans_cameras(t->cams, t->n, k, seed, t->assign);
    if (!rc) t->k = k;
    return rc;
}
int orc_train_set_clusters(void* tp, const int32_t* assign, int n, int k) {
    train_t* t = (train_t*)tp;
    for (int i = 0; i < n; ++i) t->assign[i] = assign[i];
    t->k = k;
    return 0;
}

/* metrics::mse / psnr (image_metrics.cpp:108-119) */
double orc_mse(const double* a, const double* b, int w, int h) {
    const size_t n = 3 * (size_t)w * h;
    if (n == 0) return 0.0;
    return vssd(a, b, n) / (double)n;
}
double orc_psnr(const double* a, const double* b, int w, int h) {
    const double m = orc_mse(a, b, w, h);
    if (m < 1e-10) return 100.0;
    return 10.0 * log10(1.0 / m);
}

/* metrics::ssim (image_metrics.cpp:14-67,86-106,121-139): 11-tap Gaussian
 * window (sigma 1.5), separable filter with single reflect padding, C1 =
 * 0.01^2, C2 = 0.03^2, mean of the local SSIM over pixels and channels. */
#define SSIM_WIN 11
#define SSIM_HALF 5
static void ssim_window(double* w) {
    double sum = 0.0;
    for (int i = 0; i < SSIM_WIN; ++i) {
        const double d = i - SSIM_HALF;
        w[i] = exp(-0.5 * d * d / (1.5 * 1.5));
        sum += w[i];
    }
    for (int i = 0; i < SSIM_WIN; ++i) w[i] /= sum;
}
static int ssim_reflect(int i, int n) {
    if (i < 0) i = -i - 1;
    if (i >= n) i = 2 * n - i - 1;
    return i;
}
static void ssim_filter(const double* win, const double* src, int w, int h, double* tmp, double* dst) {
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            double acc = 0.0;
            for (int k = -SSIM_HALF; k <= SSIM_HALF; ++k)
                acc += win[k + SSIM_HALF] * src[(size_t)y * w + ssim_reflect(x + k, w)];
            tmp[(size_t)y * w + x] = acc;
        }
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            double acc = 0.0;
            for (int k = -SSIM_HALF; k <= SSIM_HALF; ++k)
                acc += win[k + SSIM_HALF] * tmp[(size_t)ssim_reflect(y + k, h) * w + x];
            dst[(size_t)y * w + x] = acc;
        }
}
double orc_ssim(const double* a, const double* b, int w, int h) {
    const size_t n = (size_t)w * h;
    if (n == 0) return 1.0;
    double win[SSIM_WIN];
    ssim_window(win);
    double* buf = (double*)malloc(sizeof(double) * n * 9);
    double *pa = buf, *pb = buf + n, *sq = buf + 2 * n, *tmp = buf + 3 * n, *ma = buf + 4 * n,
           *mb = buf + 5 * n, *eaa = buf + 6 * n, *ebb = buf + 7 * n, *eab = buf + 8 * n;
    const double c1 = 0.01 * 0.01, c2 = 0.03 * 0.03;
    double total = 0.0;
    for (int c = 0; c < 3; ++c) {
        for (size_t i = 0; i < n; ++i) {
            pa[i] = a[3 * i + c];
            pb[i] = b[3 * i + c];
        }
        ssim_filter(win, pa, w, h, tmp, ma);
        ssim_filter(win, pb, w, h, tmp, mb);
        for (size_t i = 0; i < n; ++i) sq[i] = pa[i] * pa[i];
        ssim_filter(win, sq, w, h, tmp, eaa);
        for (size_t i = 0; i < n; ++i) sq[i] = pb[i] * pb[i];
        ssim_filter(win, sq, w, h, tmp, ebb);
        for (size_t i = 0; i < n; ++i) sq[i] = pa[i] * pb[i];
        ssim_filter(win, sq, w, h, tmp, eab);
        for (size_t i = 0; i < n; ++i) {
            const double va = eaa[i] - ma[i] * ma[i], vb = ebb[i] - mb[i] * mb[i];
            const double cov = eab[i] - ma[i] * mb[i];
            const double num = (2.0 * ma[i] * mb[i] + c1) * (2.0 * cov + c2);
            const double den = (ma[i] * ma[i] + mb[i] * mb[i] + c1) * (va + vb + c2);
            total += num / den;
        }
    }
    free(buf);
    return total / (3.0 * (double)n);
}

/* effective_center_weights (image_metrics.cpp:69-78) */
static void ssim_center_weights(const double* win, int n, double* out) {
    for (int i = 0; i < n; ++i) {
        out[i] = 0.0;
        for (int k = -SSIM_HALF; k <= SSIM_HALF; ++k)
            if (ssim_reflect(i + k, n) == i) out[i] += win[k + SSIM_HALF];
    }
}

/* metrics::ssim_diag_residuals (image_metrics.cpp:141-178): per pixel and
 * channel s = sqrt(max(0, 1 - local SSIM)) and the derivative of s with
 * respect to the centre pixel of a (diagonal approximation). */
void orc_ssim_diag_residuals(const double* a, const double* b, int w, int h, double* residual,
                             double* d_center) {
    const size_t n = (size_t)w * h;
    double win[SSIM_WIN];
    ssim_window(win);
    double* wx = (double*)malloc(sizeof(double) * (w + 1));
    double* wy = (double*)malloc(sizeof(double) * (h + 1));
    ssim_center_weights(win, w, wx);
    ssim_center_weights(win, h, wy);
    double* buf = (double*)malloc(sizeof(double) * (n * 9 + 1));
    double *pa = buf, *pb = buf + n, *sq = buf + 2 * n, *tmp = buf + 3 * n, *ma = buf + 4 * n,
           *mb = buf + 5 * n, *eaa = buf + 6 * n, *ebb = buf + 7 * n, *eab = buf + 8 * n;
    const double c1 = 0.01 * 0.01, c2 = 0.03 * 0.03;
    for (size_t i = 0; i < 3 * n; ++i) residual[i] = d_center[i] = 0.0;
    for (int c = 0; c < 3; ++c) {
        for (size_t i = 0; i < n; ++i) {
            pa[i] = a[3 * i + c];
            pb[i] = b[3 * i + c];
        }
        ssim_filter(win, pa, w, h, tmp, ma);
        ssim_filter(win, pb, w, h, tmp, mb);
        for (size_t i = 0; i < n; ++i) sq[i] = pa[i] * pa[i];
        ssim_filter(win, sq, w, h, tmp, eaa);
        for (size_t i = 0; i < n; ++i) sq[i] = pb[i] * pb[i];
        ssim_filter(win, sq, w, h, tmp, ebb);
        for (size_t i = 0; i < n; ++i) sq[i] = pa[i] * pb[i];
        ssim_filter(win, sq, w, h, tmp, eab);
        for (size_t i = 0; i < n; ++i) {
            const double mua = ma[i], mub = mb[i];
            const double va = eaa[i] - mua * mua, vb = ebb[i] - mub * mub;
            const double cov = eab[i] - mua * mub;
            const double a1 = 2.0 * mua * mub + c1, a2 = 2.0 * cov + c2;
            const double b1 = mua * mua + mub * mub + c1, b2 = va + vb + c2;
            const double local = (a1 * a2) / (b1 * b2);
            const double sval = sqrt(1.0 - local > 0.0 ? 1.0 - local : 0.0);
            residual[3 * i + c] = sval;
            if (sval < 1e-12) continue;
            const double av = a[3 * i + c], bv = b[3 * i + c];
            const double wc = wx[i % w] * wy[i / w];
            const double dnum = mub * a2 + a1 * (bv - mub);
            const double dden = mua * b2 + b1 * (av - mua);
            const double dlocal = 2.0 * wc * (dnum * b1 * b2 - a1 * a2 * dden) / (b1 * b2 * b1 * b2);
            d_center[3 * i + c] = -dlocal / (2.0 * sval);
        }
    }
    free(buf);
    free(wx);
    free(wy);
}

/* the mse+ssim loss term of one image (lm.cpp:44-49, 143-147): w * sum(s^2) / (3n) */
static double ssim_loss_term(const double* img, const double* gt, int w, int h, double weight) {
    const size_t n3 = 3 * (size_t)w * h;
    double* r = (double*)malloc(sizeof(double) * (2 * n3 + 1));
    orc_ssim_diag_residuals(img, gt, w, h, r, r + n3);
    double ssq = 0.0;
    for (size_t i = 0; i < n3; ++i) ssq += r[i] * r[i];
    free(r);
    return weight * ssq / (double)n3;
}

/* batch_loss (lm.cpp:39-54) */
static int batch_loss_d(const slm_gaussians* g, const slm_camera* cams, const int* batch, int nb,
                        double* const* gts, int loss, double ssim_weight, double* out) {
    double acc = 0.0;
    for (int i = 0; i < nb; ++i) {
        const slm_camera* cam = &cams[batch[i]];
        const size_t sz = 3 * (size_t)cam->width * cam->height;
        double* img = (double*)malloc(sizeof(double) * (sz + 1));
        const int rc = orc_render_full(g, cam, img, NULL, NULL);
        if (rc) {
            free(img);
            return rc;
        }
        double term = orc_mse(img, gts[i], cam->width, cam->height);
        if (loss == SLM_LOSS_MSE_SSIM) term += ssim_loss_term(img, gts[i], cam->width, cam->height, ssim_weight);
        acc += term;
        free(img);
    }
    *out = nb == 0 ? 0.0 : acc / (double)nb;
    return 0;
}

int orc_batch_loss(const slm_gaussians* g, const slm_camera* cams, int n, const float* gts,
                   int loss, double ssim_weight, double* out) {
    double** imgs = (double**)calloc(n + 1, sizeof(double*));
    int* batch = (int*)malloc(sizeof(int) * (n + 1));
    const float* src = gts;
    for (int i = 0; i < n; ++i) {
        const size_t sz = 3 * (size_t)cams[i].width * cams[i].height;
        imgs[i] = (double*)malloc(sizeof(double) * sz);
        for (size_t e = 0; e < sz; ++e) imgs[i][e] = (double)src[e];
        src += sz;
        batch[i] = i;
    }
    const int rc = batch_loss_d(g, cams, batch, n, imgs, loss, ssim_weight, out);
    for (int i = 0; i < n; ++i) free(imgs[i]);
    free(imgs);
    free(batch);
    return rc;
}

/* lm_step (lm.cpp:56-157), both losses: with mse+ssim the diagonal SSIM rows
 * fold into the rhs and per-channel weights (lm.cpp:86-119) */
int orc_lm_step(slm_gaussians* g, void* tp, const slm_lm_config* cfg, int iteration, void* rngp,
                slm_step_report* rep) {
    train_t* t = (train_t*)tp;
    rng64* rng = (rng64*)rngp;
    if (t->k < 1) return set_err(E_INVALID, "lm_step: no view clusters");
    const int ssim = cfg->loss == SLM_LOSS_MSE_SSIM;
    rep->iteration = iteration;
    /* 1. one camera per cluster (sample_view_batch, view_sampler.cpp:173-184) */
    const int nb = t->k;
    int* batch = (int*)malloc(sizeof(int) * nb);
    int* members = (int*)malloc(sizeof(int) * (t->n + 1));
    for (int c = 0; c < nb; ++c) {
        int m = 0;
        for (int i = 0; i < t->n; ++i)
            if (t->assign[i] == c) members[m++] = i;
        if (m == 0) {
            free(batch);
            free(members);
            return set_err(E_INVALID, "empty cluster in batch sampler");
        }
        batch[c] = members[uniform_u64(rng, 0, (uint64_t)(m - 1))];
    }
    free(members);
    slm_camera* cams = (slm_camera*)malloc(sizeof(slm_camera) * nb);
    double** gts = (double**)malloc(sizeof(double*) * nb);
    double** renders = (double**)malloc(sizeof(double*) * nb);
    int32_t** contrib = (int32_t**)malloc(sizeof(int32_t*) * nb);
    for (int i = 0; i < nb; ++i) {
        cams[i] = t->cams[batch[i]];
        gts[i] = t->images[batch[i]];
        const size_t px = (size_t)cams[i].width * cams[i].height;
        renders[i] = (double*)malloc(sizeof(double) * 3 * px);
        contrib[i] = (int32_t*)malloc(sizeof(int32_t) * px);
        /* 2./3. forward render and residuals */
        const int rc = orc_render_full(g, &cams[i], renders[i], NULL, contrib[i]);
        if (rc) return rc;
    }
    /* 4. plan */
    plan_t* plan = (plan_t*)orc_build_sample_plan(cams, nb, cfg->samples_per_tile, cfg->dist,
                                                  cfg->sample_lane_width, rng,
                                                  (const double* const*)renders,
                                                  (const int32_t* const*)contrib,
                                                  (const double* const*)gts);
    if (!plan) return E_INVALID;
    slm_plan cp = {plan->n_views, plan->samples_per_tile, plan->dist, plan->view_camera,
                   plan->view_offset, plan->px, plan->py, plan->tile, plan->weight};
    jac_t* jac = (jac_t*)orc_jac_new(g, cams, nb, &cp);
    if (!jac) return E_DOMAIN;
    /* rhs = -w (r + ssim_weight sp sv), weights w (1 + ssim_weight sp^2) (lm.cpp:86-119) */
    double** sres = (double**)calloc(nb + 1, sizeof(double*));
    double* sterm = (double*)calloc(nb + 1, sizeof(double));
    if (ssim)
        for (int v = 0; v < nb; ++v) {
            const size_t n3 = 3 * (size_t)cams[v].width * cams[v].height;
            sres[v] = (double*)malloc(sizeof(double) * (2 * n3 + 1));
            orc_ssim_diag_residuals(renders[v], gts[v], cams[v].width, cams[v].height, sres[v], sres[v] + n3);
            double ssq = 0.0;
            for (size_t i = 0; i < n3; ++i) ssq += sres[v][i] * sres[v][i];
            sterm[v] = cfg->ssim_weight * ssq / (double)n3;
        }
    double* rhs = (double*)malloc(sizeof(double) * (jac->rdim + 1));
    double* w2 = (double*)malloc(sizeof(double) * (jac->rdim + 1));
    for (int v = 0; v < plan->n_views; ++v) {
        const int w = cams[v].width;
        const size_t n3 = 3 * (size_t)w * cams[v].height;
        for (int64_t s = plan->view_offset[v]; s < plan->view_offset[v + 1]; ++s)
            for (int c = 0; c < 3; ++c) {
                const size_t e = ((size_t)plan->py[s] * w + plan->px[s]) * 3 + c;
                const double r = renders[v][e] - gts[v][e];
                const double bw = jac->weights[3 * s + c];
                double u = r;
                w2[3 * s + c] = bw;
                if (ssim) {
                    const double sv = sres[v][e], sp = sres[v][n3 + e];
                    u += cfg->ssim_weight * sp * sv;
                    w2[3 * s + c] = bw * (1.0 + cfg->ssim_weight * sp * sp);
                }
                rhs[3 * s + c] = -bw * u;
            }
    }
    if (ssim) orc_jac_set_weights(jac, w2);
    free(w2);
    for (int v = 0; v < nb; ++v) free(sres[v]);
    free(sres);
    const size_t P = (size_t)jac->pdim;
    double* b = (double*)malloc(sizeof(double) * (P + 1));
    double* minv = (double*)malloc(sizeof(double) * (P + 1));
    double* x = (double*)malloc(sizeof(double) * (P + 1));
    orc_jac_vjp(jac, rhs, b);
    orc_jac_jtj_diag(jac, minv);
    for (size_t k = 0; k < P; ++k) minv[k] = 1.0 / (minv[k] + cfg->damping);
    slm_pcg_result pr;
    const int iters = iteration >= cfg->pcg_switch_iteration ? cfg->pcg_iters_late : cfg->pcg_iters_initial;
    orc_jac_pcg(jac, cfg->damping, b, minv, iters, x, &pr);
    rep->pcg_iterations = pr.iterations;
    rep->breakdown = pr.breakdown;
    rep->eta = orc_learning_rate(x, (int64_t)P, iteration, cfg);
    if (pr.breakdown) rep->eta *= 0.5;
    orc_apply_update(g, x, rep->eta);
    double before = 0.0;
    for (int i = 0; i < nb; ++i) before += orc_mse(renders[i], gts[i], cams[i].width, cams[i].height);
    if (ssim)
        for (int i = 0; i < nb; ++i) before += sterm[i];
    free(sterm);
    rep->loss_before = before / (double)nb;
    int* idx = (int*)malloc(sizeof(int) * nb);
    for (int i = 0; i < nb; ++i) idx[i] = i;
    const int rc = batch_loss_d(g, cams, idx, nb, gts, cfg->loss, cfg->ssim_weight, &rep->loss_after);
    free(idx);
    rep->batch_size = nb;
    for (int i = 0; i < nb && i < rep->batch_capacity; ++i) rep->batch[i] = batch[i];
    for (int i = 0; i < nb; ++i) {
        free(renders[i]);
        free(contrib[i]);
    }
    free(renders);
    free(contrib);
    free(gts);
    free(cams);
    free(batch);
    free(rhs);
    free(b);
    free(minv);
    free(x);
    orc_jac_free(jac);
    orc_plan_free(plan);
    if (rc) return rc;
    if (!isfinite(rep->loss_after)) return set_err(E_RUNTIME, "lm_step: non-finite loss after update");
    return 0;
}

/* ------------------------------------------------ first-order baselines */
/* baselines::full_gradient (first_order.cpp:11-44): exhaustive plan, dL/dr =
 * 2/M (r + w s s') at every pixel channel, J^T of that. */
int orc_full_gradient(const slm_gaussians* g, const slm_camera* cams, int n, const float* gts, int loss,
                      double ssim_weight, double* out) {
    plan_t* plan = (plan_t*)orc_exhaustive_plan(cams, n);
    slm_plan cp = {plan->n_views, plan->samples_per_tile, plan->dist, plan->view_camera,
                   plan->view_offset, plan->px, plan->py, plan->tile, plan->weight};
    jac_t* jac = (jac_t*)orc_jac_new(g, cams, n, &cp);
    if (!jac) {
        orc_plan_free(plan);
        return E_DOMAIN;
    }
    double entries = 0.0;
    for (int v = 0; v < n; ++v) entries += 3.0 * cams[v].width * cams[v].height;
    const double scale = 2.0 / entries;
    double* u = (double*)malloc(sizeof(double) * (jac->rdim + 1));
    const float* src = gts;
    size_t entry = 0;
    for (int v = 0; v < n; ++v) {
        const int w = cams[v].width, h = cams[v].height;
        const size_t n3 = 3 * (size_t)w * h;
        double* img = (double*)malloc(sizeof(double) * (4 * n3 + 1));
        double *gt = img + n3, *sres = img + 2 * n3, *sdc = img + 3 * n3;
        for (size_t e = 0; e < n3; ++e) gt[e] = (double)src[e];
        src += n3;
        const int rc = orc_render_full(g, &cams[v], img, NULL, NULL);
        if (rc) return rc;
        if (loss == SLM_LOSS_MSE_SSIM) orc_ssim_diag_residuals(img, gt, w, h, sres, sdc);
        for (int64_t s = plan->view_offset[v]; s < plan->view_offset[v + 1]; ++s)
            for (int c = 0; c < 3; ++c, ++entry) {
                const size_t e = ((size_t)plan->py[s] * w + plan->px[s]) * 3 + c;
                double r = img[e] - gt[e];
                if (loss == SLM_LOSS_MSE_SSIM) r += ssim_weight * sdc[e] * sres[e];
                u[entry] = scale * r;
            }
        free(img);
    }
    const int rc = orc_jac_vjp(jac, u, out);
    free(u);
    orc_jac_free(jac);
    orc_plan_free(plan);
    return rc;
}

/* GaussianSet::pack / unpack (types.cpp:20-46) */
static void orc_pack(const slm_gaussians* g, double* p) {
    for (int i = 0; i < g->count; ++i) {
        double* b = p + (size_t)NP * i;
        for (int k = 0; k < 3; ++k) b[k] = g->means[3 * i + k];
        for (int k = 0; k < 3; ++k) b[3 + k] = g->log_scales[3 * i + k];
        for (int k = 0; k < 4; ++k) b[6 + k] = g->rotations[4 * i + k];
        b[10] = g->opacity_logits[i];
        for (int k = 0; k < 3; ++k) b[11 + k] = g->colors[3 * i + k];
    }
}
static void orc_unpack(const double* p, slm_gaussians* g) {
    for (int i = 0; i < g->count; ++i) {
        const double* b = p + (size_t)NP * i;
        for (int k = 0; k < 3; ++k) g->means[3 * i + k] = b[k];
        for (int k = 0; k < 3; ++k) g->log_scales[3 * i + k] = b[3 + k];
        for (int k = 0; k < 4; ++k) g->rotations[4 * i + k] = b[6 + k];
        g->opacity_logits[i] = b[10];
        for (int k = 0; k < 3; ++k) g->colors[3 * i + k] = b[11 + k];
    }
}

/* group_lr (first_order.cpp:46-52) */
static double fo_group_lr(const slm_first_order_config* c, int k) {
    if (k < 3) return c->lr_mean;
    if (k < 6) return c->lr_scale;
    if (k < 10) return c->lr_rotation;
    if (k == 10) return c->lr_opacity;
    return c->lr_color;
}

/* adam / rmsprop / sgd_momentum steps (first_order.cpp:56-122) on the packed
 * ParamVector, then renormalize_rotations. */
int orc_first_order_step(slm_gaussians* g, double* m1, double* m2, int64_t* step, const double* grad,
                         const slm_first_order_config* cfg) {
    const size_t P = (size_t)NP * g->count;
    double* p = (double*)malloc(sizeof(double) * (P + 1));
    orc_pack(g, p);
    ++*step;
    const long t = (long)(*step - 1);
    double mean_factor = 1.0;
    if (cfg->decay_iterations > 0) {
        const double tt = (double)t / cfg->decay_iterations;
        mean_factor = pow(cfg->mean_lr_final_factor, tt < 1.0 ? tt : 1.0);
    }
    const double c1 = 1.0 - pow(cfg->adam_beta1, (double)*step);
    const double c2 = 1.0 - pow(cfg->adam_beta2, (double)*step);
    for (size_t j = 0; j < P; ++j) {
        const int k = (int)(j % NP);
        double lr = fo_group_lr(cfg, k);
        if (k < 3) lr *= mean_factor;
        const double gj = grad[j];
        if (cfg->kind == SLM_FO_ADAM) {
            m1[j] = cfg->adam_beta1 * m1[j] + (1.0 - cfg->adam_beta1) * gj;
            m2[j] = cfg->adam_beta2 * m2[j] + (1.0 - cfg->adam_beta2) * gj * gj;
            const double mhat = m1[j] / c1, vhat = m2[j] / c2;
            p[j] -= lr * mhat / (sqrt(vhat) + cfg->adam_eps);
        } else if (cfg->kind == SLM_FO_RMSPROP) {
            m2[j] = cfg->rms_decay * m2[j] + (1.0 - cfg->rms_decay) * gj * gj;
            p[j] -= lr * gj / (sqrt(m2[j]) + cfg->rms_eps);
        } else {
            m1[j] = cfg->momentum * m1[j] - lr * gj;
            p[j] += m1[j];
        }
    }
    orc_unpack(p, g);
    renormalize(g);
    free(p);
    return 0;
}
