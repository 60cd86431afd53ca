/*
 * slm_b200.h — C ABI of the B200-native LM/PCG hot path (libslm_b200.so).
 *
 * The entry points are what a binding of the reference's C++ API would call:
 * each one names the reference function/method it replaces (paths relative
 * to /root/reference/proj).  Conventions:
 *   - every function returns 0 on success, else an error code
 *     (SLM_E_INVALID <- std::invalid_argument, SLM_E_DOMAIN <- std::domain_error,
 *      SLM_E_RUNTIME <- std::runtime_error, SLM_E_CUDA on a CUDA/NCCL failure);
 *     slm_last_error() returns the thread's last message.  No exceptions cross
 *     the ABI.
 *   - host buffers are caller-owned; ParamVectors are the reference's AoS
 *     14-stride layout (types.hpp:11-20) in f64; residual vectors are ordered
 *     (view, sample, channel) (jacobian.hpp:13-15).
 *   - "_dev" variants take device pointers to f32 SoA [14][Gp] vectors
 *     (slm_scene_count returns Gp) and never synchronise the host.
 *   - a context owns one CUDA stream; calls on one context are not
 *     thread-safe (reference: SPEC.md:370).
 * There is no CPU fallback: without a CUDA device every compute call fails
 * with SLM_E_CUDA.
 */
#ifndef SLM_B200_H
#define SLM_B200_H

#include <stddef.h>
#include <stdint.h>

#include "slm_types.h"

#ifdef __cplusplus
extern "C" {
#endif

enum { SLM_OK = 0, SLM_E_INVALID = 1, SLM_E_DOMAIN = 2, SLM_E_RUNTIME = 3, SLM_E_CUDA = 4 };

typedef struct slm_context slm_context;   /* device + stream + optional NCCL comm */
typedef struct slm_scene slm_scene;       /* device-resident GaussianSet (types.hpp:31-57) */
typedef struct slm_jacobian slm_jacobian; /* autodiff::SampledJacobian (jacobian.hpp:25-76) */
typedef struct slm_train slm_train;       /* solver::TrainData (lm.hpp:53-60) */
typedef struct slm_rng slm_rng;           /* std::mt19937_64 shared by init/batch/sampler */
typedef struct slm_plan_h slm_plan_h;     /* sampling::SamplePlan owned by the library */

const char* slm_last_error(void);
int slm_version(void);
int slm_device_count(int* out);

/* ---- context (no reference counterpart: the reference is one process, host threads only) */
int slm_context_create(int device, slm_context** out);
int slm_context_destroy(slm_context* ctx);
int slm_context_synchronize(slm_context* ctx);
/* Multi-GPU view sharding: rank 0 creates the id, every rank calls init_comm. */
int slm_nccl_unique_id(uint8_t out[128]);
int slm_context_init_comm(slm_context* ctx, const uint8_t id[128], int rank, int world);
int slm_context_rank(slm_context* ctx, int* rank, int* world);
/* In-process rank group: `world` contexts of ONE process (on one GPU or several),
 * each driven by its own host thread, joined with slm_context_init_local; their
 * collectives sum the ranks' vectors in rank order.  The same view-sharded code
 * path as NCCL, runnable on a single GPU (tests). */
typedef struct slm_local_group slm_local_group;
int slm_local_group_create(int world, slm_local_group** out);
void slm_local_group_destroy(slm_local_group* group);
int slm_context_init_local(slm_context* ctx, slm_local_group* group, int rank);
/* world > 1: the J^T W J p product's chain runs over this many Gaussian chunks,
 * each chunk's allreduce overlapping the next chunk (default 4). */
int slm_context_set_comm_chunks(slm_context* ctx, int chunks);
/* J^T / diag(J^T W J) accumulation order.  on (the default): every (view,
 * Gaussian)'s per-entry contributions are summed in a fixed per-plan order, so
 * jvp / vjp / jtj_diag / gn_apply / pcg / lm_step are bitwise reproducible run
 * to run (the reference's determinism contract, jacobian.cpp:19-21,246-247,
 * test_solver.cpp:268-286).  off: float red.global.add (order follows the
 * scheduler).  Takes effect at the next plan (Jacobian / lm_step). */
int slm_context_set_deterministic(slm_context* ctx, int on);
/* The sampled pixels of this context's last lm_step (this rank's views), in plan
 * order (view, tile, draw) -- drawn on the host (uniform) or on the device from
 * the FP64 render's CDFs (weighted) -- with their residual weights
 * (1/q)/N_total as the products use them (f32, mse loss).  Call with capacity 0
 * to get n. */
int slm_context_last_samples(slm_context* ctx, int64_t capacity, int64_t* n, int32_t* px, int32_t* py,
                             float* weight);
/* Counters of this context's last lm_step: [views, sum_v G_v, tile-list entries,
 * samples, pixels, PCG iterations, sum_v G_v and entries after the update]. */
int slm_context_step_stats(slm_context* ctx, int64_t out[8]);
/* Per-stage CUDA-event timings of the last lm_step / gn_apply (ms). */
int slm_context_timings(slm_context* ctx, double* out, int capacity, int* n);

/* ---- RNG: std::mt19937_64 (io/run.cpp:126-127) */
int slm_rng_create(uint64_t seed, slm_rng** out);
void slm_rng_destroy(slm_rng* rng);
uint64_t slm_rng_next(slm_rng* rng);
/* Engine state in libstdc++'s text form (operator<< / >>), so a C++ caller's
 * own std::mt19937_64 can drive lm_step / build_sample_plan. */
int slm_rng_get_state(slm_rng* rng, char* buf, int64_t capacity, int64_t* length);
int slm_rng_set_state(slm_rng* rng, const char* text);
/* Contiguous slice [lo, hi) of an n-view batch owned by `rank` of `world`. */
int slm_view_slice(int n, int rank, int world, int* lo, int* hi);

/* ---- scene (GaussianSet) */
int slm_scene_create(slm_context* ctx, const slm_gaussians* host, slm_scene** out);
void slm_scene_destroy(slm_scene* s);
int slm_scene_upload(slm_scene* s, const slm_gaussians* host);
int slm_scene_download(slm_scene* s, slm_gaussians* host);
int slm_scene_count(slm_scene* s, int* count, int* padded);
/* GaussianSet::apply_update (types.cpp:48-60): beta += eta*delta, re-normalise. */
int slm_scene_apply_update(slm_scene* s, const double* delta_aos, double eta);

/* ---- render (render/rasterizer.hpp) */
/* render::bin_and_sort (rasterizer.hpp:154-156): CSR tile lists, offsets[tiles+1]. */
int slm_bin_and_sort(slm_context* ctx, const slm_gaussians* g, const slm_camera* cam,
                     int32_t* offsets, int32_t* indices, int64_t capacity, int64_t* n_entries);
/* render::prepare_camera value parts (rasterizer.cpp:10-19), f32 records -> f64. */
int slm_prepare(slm_context* ctx, const slm_gaussians* g, const slm_camera* cam, double* mean2d,
                double* conic, double* opacity, double* color, double* depth, double* radius,
                int32_t* valid);
/* render::render_full (rasterizer.cpp:93-95); any output may be NULL. */
int slm_render_full(slm_context* ctx, const slm_gaussians* g, const slm_camera* cam, double* image,
                    double* transmittance, int32_t* contrib);
/* render::render_pixel (rasterizer.hpp:160-165, rasterizer.cpp:52-60): blend_pixel at pixel
 * centre (px, py) over an explicitly ordered list of prepared splats (render::SplatD,
 * 10 doubles each: mean2d x, y, conic a, b, c, opacity, colour r, g, b, unused).
 * out = {r, g, b, transmittance}.  Computed on the device in FP64. */
int slm_render_pixel(slm_context* ctx, int n, const double* splats, double px, double py, double out[4],
                     int32_t* contrib);
/* render::render_with_context (rasterizer.hpp:175, rasterizer.cpp:62-91): the FP64 render
 * of a camera from caller-prepared splats (layout as slm_render_pixel) and their tile
 * grid as CSR (offsets[tiles + 1], indices[offsets[tiles]]). */
int slm_render_splats(slm_context* ctx, const slm_camera* cam, int n_splats, const double* splats,
                      const int32_t* offsets, const int32_t* indices, double* image, double* transmittance,
                      int32_t* contrib);
/* render::residuals (rasterizer.cpp:97-104): out = rendered - truth over n doubles (host). */
int slm_residuals(const double* rendered, const double* truth, int64_t n, double* out);
int slm_scene_render(slm_scene* s, const slm_camera* cam, float* image, float* transmittance,
                     int32_t* contrib);

/* ---- sampling (sampling/ headers), host side with the reference's libstdc++ RNG */
/* build_sample_plan (sample_plan.cpp:62-171); aux_* are per-camera rendered
 * image (H*W*3), contrib counts (H*W) and ground truth (H*W*3), only read for
 * the weighted distributions. */
int slm_build_sample_plan(const slm_camera* cams, int n_cams, int samples_per_tile, int dist,
                          int lane_width, slm_rng* rng, const double* const* aux_image,
                          const int32_t* const* aux_contrib, const double* const* aux_gt,
                          slm_plan_h** out);
int slm_exhaustive_plan(const slm_camera* cams, int n_cams, slm_plan_h** out); /* :173-197 */
void slm_plan_destroy(slm_plan_h* p);
int slm_plan_size(slm_plan_h* p, int* n_views, int64_t* total);
int slm_plan_export(slm_plan_h* p, int32_t* view_camera, int64_t* view_offset, int32_t* px,
                    int32_t* py, int32_t* tile, double* weight);
/* estimate_loss (sample_plan.cpp:199-222) on host residual fields. */
int slm_estimate_loss(const slm_camera* cams, const slm_plan* plan,
                      const double* const* residual_fields, double* out);
/* camera_features / kmeans_cameras / sample_view_batch (view_sampler.cpp:10-184). */
int slm_camera_features(const slm_camera* cams, int n_cams, double* feats);
int slm_kmeans_cameras(const slm_camera* cams, int n_cams, int k, uint64_t seed, int32_t* assign);
int slm_sample_view_batch(const int32_t* assign, int n_cams, int k, slm_rng* rng, int32_t* batch);

/* ---- SampledJacobian (autodiff/jacobian.hpp:25-76) */
int slm_jacobian_create(slm_context* ctx, const slm_gaussians* g, const slm_camera* cams, int n_cams,
                        const slm_plan* plan, slm_jacobian** out);
int slm_jacobian_create_scene(slm_scene* s, const slm_camera* cams, int n_cams,
                              const slm_plan* plan, slm_jacobian** out);
void slm_jacobian_destroy(slm_jacobian* j);
int slm_jacobian_dims(slm_jacobian* j, int64_t* residual_dim, int64_t* param_dim);
int slm_jacobian_jvp(slm_jacobian* j, const double* v, double* out);          /* :191-211 */
int slm_jacobian_vjp(slm_jacobian* j, const double* u, double* out);          /* :219-264 */
int slm_jacobian_jtj_diag(slm_jacobian* j, double* out);                      /* :272-337 */
int slm_jacobian_gn_apply(slm_jacobian* j, double lambda, const double* p, double* out); /* :339-344 */
int slm_jacobian_weights(slm_jacobian* j, double* out);                       /* jacobian.hpp:43 */
int slm_jacobian_set_weights(slm_jacobian* j, const double* w);              /* :121-125 */
/* Device-resident products on f32 SoA vectors (the hot path lm_step uses). */
int slm_jacobian_gn_apply_dev(slm_jacobian* j, float lambda, const float* d_p, float* d_out);
/* pcg_solve (pcg.cpp:10-53) on (J^T W J + lambda I) x = b, entirely on device. */
int slm_jacobian_pcg(slm_jacobian* j, double lambda, const double* b, const double* minv,
                     int max_iters, double* x, slm_pcg_result* res);

/* ---- PCG on a caller-supplied operator (pcg.hpp:16-23): vector algebra on
 * the device, the operator callback receives/returns host f64 vectors. */
typedef void (*slm_apply_fn)(void* user, const double* p, double* out);
int slm_pcg_solve(slm_context* ctx, slm_apply_fn apply, void* user, const double* b,
                  const double* minv, int64_t n, int max_iters, double* x, slm_pcg_result* res);

/* ---- solver (solver/lm.hpp) */
int slm_learning_rate(slm_context* ctx, const double* delta, int64_t n, int iteration,
                      const slm_lm_config* cfg, double* eta);                 /* lm.cpp:26-37 */
void slm_default_lm_config(slm_lm_config* cfg);
/* TrainData with the f32 dataset images (H*W*3 per camera) resident in HBM. */
int slm_train_create(slm_context* ctx, const slm_camera* cams, int n_cams, const float* images,
                     slm_train** out);
void slm_train_destroy(slm_train* t);
int slm_train_rebuild_clusters(slm_train* t, int k, uint64_t seed);       /* lm.cpp:21-24 */
int slm_train_set_clusters(slm_train* t, const int32_t* assign, int k);
int slm_train_clusters(slm_train* t, int32_t* assign, int* k);
/* lm_step (lm.cpp:56-157) on a device-resident scene. */
int slm_lm_step(slm_scene* s, slm_train* t, const slm_lm_config* cfg, int iteration, slm_rng* rng,
                slm_step_report* report);
/* Drop-in host form: state is the caller's GaussianSet, updated in place. */
int slm_lm_step_host(slm_context* ctx, slm_gaussians* state, slm_train* t,
                     const slm_lm_config* cfg, int iteration, slm_rng* rng,
                     slm_step_report* report);
/* batch_loss (lm.cpp:39-54), MSE; cameras index the TrainData. */
int slm_batch_loss(slm_scene* s, slm_train* t, const int32_t* cams, int n, double* out);
/* batch_loss with the loss kind (SLM_LOSS_MSE / SLM_LOSS_MSE_SSIM) and SSIM weight. */
int slm_batch_loss_kind(slm_scene* s, slm_train* t, const int32_t* cams, int n, int loss, double ssim_weight,
                        double* out);

/* ---- first-order baselines (baselines/first_order.hpp) on the device */
typedef struct slm_first_order slm_first_order; /* FirstOrderState: f64 moments in HBM + step */
void slm_default_first_order_config(slm_first_order_config* cfg);
/* full_gradient (first_order.cpp:11-44) over every camera of the TrainData:
 * exhaustive plan, dL/dr = 2/M (r + w s s'), J^T on the device; AoS f64 out. */
int slm_full_gradient(slm_scene* s, slm_train* t, int loss, double ssim_weight, double* grad_aos);
/* Optimizer state bound to a device-resident scene (zero moments, step 0). */
int slm_first_order_create(slm_scene* s, slm_first_order** out);
void slm_first_order_destroy(slm_first_order* f);
int slm_first_order_moments(slm_first_order* f, double* m1_aos, double* m2_aos, int64_t* step);
int slm_first_order_set_moments(slm_first_order* f, const double* m1_aos, const double* m2_aos, int64_t step);
/* first_order_step (first_order.cpp:115-122) with a caller gradient (AoS f64). */
int slm_first_order_apply(slm_first_order* f, const double* grad_aos, const slm_first_order_config* cfg);
/* One train_run iteration (run.cpp:176-182): full_gradient + step + batch_loss
 * over all TrainData cameras (train_loss may be NULL to skip the loss). */
int slm_first_order_step(slm_first_order* f, slm_train* t, const slm_first_order_config* cfg,
                         double* train_loss);

/* ---- metrics (metrics/image_metrics.hpp, io/run.cpp:77-92), computed on the device */
/* metrics::evaluate (image_metrics.cpp:180-186) on two interleaved-RGB f64 images. */
int slm_evaluate(slm_context* ctx, const double* rendered, const double* ground_truth, int width,
                 int height, slm_metric_report* out);
/* metrics::ssim_diag_residuals (image_metrics.cpp:141-178): per pixel and channel
 * s = sqrt(max(0, 1 - local SSIM)) and ds/d(centre pixel of a); H*W*3 f64 each. */
int slm_ssim_diag_residuals(slm_context* ctx, const double* a, const double* b, int width, int height,
                            double* residual, double* d_center);
/* io::evaluate_split: render every camera of the split (TrainData images are
 * the ground truth) and average mse / psnr / ssim over the cameras. */
int slm_evaluate_split(slm_scene* s, slm_train* split, slm_metric_report* out);

/* ---- checkpoints (io/checkpoint.hpp; byte format SPLMGS01, checkpoint.cpp:12-82) */
int slm_save_checkpoint(const char* path, const slm_gaussians* g); /* + path.meta.txt */
int slm_checkpoint_count(const char* path, int* count);
int slm_load_checkpoint(const char* path, slm_gaussians* out);     /* out->count must match */

/* ---- io helpers the harness uses (io/dataset.cpp:138-166, io/scene_gen.cpp) */
int slm_random_init(int count, const double* cube_min, const double* cube_max, slm_rng* rng,
                    slm_gaussians* out);
/* io::generate_toy_scene's ground-truth Gaussians (scene_gen.cpp:38-71), seeded
 * std::mt19937_64(seed); cameras: slm_ring_camera, images: slm_render. */
int slm_toy_gaussians(int count, uint64_t seed, slm_gaussians* out);
int slm_ring_camera(double angle, double radius, double height, int width, int height_px,
                    slm_camera* out);

/* ---- instrumentation (no reference counterpart) */
/* Run the context's work on a caller stream (e.g. torch.cuda.Stream().cuda_stream),
 * so the caller's CUDA events bracket the library's kernels. */
int slm_context_set_stream(slm_context* ctx, void* stream);
int slm_context_set_timing(slm_context* ctx, int on);
const char* slm_context_timing_names(slm_context* ctx); /* comma-separated stage names */
long long slm_launch_count(void); /* kernels launched by this library so far */
/* CUDA events around the three kernels of every J^T W J p product
 * (tangents, fused raster, chain); collect returns summed ms and the count. */
int slm_context_set_profiling(slm_context* ctx, int on);
int slm_context_profile_collect(slm_context* ctx, double out[3], int* n);
int slm_scene_beta_ptrs(slm_scene* s, double** beta, float** beta32);
int slm_jacobian_device_ptrs(slm_jacobian* j, void* stream_out[1]);
/* [views, sum_v G_v (valid view-Gaussian pairs), tile-list entries, samples, warp groups, tiles] */
int slm_jacobian_stats(slm_jacobian* j, int64_t* out);
/* Diagnostic: blend-mask density / lane-balance counters (18 values, see
 * raster.cu k_mask_stats); used by tools/mask_stats.py. */
int slm_jacobian_mask_stats(slm_jacobian* j, uint64_t* out);
/* Diagnostic: k_render work counters over the given views (10 values: entry
 * iterations, entries past the warp box test, live pixel-entry gates, blends,
 * staged entries -- per thread --, the batch's entries, pixels, tiles, and per
 * warp the entries past an exact ellipse/half-tile test and the entries some
 * pixel of the warp blended). */
int slm_debug_render_stats(slm_scene* s, const slm_camera* cams, int n_cams, uint64_t* out);
/* Diagnostic: the NCCL seam in one process (a one-rank communicator on the
 * context's device): dlopen + unique id + init, then the product's two
 * collectives (allreduce of f32 and f64 vectors, the grouped row allreduce) on
 * known data.  out[0] = largest |result - input| (0 for one rank), out[1] =
 * elements checked.  Fails with the NCCL error when the library is missing. */
int slm_debug_nccl_selftest(slm_context* ctx, double* out);

#ifdef __cplusplus
}
#endif

#endif /* SLM_B200_H */
