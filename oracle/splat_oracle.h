/*
 * splat_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference hot path (arXiv 2504.12905 "LM-RS",
 * CPU reference /root/reference/proj).  Built into oracle/liboracle.so and
 * driven from Python via oracle/cpu_bind.py with prefix "orc_"; it exports
 * the same entry points as oracle/ref_capi.cpp (prefix "ref_") so tests can
 * run either checker.  Pinned against the real reference by
 * tests/test_oracle.py (golden fixtures in tests/golden/ made by
 * tests/golden/make_golden.py from oracle/_ref).
 *
 * Never linked or loaded by the product (paper_2504_12905_b200/).
 */
#ifndef SPLAT_ORACLE_H
#define SPLAT_ORACLE_H

#include "slm_types.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);
void orc_set_threads(int n);
int orc_threads(void);

void* orc_rng_new(uint64_t seed);
void orc_rng_free(void* r);
uint64_t orc_rng_next(void* r);

int orc_random_init(int count, const double* cube_min, const double* cube_max, void* rng,
                    slm_gaussians* out);
int orc_ring_camera(double angle, double radius, double height, int size, slm_camera* out);
int orc_toy_scene(int gaussians, int train_cams, int test_cams, int image_size, uint64_t seed,
                  slm_gaussians* gt, slm_camera* cams_out, float* images_out);

int orc_prepare(const slm_gaussians* g, const slm_camera* cam, double* mean2d, double* conic,
                double* opacity, double* color, double* depth, double* radius, int32_t* valid);
int orc_bin_and_sort(const slm_gaussians* g, const slm_camera* cam, int32_t* offsets,
                     int32_t* indices, int64_t capacity, int64_t* n_entries);
int orc_render_full(const slm_gaussians* g, const slm_camera* cam, double* image,
                    double* transmittance, int32_t* contrib);

void* orc_build_sample_plan(const slm_camera* cams, int n_cams, int samples_per_tile, int dist,
                            int lane_width, void* rng, const double* const* aux_image,
                            const int32_t* const* aux_contrib, const double* const* aux_gt);
void* orc_exhaustive_plan(const slm_camera* cams, int n_cams);
void orc_plan_free(void* p);
int orc_plan_views(void* p);
int64_t orc_plan_total(void* p);
void orc_plan_export(void* p, int32_t* view_camera, int64_t* view_offset, int32_t* px,
                     int32_t* py, int32_t* tile, double* weight);
int orc_estimate_loss(const slm_camera* cams, const slm_plan* plan,
                      const double* const* residual_fields, double* out);
int orc_kmeans_cameras(const slm_camera* cams, int n_cams, int k, uint64_t seed, int32_t* assign);
int orc_camera_features(const slm_camera* cams, int n_cams, double* feats);

void* orc_jac_new(const slm_gaussians* g, const slm_camera* cams, int n_cams,
                  const slm_plan* plan);
void orc_jac_free(void* j);
int64_t orc_jac_residual_dim(void* j);
int64_t orc_jac_param_dim(void* j);
int orc_jac_jvp(void* j, const double* v, double* out);
int orc_jac_vjp(void* j, const double* u, double* out);
int orc_jac_jtj_diag(void* j, double* out);
int orc_jac_gn_apply(void* j, double lambda, const double* p, double* out);
int orc_jac_weights(void* j, double* out);
int orc_jac_set_weights(void* j, const double* w);
int orc_jac_pcg(void* j, double lambda, const double* b, const double* minv, int iters, double* x,
                slm_pcg_result* res);
int orc_pcg_dense(const double* a, int n, const double* b, const double* minv, int iters,
                  double* x, slm_pcg_result* res);
double orc_learning_rate(const double* delta, int64_t n, int iteration, const slm_lm_config* cfg);
int orc_apply_update(slm_gaussians* g, const double* delta, double eta);

void* orc_train_new(const slm_camera* cams, int n_cams, const float* images);
void* orc_train_new_f64(const slm_camera* cams, int n_cams, const double* images);
void orc_train_free(void* t);
int orc_train_rebuild_clusters(void* t, int k, uint64_t seed);
int orc_train_set_clusters(void* t, const int32_t* assign, int n_cams, int k);
int orc_lm_step(slm_gaussians* g, void* t, const slm_lm_config* cfg, int iteration, void* rng,
                slm_step_report* report);
int orc_batch_loss(const slm_gaussians* g, const slm_camera* cams, int n_cams, const float* gts,
                   int loss, double ssim_weight, double* out);
double orc_mse(const double* a, const double* b, int w, int h);
double orc_psnr(const double* a, const double* b, int w, int h);
double orc_ssim(const double* a, const double* b, int w, int h);
int orc_full_gradient(const slm_gaussians* g, const slm_camera* cams, int n_cams, const float* gts, int loss,
                      double ssim_weight, double* out);
int orc_first_order_step(slm_gaussians* g, double* m1, double* m2, int64_t* step, const double* grad,
                         const slm_first_order_config* cfg);
void orc_ssim_diag_residuals(const double* a, const double* b, int w, int h, double* residual,
                             double* d_center);

#ifdef __cplusplus
}
#endif

#endif
