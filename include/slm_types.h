/*
 * slm_types.h — plain-C data layouts shared by the B200 library's C ABI
 * (slm_b200.h), the CPU oracle (oracle/) and the reference wrapper
 * (oracle/ref_capi.cpp).  No C++ or torch types: pointers + sizes only.
 *
 * Every struct mirrors a reference C++ type field for field:
 *   slm_camera      <- splatlm::Camera          proj/include/splatlm/core/types.hpp:61-75
 *   slm_gaussians   <- splatlm::GaussianSet     proj/include/splatlm/core/types.hpp:31-57
 *   slm_plan        <- sampling::SamplePlan     proj/include/splatlm/sampling/sample_plan.hpp:22-37
 *   slm_lm_config   <- solver::LmConfig         proj/include/splatlm/solver/lm.hpp:14-40
 *   slm_step_report <- solver::StepReport       proj/include/splatlm/solver/lm.hpp:42-50
 */
#ifndef SLM_TYPES_H
#define SLM_TYPES_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Flat parameter layout per Gaussian (types.hpp:15-20):
 * [mean(3), log_scale(3), rotation wxyz(4), opacity_logit(1), color(3)]. */
#define SLM_PARAMS_PER_GAUSSIAN 14
#define SLM_TILE 16

/* Pinhole camera, row-major world->camera rotation (types.hpp:61-75). */
typedef struct slm_camera {
    double world_to_cam[9];
    double translation[3];
    double fx, fy, cx, cy;
    double near_clip; /* reference default 0.2 (types.hpp:67) */
    int32_t width, height;
} slm_camera;

/* Caller-owned SoA parameter arrays (GaussianSet, types.hpp:31-57). */
typedef struct slm_gaussians {
    int32_t count;
    double* means;          /* 3*count */
    double* log_scales;     /* 3*count */
    double* rotations;      /* 4*count, (w,x,y,z) */
    double* opacity_logits; /* count */
    double* colors;         /* 3*count, SH level-0 coefficients */
} slm_gaussians;

/* ResidualDist (sample_plan.hpp:13). */
enum { SLM_DIST_UNIFORM = 0, SLM_DIST_RESIDUAL = 1, SLM_DIST_GAUSSIAN_COUNT = 2 };
/* LossKind (lm.hpp:12). */
enum { SLM_LOSS_MSE = 0, SLM_LOSS_MSE_SSIM = 1 };

/* Flattened SamplePlan: view v owns samples [view_offset[v], view_offset[v+1]).
 * Sample order inside a view is the reference emission order (tile-major,
 * sample_plan.cpp:96-168), so residual rows are (view, sample, channel). */
typedef struct slm_plan {
    int32_t n_views;
    int32_t samples_per_tile;
    int32_t dist;
    const int32_t* view_camera; /* [n_views] index into the camera batch */
    const int64_t* view_offset; /* [n_views+1] */
    const int32_t* px;          /* [total] */
    const int32_t* py;          /* [total] */
    const int32_t* tile;        /* [total] */
    const double* weight;       /* [total] importance weight 1/q */
} slm_plan;

/* LmConfig (lm.hpp:14-40) with the reference defaults documented there. */
typedef struct slm_lm_config {
    double damping;               /* 0.1 */
    int32_t pcg_iters_initial;    /* 3 */
    int32_t pcg_iters_late;       /* 8 */
    int32_t pcg_switch_iteration; /* 50 */
    int32_t batch_size_initial;   /* 8 */
    int32_t batch_size_late;      /* 8 */
    int32_t batch_switch_iteration; /* 50 */
    int32_t samples_per_tile;     /* 32 */
    int32_t sample_lane_width;    /* 32 */
    double lr_cap;                /* 0.2 */
    double warmup_lr;             /* 0.05 */
    int32_t warmup_iterations;    /* 10 */
    int32_t dist;                 /* SLM_DIST_UNIFORM */
    int32_t loss;                 /* SLM_LOSS_MSE */
    double ssim_weight;           /* 0.2 */
} slm_lm_config;

/* StepReport (lm.hpp:42-50); batch is caller-allocated with batch_capacity. */
typedef struct slm_step_report {
    int32_t iteration;
    double loss_before;
    double loss_after;
    double eta;
    int32_t pcg_iterations;
    int32_t breakdown;
    int32_t batch_size;
    int32_t* batch;
    int32_t batch_capacity;
} slm_step_report;

/* PcgResult (pcg.hpp:9-14) minus x, which is an output buffer. */
typedef struct slm_pcg_result {
    int32_t iterations;
    int32_t breakdown;
    double rel_residual;
} slm_pcg_result;

/* baselines::FirstOrderConfig (baselines/first_order.hpp:12-37); per-group
 * learning rates in raw (pre-activation) coordinates. */
enum { SLM_FO_ADAM = 0, SLM_FO_RMSPROP = 1, SLM_FO_SGD_MOMENTUM = 2 };
typedef struct slm_first_order_config {
    int32_t kind;                 /* SLM_FO_ADAM */
    double lr_mean;               /* 1.6e-3 */
    double lr_color;              /* 2.5e-2 */
    double lr_opacity;            /* 5e-2 */
    double lr_scale;              /* 5e-3 */
    double lr_rotation;           /* 1e-3 */
    double adam_beta1;            /* 0.9 */
    double adam_beta2;            /* 0.999 */
    double adam_eps;              /* 1e-15 */
    double rms_decay;             /* 0.99 */
    double rms_eps;               /* 1e-15 */
    double momentum;              /* 0.99 */
    double mean_lr_final_factor;  /* 0.01 */
    int32_t decay_iterations;     /* 0 = no decay */
    int32_t loss;                 /* SLM_LOSS_MSE */
    double ssim_weight;           /* 0.2 */
} slm_first_order_config;

/* MetricReport (metrics/image_metrics.hpp:7-11). */
typedef struct slm_metric_report {
    double mse;
    double psnr;
    double ssim;
} slm_metric_report;

#ifdef __cplusplus
}
#endif

#endif /* SLM_TYPES_H */
