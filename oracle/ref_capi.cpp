// ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" wrapper around the UNMODIFIED reference library
// (/root/reference/proj, built by oracle/Makefile into oracle/_ref/), so that
// Python tests, the golden-vector generator (tests/golden/make_golden.py) and
// bench.py's reference arm can drive the reference through ctypes.  Nothing in
// the product (paper_2504_12905_b200/) links or loads this.
//
// Each entry point names the reference function it forwards to.

#include <algorithm>
#include <cstring>
#include <exception>
#include <random>
#include <span>
#include <string>
#include <vector>

#include "slm_types.h"
#include "splatlm/autodiff/jacobian.hpp"
#include "splatlm/baselines/first_order.hpp"
#include "splatlm/core/parallel.hpp"
#include "splatlm/io/checkpoint.hpp"
#include "splatlm/io/dataset.hpp"
#include "splatlm/io/run.hpp"
#include "splatlm/io/scene_gen.hpp"
#include "splatlm/metrics/image_metrics.hpp"
#include "splatlm/render/rasterizer.hpp"
#include "splatlm/sampling/sample_plan.hpp"
#include "splatlm/sampling/view_sampler.hpp"
#include "splatlm/solver/lm.hpp"
#include "splatlm/solver/pcg.hpp"

using namespace splatlm;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

Camera to_cam(const slm_camera& c) {
    Camera cam;
    for (int i = 0; i < 9; ++i) cam.world_to_cam[i] = c.world_to_cam[i];
    for (int i = 0; i < 3; ++i) cam.translation[i] = c.translation[i];
    cam.fx = c.fx;
    cam.fy = c.fy;
    cam.cx = c.cx;
    cam.cy = c.cy;
    cam.near_clip = c.near_clip;
    cam.width = c.width;
    cam.height = c.height;
    return cam;
}

slm_camera from_cam(const Camera& cam) {
    slm_camera c{};
    for (int i = 0; i < 9; ++i) c.world_to_cam[i] = cam.world_to_cam[i];
    for (int i = 0; i < 3; ++i) c.translation[i] = cam.translation[i];
    c.fx = cam.fx;
    c.fy = cam.fy;
    c.cx = cam.cx;
    c.cy = cam.cy;
    c.near_clip = cam.near_clip;
    c.width = cam.width;
    c.height = cam.height;
    return c;
}

std::vector<Camera> to_cams(const slm_camera* c, int n) {
    std::vector<Camera> v;
    for (int i = 0; i < n; ++i) v.push_back(to_cam(c[i]));
    return v;
}

GaussianSet to_set(const slm_gaussians& g) {
    GaussianSet s = GaussianSet::zeros(g.count);
    std::copy(g.means, g.means + 3 * g.count, s.means.begin());
    std::copy(g.log_scales, g.log_scales + 3 * g.count, s.log_scales.begin());
    std::copy(g.rotations, g.rotations + 4 * g.count, s.rotations.begin());
    std::copy(g.opacity_logits, g.opacity_logits + g.count, s.opacity_logits.begin());
    std::copy(g.colors, g.colors + 3 * g.count, s.colors.begin());
    return s;
}

void from_set(const GaussianSet& s, slm_gaussians& g) {
    std::copy(s.means.begin(), s.means.end(), g.means);
    std::copy(s.log_scales.begin(), s.log_scales.end(), g.log_scales);
    std::copy(s.rotations.begin(), s.rotations.end(), g.rotations);
    std::copy(s.opacity_logits.begin(), s.opacity_logits.end(), g.opacity_logits);
    std::copy(s.colors.begin(), s.colors.end(), g.colors);
}

sampling::SamplePlan to_plan(const slm_plan& p) {
    sampling::SamplePlan plan;
    plan.samples_per_tile = p.samples_per_tile;
    plan.dist = static_cast<sampling::ResidualDist>(p.dist);
    for (int v = 0; v < p.n_views; ++v) {
        sampling::SampleView view;
        view.camera = p.view_camera[v];
        for (int64_t s = p.view_offset[v]; s < p.view_offset[v + 1]; ++s) {
            view.px.push_back(p.px[s]);
            view.py.push_back(p.py[s]);
            view.tile.push_back(p.tile[s]);
            view.weight.push_back(p.weight[s]);
        }
        plan.views.push_back(std::move(view));
    }
    return plan;
}

solver::LmConfig to_cfg(const slm_lm_config& c) {
    solver::LmConfig cfg;
    cfg.damping = c.damping;
    cfg.pcg_iters_initial = c.pcg_iters_initial;
    cfg.pcg_iters_late = c.pcg_iters_late;
    cfg.pcg_switch_iteration = c.pcg_switch_iteration;
    cfg.batch_size_initial = c.batch_size_initial;
    cfg.batch_size_late = c.batch_size_late;
    cfg.batch_switch_iteration = c.batch_switch_iteration;
    cfg.samples_per_tile = c.samples_per_tile;
    cfg.sample_lane_width = c.sample_lane_width;
    cfg.lr_cap = c.lr_cap;
    cfg.warmup_lr = c.warmup_lr;
    cfg.warmup_iterations = c.warmup_iterations;
    cfg.dist = static_cast<sampling::ResidualDist>(c.dist);
    cfg.loss = static_cast<solver::LossKind>(c.loss);
    cfg.ssim_weight = c.ssim_weight;
    return cfg;
}

struct RefPlan {
    sampling::SamplePlan plan;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_threads(int n) { set_thread_count(n); }
int ref_threads() { return thread_count(); }

void ref_default_lm_config(slm_lm_config* out) {
    solver::LmConfig c;
    out->damping = c.damping;
    out->pcg_iters_initial = c.pcg_iters_initial;
    out->pcg_iters_late = c.pcg_iters_late;
    out->pcg_switch_iteration = c.pcg_switch_iteration;
    out->batch_size_initial = c.batch_size_initial;
    out->batch_size_late = c.batch_size_late;
    out->batch_switch_iteration = c.batch_switch_iteration;
    out->samples_per_tile = c.samples_per_tile;
    out->sample_lane_width = c.sample_lane_width;
    out->lr_cap = c.lr_cap;
    out->warmup_lr = c.warmup_lr;
    out->warmup_iterations = c.warmup_iterations;
    out->dist = static_cast<int>(c.dist);
    out->loss = static_cast<int>(c.loss);
    out->ssim_weight = c.ssim_weight;
}

// ---- RNG (std::mt19937_64 shared by random_init / view batch / sampler) ----
void* ref_rng_new(uint64_t seed) { return new std::mt19937_64(seed); }
void ref_rng_free(void* r) { delete static_cast<std::mt19937_64*>(r); }
uint64_t ref_rng_next(void* r) { return (*static_cast<std::mt19937_64*>(r))(); }

// io::random_init (dataset.cpp:138-166)
int ref_random_init(int count, const double* cube_min, const double* cube_max, void* rng,
                    slm_gaussians* out) {
    return guarded([&] {
        const GaussianSet g = io::random_init(count, {cube_min[0], cube_min[1], cube_min[2]},
                                              {cube_max[0], cube_max[1], cube_max[2]},
                                              *static_cast<std::mt19937_64*>(rng));
        from_set(g, *out);
    });
}

// io::ring_camera (scene_gen.cpp:11-36)
int ref_ring_camera(double angle, double radius, double height, int size, slm_camera* out) {
    return guarded([&] { *out = from_cam(io::ring_camera(angle, radius, height, size)); });
}

// io::generate_toy_scene (scene_gen.cpp:38-86).  Images are the float32
// dataset buffers (H*W*3 each), train then test.
int ref_toy_scene(int gaussians, int train_cams, int test_cams, int image_size, uint64_t seed,
                  slm_gaussians* gt, slm_camera* cams_out, float* images_out) {
    return guarded([&] {
        std::mt19937_64 rng(seed);
        io::ToySceneConfig cfg;
        cfg.gaussians = gaussians;
        cfg.train_cameras = train_cams;
        cfg.test_cameras = test_cams;
        cfg.image_size = image_size;
        const io::ToyScene scene = io::generate_toy_scene(cfg, rng);
        from_set(scene.ground_truth, *gt);
        size_t k = 0;
        float* dst = images_out;
        for (const auto* ds : {&scene.train, &scene.test}) {
            for (size_t i = 0; i < ds->cameras.size(); ++i) {
                cams_out[k++] = from_cam(ds->cameras[i]);
                std::copy(ds->images[i].data.begin(), ds->images[i].data.end(), dst);
                dst += ds->images[i].data.size();
            }
        }
    });
}

// render::prepare_camera -> per-Gaussian PreparedSplat value parts
// (rasterizer.cpp:10-19, rasterizer.hpp:58-94)
int ref_prepare(const slm_gaussians* g, const slm_camera* cam, double* mean2d, double* conic,
                double* opacity, double* color, double* depth, double* radius, int32_t* valid) {
    return guarded([&] {
        const auto ctx = render::prepare_camera(to_set(*g), to_cam(*cam));
        for (int i = 0; i < g->count; ++i) {
            const auto& s = ctx.splats[i];
            mean2d[2 * i] = s.mean2d.x;
            mean2d[2 * i + 1] = s.mean2d.y;
            conic[3 * i] = s.conic_a;
            conic[3 * i + 1] = s.conic_b;
            conic[3 * i + 2] = s.conic_c;
            opacity[i] = s.opacity;
            for (int c = 0; c < 3; ++c) color[3 * i + c] = s.color[c];
            depth[i] = s.depth;
            radius[i] = s.radius;
            valid[i] = s.valid ? 1 : 0;
        }
    });
}

// render::bin_and_sort (rasterizer.hpp:154-156).  offsets has tiles+1
// entries; returns the entry count via *n_entries, writing at most capacity.
int ref_bin_and_sort(const slm_gaussians* g, const slm_camera* cam, int32_t* offsets,
                     int32_t* indices, int64_t capacity, int64_t* n_entries) {
    return guarded([&] {
        const auto grid = render::bin_and_sort(to_set(*g), to_cam(*cam));
        int64_t n = 0;
        offsets[0] = 0;
        for (size_t t = 0; t < grid.lists.size(); ++t) {
            for (int idx : grid.lists[t]) {
                if (n < capacity) indices[n] = idx;
                ++n;
            }
            offsets[t + 1] = static_cast<int32_t>(n);
        }
        *n_entries = n;
    });
}

// render::render_full (rasterizer.cpp:93-95)
int ref_render_full(const slm_gaussians* g, const slm_camera* cam, double* image,
                    double* transmittance, int32_t* contrib) {
    return guarded([&] {
        const auto out = render::render_full(to_set(*g), to_cam(*cam));
        std::copy(out.image.data.begin(), out.image.data.end(), image);
        if (transmittance)
            std::copy(out.final_transmittance.begin(), out.final_transmittance.end(),
                      transmittance);
        if (contrib) std::copy(out.contrib_count.begin(), out.contrib_count.end(), contrib);
    });
}

// ---- sampling ----
// sampling::build_sample_plan (sample_plan.cpp:62-171); aux arrays are only
// read for the weighted distributions (per camera: rendered image, contrib
// counts, ground truth, all H*W(*3)).
void* ref_build_sample_plan(const slm_camera* cams, int n_cams, int samples_per_tile, int dist,
                            int lane_width, void* rng, const double* const* aux_image,
                            const int32_t* const* aux_contrib, const double* const* aux_gt) {
    RefPlan* out = nullptr;
    std::vector<render::RenderOutput> rendered;
    std::vector<Image> gts;
    const int rc = guarded([&] {
        const auto cv = to_cams(cams, n_cams);
        std::vector<sampling::PlanAux> aux;
        if (dist != SLM_DIST_UNIFORM && aux_image) {
            rendered.resize(n_cams);
            gts.resize(n_cams);
            for (int i = 0; i < n_cams; ++i) {
                const int w = cv[i].width, h = cv[i].height;
                rendered[i].image = Image(w, h);
                std::copy(aux_image[i], aux_image[i] + 3 * w * h, rendered[i].image.data.begin());
                rendered[i].final_transmittance.assign(w * h, 1.0);
                rendered[i].contrib_count.assign(aux_contrib[i], aux_contrib[i] + w * h);
                gts[i] = Image(w, h);
                if (aux_gt) std::copy(aux_gt[i], aux_gt[i] + 3 * w * h, gts[i].data.begin());
                aux.push_back({&rendered[i], aux_gt ? &gts[i] : nullptr});
            }
        }
        auto plan = sampling::build_sample_plan(cv, samples_per_tile,
                                                static_cast<sampling::ResidualDist>(dist), aux,
                                                *static_cast<std::mt19937_64*>(rng), lane_width);
        out = new RefPlan{std::move(plan)};
    });
    return rc == 0 ? out : nullptr;
}

// sampling::exhaustive_plan (sample_plan.cpp:173-197)
void* ref_exhaustive_plan(const slm_camera* cams, int n_cams) {
    RefPlan* out = nullptr;
    guarded([&] { out = new RefPlan{sampling::exhaustive_plan(to_cams(cams, n_cams))}; });
    return out;
}

void ref_plan_free(void* p) { delete static_cast<RefPlan*>(p); }
int ref_plan_views(void* p) { return static_cast<int>(static_cast<RefPlan*>(p)->plan.views.size()); }
int64_t ref_plan_total(void* p) {
    return static_cast<int64_t>(static_cast<RefPlan*>(p)->plan.total_samples());
}
// Copy the plan out in the slm_plan flattened layout.
void ref_plan_export(void* p, int32_t* view_camera, int64_t* view_offset, int32_t* px,
                     int32_t* py, int32_t* tile, double* weight) {
    const auto& plan = static_cast<RefPlan*>(p)->plan;
    int64_t k = 0;
    for (size_t v = 0; v < plan.views.size(); ++v) {
        const auto& view = plan.views[v];
        view_camera[v] = view.camera;
        view_offset[v] = k;
        for (size_t s = 0; s < view.size(); ++s, ++k) {
            px[k] = view.px[s];
            py[k] = view.py[s];
            tile[k] = view.tile[s];
            weight[k] = view.weight[s];
        }
    }
    view_offset[plan.views.size()] = k;
}

// sampling::estimate_loss (sample_plan.cpp:199-222); residual fields H*W*3
// per plan view.
int ref_estimate_loss(const slm_camera* cams, const slm_plan* plan,
                      const double* const* residual_fields, double* out) {
    return guarded([&] {
        const auto p = to_plan(*plan);
        std::vector<Image> fields;
        for (int v = 0; v < plan->n_views; ++v) {
            const auto& cam = cams[plan->view_camera[v]];
            Image img(cam.width, cam.height);
            std::copy(residual_fields[v], residual_fields[v] + img.data.size(), img.data.begin());
            fields.push_back(std::move(img));
        }
        *out = sampling::estimate_loss(p, fields);
    });
}

// sampling::camera_features / kmeans_cameras / sample_view_batch
// (view_sampler.cpp:10-184).  Clusters are returned as assign[n_cams].
int ref_kmeans_cameras(const slm_camera* cams, int n_cams, int k, uint64_t seed,
                       int32_t* assign) {
    return guarded([&] {
        const auto cv = to_cams(cams, n_cams);
        const auto feats = sampling::camera_features(cv);
        const auto clusters = sampling::kmeans_cameras(feats, k, seed);
        for (size_t c = 0; c < clusters.size(); ++c)
            for (int i : clusters[c]) assign[i] = static_cast<int32_t>(c);
    });
}

// sampling::sample_view_batch (view_sampler.cpp:173-184) over the clusters
// given as assign[n_cams] in [0, k) (each cluster's members in index order).
int ref_sample_view_batch(const int32_t* assign, int n_cams, int k, void* rng, int32_t* batch) {
    return guarded([&] {
        std::vector<std::vector<int>> clusters(k);
        for (int i = 0; i < n_cams; ++i) clusters.at(assign[i]).push_back(i);
        const auto b = sampling::sample_view_batch(clusters, *static_cast<std::mt19937_64*>(rng));
        for (size_t i = 0; i < b.size(); ++i) batch[i] = b[i];
    });
}

int ref_camera_features(const slm_camera* cams, int n_cams, double* feats) {
    return guarded([&] {
        const auto f = sampling::camera_features(to_cams(cams, n_cams));
        for (int i = 0; i < n_cams; ++i)
            for (int d = 0; d < 6; ++d) feats[6 * i + d] = f[i].v[d];
    });
}

// ---- SampledJacobian (jacobian.hpp:25-76) ----
struct RefJac {
    autodiff::SampledJacobian jac;
};

void* ref_jac_new(const slm_gaussians* g, const slm_camera* cams, int n_cams,
                  const slm_plan* plan) {
    RefJac* out = nullptr;
    guarded([&] {
        const auto cv = to_cams(cams, n_cams);
        out = new RefJac{autodiff::SampledJacobian(to_set(*g), cv, to_plan(*plan))};
    });
    return out;
}
void ref_jac_free(void* j) { delete static_cast<RefJac*>(j); }
int64_t ref_jac_residual_dim(void* j) {
    return static_cast<int64_t>(static_cast<RefJac*>(j)->jac.residual_dim());
}
int64_t ref_jac_param_dim(void* j) {
    return static_cast<int64_t>(static_cast<RefJac*>(j)->jac.param_dim());
}
int ref_jac_jvp(void* j, const double* v, double* out) {
    return guarded([&] {
        auto& jac = static_cast<RefJac*>(j)->jac;
        ParamVector pv(v, v + jac.param_dim());
        jac.jvp(pv, std::span<double>(out, jac.residual_dim()));
    });
}
int ref_jac_vjp(void* j, const double* u, double* out) {
    return guarded([&] {
        auto& jac = static_cast<RefJac*>(j)->jac;
        const ParamVector r = jac.vjp(std::span<const double>(u, jac.residual_dim()));
        std::copy(r.begin(), r.end(), out);
    });
}
int ref_jac_jtj_diag(void* j, double* out) {
    return guarded([&] {
        const ParamVector r = static_cast<RefJac*>(j)->jac.jtj_diag();
        std::copy(r.begin(), r.end(), out);
    });
}
int ref_jac_gn_apply(void* j, double lambda, const double* p, double* out) {
    return guarded([&] {
        auto& jac = static_cast<RefJac*>(j)->jac;
        ParamVector pv(p, p + jac.param_dim());
        const ParamVector r = jac.gn_apply(lambda, pv);
        std::copy(r.begin(), r.end(), out);
    });
}
int ref_jac_weights(void* j, double* out) {
    return guarded([&] {
        const auto& w = static_cast<RefJac*>(j)->jac.residual_weights();
        std::copy(w.begin(), w.end(), out);
    });
}
int ref_jac_set_weights(void* j, const double* w) {
    return guarded([&] {
        auto& jac = static_cast<RefJac*>(j)->jac;
        jac.set_residual_weights(std::vector<double>(w, w + jac.residual_dim()));
    });
}
// solver::pcg_solve (pcg.cpp:10-53) on (J^T W J + lambda I)
int ref_jac_pcg(void* j, double lambda, const double* b, const double* minv, int iters,
                double* x, slm_pcg_result* res) {
    return guarded([&] {
        auto& jac = static_cast<RefJac*>(j)->jac;
        const size_t n = jac.param_dim();
        const auto r = solver::pcg_solve(
            [&](const ParamVector& p, ParamVector& out) { jac.gn_apply(lambda, p, out); },
            ParamVector(b, b + n), ParamVector(minv, minv + n), iters);
        std::copy(r.x.begin(), r.x.end(), x);
        res->iterations = r.iterations;
        res->breakdown = r.breakdown;
        res->rel_residual = r.rel_residual;
    });
}

// solver::pcg_solve on a dense row-major operator
int ref_pcg_dense(const double* a, int n, const double* b, const double* minv, int iters,
                  double* x, slm_pcg_result* res) {
    return guarded([&] {
        const auto r = solver::pcg_solve(
            [&](const ParamVector& p, ParamVector& out) {
                out.assign(n, 0.0);
                for (int i = 0; i < n; ++i) {
                    double acc = 0.0;
                    for (int k = 0; k < n; ++k) acc += a[i * n + k] * p[k];
                    out[i] = acc;
                }
            },
            ParamVector(b, b + n), ParamVector(minv, minv + n), iters);
        std::copy(r.x.begin(), r.x.end(), x);
        res->iterations = r.iterations;
        res->breakdown = r.breakdown;
        res->rel_residual = r.rel_residual;
    });
}

// solver::learning_rate (lm.cpp:26-37)
double ref_learning_rate(const double* delta, int64_t n, int iteration,
                         const slm_lm_config* cfg) {
    double eta = 0.0;
    guarded([&] { eta = solver::learning_rate(ParamVector(delta, delta + n), iteration, to_cfg(*cfg)); });
    return eta;
}

// GaussianSet::apply_update (types.cpp:48-60)
int ref_apply_update(slm_gaussians* g, const double* delta, double eta) {
    return guarded([&] {
        GaussianSet s = to_set(*g);
        s.apply_update(ParamVector(delta, delta + s.param_count()), eta);
        from_set(s, *g);
    });
}

// ---- TrainData + lm_step (lm.hpp:53-71) ----
struct RefTrain {
    solver::TrainData data;
};

// images: per camera H*W*3 float32 dataset buffers, widened like run.cpp:132
void* ref_train_new(const slm_camera* cams, int n_cams, const float* images) {
    RefTrain* t = new RefTrain;
    const float* src = images;
    for (int i = 0; i < n_cams; ++i) {
        const Camera cam = to_cam(cams[i]);
        t->data.cameras.push_back(cam);
        Image img(cam.width, cam.height);
        for (size_t k = 0; k < img.data.size(); ++k) img.data[k] = src[k];
        src += img.data.size();
        t->data.images.push_back(std::move(img));
    }
    return t;
}
// double-precision images (tests that need exact-zero residuals)
void* ref_train_new_f64(const slm_camera* cams, int n_cams, const double* images) {
    RefTrain* t = new RefTrain;
    const double* src = images;
    for (int i = 0; i < n_cams; ++i) {
        const Camera cam = to_cam(cams[i]);
        t->data.cameras.push_back(cam);
        Image img(cam.width, cam.height);
        std::copy(src, src + img.data.size(), img.data.begin());
        src += img.data.size();
        t->data.images.push_back(std::move(img));
    }
    return t;
}
void ref_train_free(void* t) { delete static_cast<RefTrain*>(t); }
int ref_train_rebuild_clusters(void* t, int k, uint64_t seed) {
    return guarded([&] { static_cast<RefTrain*>(t)->data.rebuild_clusters(k, seed); });
}
int ref_train_set_clusters(void* t, const int32_t* assign, int n_cams, int k) {
    return guarded([&] {
        auto& cl = static_cast<RefTrain*>(t)->data.clusters;
        cl.assign(k, {});
        for (int i = 0; i < n_cams; ++i) cl[assign[i]].push_back(i);
    });
}

int ref_lm_step(slm_gaussians* g, void* t, const slm_lm_config* cfg, int iteration, void* rng,
                slm_step_report* report) {
    return guarded([&] {
        GaussianSet s = to_set(*g);
        const auto r = solver::lm_step(s, static_cast<RefTrain*>(t)->data, to_cfg(*cfg),
                                       iteration, *static_cast<std::mt19937_64*>(rng));
        from_set(s, *g);
        report->iteration = r.iteration;
        report->loss_before = r.loss_before;
        report->loss_after = r.loss_after;
        report->eta = r.eta;
        report->pcg_iterations = r.pcg_iterations;
        report->breakdown = r.breakdown;
        report->batch_size = static_cast<int32_t>(r.batch.size());
        for (size_t i = 0; i < r.batch.size() && static_cast<int>(i) < report->batch_capacity; ++i)
            report->batch[i] = r.batch[i];
    });
}

// solver::batch_loss (lm.cpp:39-54); gts are float32 dataset buffers
int ref_batch_loss(const slm_gaussians* g, const slm_camera* cams, int n_cams, const float* gts,
                   int loss, double ssim_weight, double* out) {
    return guarded([&] {
        const auto cv = to_cams(cams, n_cams);
        std::vector<Image> imgs;
        const float* src = gts;
        for (const auto& cam : cv) {
            Image img(cam.width, cam.height);
            for (size_t k = 0; k < img.data.size(); ++k) img.data[k] = src[k];
            src += img.data.size();
            imgs.push_back(std::move(img));
        }
        *out = solver::batch_loss(to_set(*g), cv, imgs, static_cast<solver::LossKind>(loss), ssim_weight);
    });
}

// metrics::mse / psnr (image_metrics.cpp:108-119) on double images
double ref_mse(const double* a, const double* b, int w, int h) {
    Image ia(w, h), ib(w, h);
    std::copy(a, a + ia.data.size(), ia.data.begin());
    std::copy(b, b + ib.data.size(), ib.data.begin());
    return metrics::mse(ia, ib);
}
double ref_psnr(const double* a, const double* b, int w, int h) {
    Image ia(w, h), ib(w, h);
    std::copy(a, a + ia.data.size(), ia.data.begin());
    std::copy(b, b + ib.data.size(), ib.data.begin());
    return metrics::psnr(ia, ib);
}
double ref_ssim(const double* a, const double* b, int w, int h) {
    Image ia(w, h), ib(w, h);
    std::copy(a, a + ia.data.size(), ia.data.begin());
    std::copy(b, b + ib.data.size(), ib.data.begin());
    return metrics::ssim(ia, ib);
}
void ref_ssim_diag_residuals(const double* a, const double* b, int w, int h, double* residual,
                             double* d_center) {
    Image ia(w, h), ib(w, h);
    std::copy(a, a + ia.data.size(), ia.data.begin());
    std::copy(b, b + ib.data.size(), ib.data.begin());
    const auto r = metrics::ssim_diag_residuals(ia, ib);
    std::copy(r.residual.data.begin(), r.residual.data.end(), residual);
    std::copy(r.d_center.data.begin(), r.d_center.data.end(), d_center);
}
// baselines::full_gradient (first_order.cpp:11-44); gts are float32 dataset buffers
int ref_full_gradient(const slm_gaussians* g, const slm_camera* cams, int n_cams, const float* gts, int loss,
                      double ssim_weight, double* out) {
    return guarded([&] {
        const auto cv = to_cams(cams, n_cams);
        std::vector<Image> imgs;
        const float* src = gts;
        for (const auto& cam : cv) {
            Image img(cam.width, cam.height);
            for (size_t k = 0; k < img.data.size(); ++k) img.data[k] = src[k];
            src += img.data.size();
            imgs.push_back(std::move(img));
        }
        const auto grad = baselines::full_gradient(to_set(*g), cv, imgs, static_cast<solver::LossKind>(loss),
                                                   ssim_weight);
        std::copy(grad.begin(), grad.end(), out);
    });
}

static baselines::FirstOrderConfig to_fo(const slm_first_order_config& c) {
    baselines::FirstOrderConfig f;
    f.kind = static_cast<baselines::FirstOrderKind>(c.kind);
    f.lrs = {c.lr_mean, c.lr_color, c.lr_opacity, c.lr_scale, c.lr_rotation};
    f.adam_beta1 = c.adam_beta1;
    f.adam_beta2 = c.adam_beta2;
    f.adam_eps = c.adam_eps;
    f.rms_decay = c.rms_decay;
    f.rms_eps = c.rms_eps;
    f.momentum = c.momentum;
    f.mean_lr_final_factor = c.mean_lr_final_factor;
    f.decay_iterations = c.decay_iterations;
    f.loss = static_cast<solver::LossKind>(c.loss);
    f.ssim_weight = c.ssim_weight;
    return f;
}

void ref_default_first_order_config(slm_first_order_config* out) {
    const baselines::FirstOrderConfig f;
    *out = slm_first_order_config{static_cast<int32_t>(f.kind), f.lrs.mean, f.lrs.color, f.lrs.opacity,
                                  f.lrs.scale, f.lrs.rotation, f.adam_beta1, f.adam_beta2, f.adam_eps,
                                  f.rms_decay, f.rms_eps, f.momentum, f.mean_lr_final_factor,
                                  f.decay_iterations, static_cast<int32_t>(f.loss), f.ssim_weight};
}

// baselines::first_order_step (first_order.cpp:115-122) on caller-held moments
int ref_first_order_step(slm_gaussians* g, double* m1, double* m2, int64_t* step, const double* grad,
                         const slm_first_order_config* cfg) {
    return guarded([&] {
        GaussianSet s = to_set(*g);
        const size_t n = static_cast<size_t>(s.param_count());
        baselines::FirstOrderState st;
        st.m1.assign(m1, m1 + n);
        st.m2.assign(m2, m2 + n);
        st.step = static_cast<long>(*step);
        baselines::first_order_step(st, s, ParamVector(grad, grad + n), to_fo(*cfg));
        from_set(s, *g);
        std::copy(st.m1.begin(), st.m1.end(), m1);
        std::copy(st.m2.begin(), st.m2.end(), m2);
        *step = st.step;
    });
}
// io::train_run (run.cpp:120-212) on the toy scene; outputs under out_dir
int ref_train_run_toy(const char* out_dir, const char* optimizer, int iterations, uint64_t seed, int gaussians,
                      int eval_every, int deterministic, uint64_t scene_seed, int toy_gaussians, int train_cams,
                      int test_cams, int image_size, const slm_lm_config* lm, const slm_first_order_config* fo,
                      double* final_train_loss, double* final_test) {
    return guarded([&] {
        io::RunConfig cfg;
        cfg.scene = "toy";
        cfg.optimizer = optimizer;
        cfg.iterations = iterations;
        cfg.seed = seed;
        cfg.out_dir = out_dir;
        cfg.gaussians = gaussians;
        cfg.lm = to_cfg(*lm);
        cfg.first_order = to_fo(*fo);
        cfg.eval_every = eval_every;
        cfg.deterministic = deterministic != 0;
        cfg.scene_seed = scene_seed;
        cfg.toy.gaussians = toy_gaussians;
        cfg.toy.train_cameras = train_cams;
        cfg.toy.test_cameras = test_cams;
        cfg.toy.image_size = image_size;
        const auto r = io::train_run(cfg);
        *final_train_loss = r.final_train_loss;
        final_test[0] = r.final_test.mse;
        final_test[1] = r.final_test.psnr;
        final_test[2] = r.final_test.ssim;
    });
}

// io::load_checkpoint / save_checkpoint (checkpoint.cpp:45-82)
int ref_load_checkpoint(const char* path, double* params_aos, int64_t capacity, int64_t* count) {
    return guarded([&] {
        const GaussianSet g = io::load_checkpoint(path);
        *count = g.count;
        const auto p = g.pack();
        if (static_cast<int64_t>(p.size()) <= capacity) std::copy(p.begin(), p.end(), params_aos);
    });
}
int ref_save_checkpoint(const char* path, const double* params_aos, int64_t count) {
    return guarded([&] {
        io::save_checkpoint(path, GaussianSet::unpack(ParamVector(params_aos, params_aos + 14 * count)));
    });
}

}  // extern "C"
