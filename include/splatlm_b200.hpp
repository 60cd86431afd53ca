// splatlm_b200.hpp — header-only C++ adapter: the reference's own solver API
// (proj/include/splatlm/**) served by libslm_b200.so through the C ABI.
//
// Include it INSIDE the reference tree (it uses the reference's types:
// splatlm::GaussianSet, Camera, sampling::SamplePlan, solver::LmConfig,
// solver::TrainData, solver::StepReport) and link libslm_b200.so.  A caller
// switches from the CPU path to the B200 path by changing the namespace:
//
//     splatlm::solver::lm_step(state, data, cfg, it, rng)        // reference, lm.cpp:56
//     splatlm_b200::lm_step(dev, state, data, cfg, it, rng)      // this adapter
//
// Semantics kept: the caller's std::mt19937_64 is consumed exactly like the
// reference (view batch, then the sample plan), `state` is updated in place,
// errors are thrown as the reference's exception types.
#pragma once

#include <map>
#include <random>
#include <sstream>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "slm_b200.h"
#include "splatlm/autodiff/jacobian.hpp"
#include "splatlm/baselines/first_order.hpp"
#include "splatlm/core/types.hpp"
#include "splatlm/io/dataset.hpp"
#include "splatlm/metrics/image_metrics.hpp"
#include "splatlm/render/rasterizer.hpp"
#include "splatlm/sampling/sample_plan.hpp"
#include "splatlm/solver/lm.hpp"
#include "splatlm/solver/pcg.hpp"

namespace splatlm_b200 {

using namespace splatlm;

inline void check(int rc) {
    if (rc == SLM_OK) return;
    const std::string msg = slm_last_error();
    if (rc == SLM_E_INVALID) throw std::invalid_argument(msg);
    if (rc == SLM_E_DOMAIN) throw std::domain_error(msg);
    throw std::runtime_error(msg);
}

inline slm_camera to_c(const Camera& cam) {
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

inline slm_gaussians to_c(GaussianSet& g) {
    return slm_gaussians{g.count, g.means.data(), g.log_scales.data(), g.rotations.data(),
                         g.opacity_logits.data(), g.colors.data()};
}

inline slm_lm_config to_c(const solver::LmConfig& c) {
    return slm_lm_config{c.damping, c.pcg_iters_initial, c.pcg_iters_late, c.pcg_switch_iteration,
                         c.batch_size_initial, c.batch_size_late, c.batch_switch_iteration,
                         c.samples_per_tile, c.sample_lane_width, c.lr_cap, c.warmup_lr,
                         c.warmup_iterations, static_cast<int32_t>(c.dist), static_cast<int32_t>(c.loss),
                         c.ssim_weight};
}

// Hand the caller's engine to the library and take it back afterwards, so
// the stream position advances exactly as the reference's would.
class RngBridge {
public:
    explicit RngBridge(std::mt19937_64& eng) : eng_(eng) {
        check(slm_rng_create(0, &h_));
        std::ostringstream os;
        os << eng_;
        check(slm_rng_set_state(h_, os.str().c_str()));
    }
    ~RngBridge() {
        int64_t n = 0;
        slm_rng_get_state(h_, nullptr, 0, &n);
        std::string buf(static_cast<size_t>(n) + 1, '\0');
        if (slm_rng_get_state(h_, buf.data(), n + 1, &n) == SLM_OK) {
            std::istringstream is(buf.c_str());
            is >> eng_;
        }
        slm_rng_destroy(h_);
    }
    slm_rng* get() { return h_; }

private:
    std::mt19937_64& eng_;
    slm_rng* h_ = nullptr;
};

// One CUDA context (device + stream); keeps TrainData resident in HBM.
class Device {
public:
    explicit Device(int device = 0) { check(slm_context_create(device, &ctx_)); }
    ~Device() {
        for (auto& kv : trains_) slm_train_destroy(kv.second);
        slm_context_destroy(ctx_);
    }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    slm_context* get() { return ctx_; }

    // The dataset images are float32 buffers widened to double by the run
    // driver (run.cpp:132), so narrowing back is exact.
    slm_train* train(const solver::TrainData& data) {
        auto it = trains_.find(&data);
        if (it == trains_.end()) {
            std::vector<slm_camera> cams;
            std::vector<float> imgs;
            for (size_t i = 0; i < data.cameras.size(); ++i) {
                cams.push_back(to_c(data.cameras[i]));
                for (double v : data.images[i].data) imgs.push_back(static_cast<float>(v));
            }
            slm_train* t = nullptr;
            check(slm_train_create(ctx_, cams.data(), static_cast<int>(cams.size()), imgs.data(), &t));
            it = trains_.emplace(&data, t).first;
        }
        std::vector<int32_t> assign(data.cameras.size(), 0);
        for (size_t c = 0; c < data.clusters.size(); ++c)
            for (int i : data.clusters[c]) assign[i] = static_cast<int32_t>(c);
        check(slm_train_set_clusters(it->second, assign.data(), static_cast<int>(data.clusters.size())));
        return it->second;
    }

private:
    slm_context* ctx_ = nullptr;
    std::map<const solver::TrainData*, slm_train*> trains_;
};

// solver::lm_step (lm.hpp:70-71)
inline solver::StepReport lm_step(Device& dev, GaussianSet& state, const solver::TrainData& data,
                                  const solver::LmConfig& cfg, int iteration, std::mt19937_64& rng) {
    if (data.clusters.empty()) throw std::invalid_argument("lm_step: no view clusters");
    slm_train* t = dev.train(data);
    slm_gaussians g = to_c(state);
    const slm_lm_config c = to_c(cfg);
    std::vector<int32_t> batch(data.clusters.size() + 1);
    slm_step_report rep{};
    rep.batch = batch.data();
    rep.batch_capacity = static_cast<int32_t>(batch.size());
    {
        RngBridge bridge(rng);
        check(slm_lm_step_host(dev.get(), &g, t, &c, iteration, bridge.get(), &rep));
    }
    solver::StepReport out;
    out.iteration = rep.iteration;
    out.loss_before = rep.loss_before;
    out.loss_after = rep.loss_after;
    out.eta = rep.eta;
    out.pcg_iterations = rep.pcg_iterations;
    out.breakdown = rep.breakdown != 0;
    out.batch.assign(batch.begin(), batch.begin() + rep.batch_size);
    return out;
}

// autodiff::SampledJacobian (jacobian.hpp:25-76)
class SampledJacobian {
public:
    SampledJacobian(Device& dev, const GaussianSet& gaussians, std::span<const Camera> cams,
                    const sampling::SamplePlan& plan) {
        GaussianSet copy = gaussians;  // the reference copies the set too (jacobian.cpp:100)
        slm_gaussians g = to_c(copy);
        std::vector<slm_camera> cc;
        for (const auto& c : cams) cc.push_back(to_c(c));
        std::vector<int32_t> vc;
        std::vector<int64_t> vo{0};
        std::vector<int32_t> px, py, tile;
        std::vector<double> w;
        for (const auto& v : plan.views) {
            vc.push_back(v.camera);
            px.insert(px.end(), v.px.begin(), v.px.end());
            py.insert(py.end(), v.py.begin(), v.py.end());
            tile.insert(tile.end(), v.tile.begin(), v.tile.end());
            w.insert(w.end(), v.weight.begin(), v.weight.end());
            vo.push_back(static_cast<int64_t>(px.size()));
        }
        const slm_plan p{static_cast<int32_t>(vc.size()), plan.samples_per_tile, static_cast<int32_t>(plan.dist),
                         vc.data(), vo.data(), px.data(), py.data(), tile.data(), w.data()};
        check(slm_jacobian_create(dev.get(), &g, cc.data(), static_cast<int>(cc.size()), &p, &h_));
        check(slm_jacobian_dims(h_, &rdim_, &pdim_));
    }
    ~SampledJacobian() { slm_jacobian_destroy(h_); }
    SampledJacobian(const SampledJacobian&) = delete;
    SampledJacobian& operator=(const SampledJacobian&) = delete;

    std::size_t residual_dim() const { return static_cast<std::size_t>(rdim_); }
    std::size_t param_dim() const { return static_cast<std::size_t>(pdim_); }

    std::vector<double> jvp(const ParamVector& v) const {
        if (v.size() != param_dim()) throw std::invalid_argument("jvp: probe vector length mismatch");
        std::vector<double> out(residual_dim());
        check(slm_jacobian_jvp(h_, v.data(), out.data()));
        return out;
    }
    ParamVector vjp(std::span<const double> u) const {
        if (u.size() != residual_dim()) throw std::invalid_argument("vjp: input length mismatch");
        ParamVector out(param_dim());
        check(slm_jacobian_vjp(h_, u.data(), out.data()));
        return out;
    }
    ParamVector jtj_diag() const {
        ParamVector out(param_dim());
        check(slm_jacobian_jtj_diag(h_, out.data()));
        return out;
    }
    ParamVector gn_apply(double lambda, const ParamVector& p) const {
        if (p.size() != param_dim()) throw std::invalid_argument("gn_apply: probe vector length mismatch");
        ParamVector out(param_dim());
        check(slm_jacobian_gn_apply(h_, lambda, p.data(), out.data()));
        return out;
    }
    std::vector<double> residual_weights() const {
        std::vector<double> w(residual_dim());
        check(slm_jacobian_weights(h_, w.data()));
        return w;
    }
    void set_residual_weights(std::vector<double> w) {
        if (w.size() != residual_dim()) throw std::invalid_argument("residual weight vector has wrong length");
        check(slm_jacobian_set_weights(h_, w.data()));
    }

private:
    slm_jacobian* h_ = nullptr;
    int64_t rdim_ = 0, pdim_ = 0;
};

// The one-shot wrappers (jacobian.hpp:80-87).
inline std::vector<double> jvp(Device& dev, const GaussianSet& g, std::span<const Camera> cams,
                               const sampling::SamplePlan& plan, const ParamVector& v) {
    return SampledJacobian(dev, g, cams, plan).jvp(v);
}
inline ParamVector vjp(Device& dev, const GaussianSet& g, std::span<const Camera> cams,
                       const sampling::SamplePlan& plan, std::span<const double> u) {
    return SampledJacobian(dev, g, cams, plan).vjp(u);
}
inline ParamVector jtj_diag(Device& dev, const GaussianSet& g, std::span<const Camera> cams,
                            const sampling::SamplePlan& plan) {
    return SampledJacobian(dev, g, cams, plan).jtj_diag();
}
inline ParamVector gn_apply(Device& dev, const GaussianSet& g, std::span<const Camera> cams,
                            const sampling::SamplePlan& plan, double lambda, const ParamVector& p) {
    return SampledJacobian(dev, g, cams, plan).gn_apply(lambda, p);
}

// ---- render:: (rasterizer.hpp:152-180) on the device, FP64 blend decisions
namespace render {

inline splatlm::render::RenderOutput make_output(int w, int h) {
    splatlm::render::RenderOutput out;
    out.image = Image(w, h);
    out.final_transmittance.assign(static_cast<size_t>(w) * h, 1.0);
    out.contrib_count.assign(static_cast<size_t>(w) * h, 0);
    return out;
}

inline std::vector<double> pack(std::span<const splatlm::render::SplatD> splats) {
    std::vector<double> d(10 * splats.size(), 0.0);
    for (size_t i = 0; i < splats.size(); ++i) {
        const auto& s = splats[i];
        const double v[10] = {s.mean2d.x, s.mean2d.y, s.conic_a, s.conic_b, s.conic_c, s.opacity,
                              s.color[0], s.color[1], s.color[2], 0.0};
        std::copy(v, v + 10, d.begin() + 10 * i);
    }
    return d;
}

// render::render_full (rasterizer.cpp:93-95)
inline splatlm::render::RenderOutput render_full(Device& dev, const GaussianSet& gaussians, const Camera& cam) {
    GaussianSet copy = gaussians;
    slm_gaussians g = to_c(copy);
    const slm_camera c = to_c(cam);
    auto out = make_output(cam.width, cam.height);
    check(slm_render_full(dev.get(), &g, &c, out.image.data.data(), out.final_transmittance.data(),
                          out.contrib_count.data()));
    return out;
}

// render::render_with_context (rasterizer.cpp:62-91): a caller-prepared context
inline splatlm::render::RenderOutput render_with_context(Device& dev, const splatlm::render::CameraContext& ctx) {
    const auto d = pack(ctx.splats);
    std::vector<int32_t> off{0}, idx;
    for (const auto& l : ctx.grid.lists) {
        idx.insert(idx.end(), l.begin(), l.end());
        off.push_back(static_cast<int32_t>(idx.size()));
    }
    const slm_camera c = to_c(ctx.cam);
    auto out = make_output(ctx.cam.width, ctx.cam.height);
    check(slm_render_splats(dev.get(), &c, static_cast<int>(ctx.splats.size()), d.data(), off.data(), idx.data(),
                            out.image.data.data(), out.final_transmittance.data(), out.contrib_count.data()));
    return out;
}

// render::render_pixel (rasterizer.cpp:52-60)
inline splatlm::render::PixelResult render_pixel(Device& dev, std::span<const splatlm::render::SplatD> sorted_splats,
                                                 double px, double py) {
    const auto d = pack(sorted_splats);
    double o[4];
    int32_t cnt = 0;
    check(slm_render_pixel(dev.get(), static_cast<int>(sorted_splats.size()), d.data(), px, py, o, &cnt));
    splatlm::render::PixelResult r;
    r.rgb[0] = o[0];
    r.rgb[1] = o[1];
    r.rgb[2] = o[2];
    r.transmittance = o[3];
    r.contrib = cnt;
    return r;
}

// render::residuals (rasterizer.cpp:97-104)
inline Image residuals(const Image& rendered, const Image& ground_truth) {
    if (rendered.width != ground_truth.width || rendered.height != ground_truth.height)
        throw std::invalid_argument("residuals: image shapes differ");
    Image out(rendered.width, rendered.height);
    check(slm_residuals(rendered.data.data(), ground_truth.data.data(), static_cast<int64_t>(out.data.size()),
                        out.data.data()));
    return out;
}

}  // namespace render

// solver::pcg_solve(ApplyFn, b, minv, max_iters) (pcg.hpp:22-23): the vector
// algebra runs on the device, `apply` on host vectors.
inline solver::PcgResult pcg_solve(Device& dev, const solver::ApplyFn& apply, const ParamVector& b,
                                   const ParamVector& minv, int max_iters) {
    if (minv.size() != b.size()) throw std::invalid_argument("pcg: preconditioner length mismatch");
    struct Ctx {
        const solver::ApplyFn* fn;
        std::size_t n;
    } c{&apply, b.size()};
    auto tramp = [](void* user, const double* p, double* out) {
        auto* cx = static_cast<Ctx*>(user);
        ParamVector pv(p, p + cx->n), ov;
        (*cx->fn)(pv, ov);
        std::copy(ov.begin(), ov.end(), out);
    };
    solver::PcgResult res;
    res.x.assign(b.size(), 0.0);
    slm_pcg_result r{};
    check(slm_pcg_solve(dev.get(), tramp, &c, b.data(), minv.data(), static_cast<int64_t>(b.size()), max_iters,
                        res.x.data(), &r));
    res.iterations = r.iterations;
    res.breakdown = r.breakdown != 0;
    res.rel_residual = r.rel_residual;
    return res;
}

// baselines::full_gradient (first_order.cpp:11-44) on the device.
inline ParamVector full_gradient(Device& dev, const GaussianSet& state, std::span<const Camera> cams,
                                 std::span<const Image> gts, solver::LossKind loss, double ssim_weight) {
    if (cams.size() != gts.size()) throw std::invalid_argument("full_gradient: camera/image count mismatch");
    std::vector<slm_camera> cc;
    std::vector<float> imgs;
    for (size_t i = 0; i < cams.size(); ++i) {
        cc.push_back(to_c(cams[i]));
        for (double v : gts[i].data) imgs.push_back(static_cast<float>(v));
    }
    GaussianSet g = state;
    slm_gaussians cg = to_c(g);
    slm_scene* s = nullptr;
    slm_train* t = nullptr;
    check(slm_scene_create(dev.get(), &cg, &s));
    ParamVector out(static_cast<size_t>(state.param_count()));
    int rc = slm_train_create(dev.get(), cc.data(), static_cast<int>(cc.size()), imgs.data(), &t);
    if (rc == SLM_OK) rc = slm_full_gradient(s, t, static_cast<int>(loss), ssim_weight, out.data());
    if (t) slm_train_destroy(t);
    slm_scene_destroy(s);
    check(rc);
    return out;
}

inline slm_first_order_config to_c(const baselines::FirstOrderConfig& c) {
    return slm_first_order_config{static_cast<int32_t>(c.kind), c.lrs.mean, c.lrs.color, c.lrs.opacity,
                                  c.lrs.scale, c.lrs.rotation, c.adam_beta1, c.adam_beta2, c.adam_eps,
                                  c.rms_decay, c.rms_eps, c.momentum, c.mean_lr_final_factor,
                                  c.decay_iterations, static_cast<int32_t>(c.loss), c.ssim_weight};
}

// baselines::first_order_step (first_order.cpp:115-122): the step runs on the
// device in f64 with the reference's operation order (bitwise equal results).
inline void first_order_step(Device& dev, baselines::FirstOrderState& st, GaussianSet& state,
                             const ParamVector& grad, const baselines::FirstOrderConfig& cfg) {
    if (grad.size() != static_cast<size_t>(state.param_count())) throw std::invalid_argument("gradient length mismatch");
    slm_gaussians cg = to_c(state);
    slm_scene* s = nullptr;
    slm_first_order* f = nullptr;
    check(slm_scene_create(dev.get(), &cg, &s));
    const slm_first_order_config c = to_c(cfg);
    int64_t step = st.step;
    int rc = slm_first_order_create(s, &f);
    if (rc == SLM_OK) rc = slm_first_order_set_moments(f, st.m1.data(), st.m2.data(), step);
    if (rc == SLM_OK) rc = slm_first_order_apply(f, grad.data(), &c);
    if (rc == SLM_OK) rc = slm_first_order_moments(f, st.m1.data(), st.m2.data(), &step);
    if (rc == SLM_OK) rc = slm_scene_download(s, &cg);
    if (f) slm_first_order_destroy(f);
    slm_scene_destroy(s);
    check(rc);
    st.step = static_cast<long>(step);
}

// metrics::evaluate (image_metrics.cpp:180-186) on the device.
inline metrics::MetricReport evaluate(Device& dev, const Image& rendered, const Image& ground_truth) {
    if (rendered.width != ground_truth.width || rendered.height != ground_truth.height)
        throw std::invalid_argument("metrics: image shapes differ");
    slm_metric_report r{};
    check(slm_evaluate(dev.get(), rendered.data.data(), ground_truth.data.data(), rendered.width,
                       rendered.height, &r));
    metrics::MetricReport out;
    out.mse = r.mse;
    out.psnr = r.psnr;
    out.ssim = r.ssim;
    return out;
}

// io::evaluate_split (run.cpp:77-92): every camera of the split rendered and
// scored on the device, mean mse / psnr / ssim.
inline metrics::MetricReport evaluate_split(Device& dev, const GaussianSet& state, const io::SceneDataset& split) {
    metrics::MetricReport out;
    if (split.cameras.empty()) return out;
    std::vector<slm_camera> cams;
    std::vector<float> imgs;
    for (size_t i = 0; i < split.cameras.size(); ++i) {
        cams.push_back(to_c(split.cameras[i]));
        imgs.insert(imgs.end(), split.images[i].data.begin(), split.images[i].data.end());
    }
    GaussianSet g = state;
    slm_gaussians cg = to_c(g);
    slm_scene* s = nullptr;
    slm_train* t = nullptr;
    check(slm_scene_create(dev.get(), &cg, &s));
    const int rc = slm_train_create(dev.get(), cams.data(), static_cast<int>(cams.size()), imgs.data(), &t);
    slm_metric_report r{};
    const int rc2 = rc == SLM_OK ? slm_evaluate_split(s, t, &r) : rc;
    if (t) slm_train_destroy(t);
    slm_scene_destroy(s);
    check(rc2);
    out.mse = r.mse;
    out.psnr = r.psnr;
    out.ssim = r.ssim;
    return out;
}

}  // namespace splatlm_b200
