// adapter_parity.cpp — the reference's own C++ caller code, run twice: once on
// the reference CPU path (splatlm::solver::lm_step) and once through the
// drop-in adapter include/splatlm_b200.hpp (splatlm_b200::lm_step on the B200).
// Built by oracle/Makefile (`make adapter`) against the reference sources;
// run by tests/test_gpu_parity.py::test_cpp_adapter_drop_in.  Prints one JSON
// line.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>

#include "splatlm/baselines/first_order.hpp"
#include "splatlm/io/dataset.hpp"
#include "splatlm/io/image_io.hpp"
#include "splatlm/io/scene_gen.hpp"
#include "splatlm/metrics/image_metrics.hpp"
#include "splatlm/render/rasterizer.hpp"
#include "splatlm_b200.hpp"

using namespace splatlm;

int main() {
    // run.cpp:120-160 shaped setup: toy scene, random_init from the run RNG,
    // TrainData with widened f32 images, k-means clusters.
    std::mt19937_64 scene_rng(20214);
    io::ToySceneConfig tc;
    tc.gaussians = 20;
    tc.train_cameras = 8;
    tc.test_cameras = 2;
    tc.image_size = 64;
    const io::ToyScene scene = io::generate_toy_scene(tc, scene_rng);
    solver::TrainData data;
    data.cameras = scene.train.cameras;
    for (const auto& img : scene.train.images) data.images.push_back(io::widen(img));
    data.rebuild_clusters(8, 1ull ^ 0x9e3779b97f4a7c15ull);
    solver::LmConfig cfg;
    cfg.pcg_iters_initial = 8;

    std::mt19937_64 rng_ref(1), rng_b2(1);
    GaussianSet ref = io::random_init(40, {-1, -1, -1}, {1, 1, 1}, rng_ref);
    GaussianSet b2 = io::random_init(40, {-1, -1, -1}, {1, 1, 1}, rng_b2);

    splatlm_b200::Device dev(0);
    bool batches_equal = true;
    double worst = 0.0;
    for (int it = 0; it < 6; ++it) {
        const auto a = solver::lm_step(ref, data, cfg, it, rng_ref);
        const auto b = splatlm_b200::lm_step(dev, b2, data, cfg, it, rng_b2);
        batches_equal = batches_equal && a.batch == b.batch && a.pcg_iterations == b.pcg_iterations;
        worst = std::max(worst, std::abs(a.loss_after - b.loss_after) / a.loss_after);
        worst = std::max(worst, std::abs(a.loss_before - b.loss_before) / a.loss_before);
    }
    const bool rng_equal = rng_ref() == rng_b2();

    // SampledJacobian::gn_apply through the adapter vs the reference class
    std::mt19937_64 prng(5);
    const std::vector<Camera> cams(data.cameras.begin(), data.cameras.begin() + 2);
    const auto plan = sampling::build_sample_plan(cams, 32, sampling::ResidualDist::kUniform, {}, prng);
    autodiff::SampledJacobian jr(ref, cams, plan);
    splatlm_b200::SampledJacobian jb(dev, ref, cams, plan);
    std::vector<double> p(jr.param_dim());
    std::uniform_real_distribution<double> u(-1, 1);
    for (double& v : p) v = u(prng);
    const auto ga = jr.gn_apply(0.1, p), gb = jb.gn_apply(0.1, p);
    double num = 0, den = 0;
    for (size_t i = 0; i < ga.size(); ++i) {
        num += (ga[i] - gb[i]) * (ga[i] - gb[i]);
        den += ga[i] * ga[i];
    }
    // io::evaluate_split (run.cpp:77-92) as the run driver computes it, vs the adapter
    metrics::MetricReport er;
    for (size_t i = 0; i < scene.test.cameras.size(); ++i) {
        const auto r = metrics::evaluate(render::render_full(ref, scene.test.cameras[i]).image,
                                         io::widen(scene.test.images[i]));
        er.mse += r.mse / scene.test.cameras.size();
        er.psnr += r.psnr / scene.test.cameras.size();
        er.ssim += r.ssim / scene.test.cameras.size();
    }
    const auto eb = splatlm_b200::evaluate_split(dev, ref, scene.test);
    // metrics::evaluate on two f64 images
    const Image ia = render::render_full(ref, scene.test.cameras[0]).image;
    const Image ib = io::widen(scene.test.images[0]);
    const auto ma = metrics::evaluate(ia, ib), mb = splatlm_b200::evaluate(dev, ia, ib);
    // baselines: full_gradient + two Adam steps through the adapter vs the reference
    const auto fa = baselines::full_gradient(ref, data.cameras, data.images, solver::LossKind::kMse, 0.2);
    const auto fb = splatlm_b200::full_gradient(dev, ref, data.cameras, data.images, solver::LossKind::kMse, 0.2);
    double gnum = 0, gden = 0;
    for (size_t i = 0; i < fa.size(); ++i) {
        gnum += (fa[i] - fb[i]) * (fa[i] - fb[i]);
        gden += fa[i] * fa[i];
    }
    baselines::FirstOrderConfig fcfg;
    auto sa = baselines::FirstOrderState::zeros(ref.param_count()), sb = sa;
    GaussianSet sta = ref, stb = ref;
    for (int k = 0; k < 2; ++k) {
        baselines::first_order_step(sa, sta, fa, fcfg);
        splatlm_b200::first_order_step(dev, sb, stb, fa, fcfg);
    }
    const bool fo_equal = sta.pack() == stb.pack() && sa.m1 == sb.m1 && sa.m2 == sb.m2 && sa.step == sb.step;
    // render:: surface: render_full, render_with_context on the reference's own prepared
    // context, render_pixel over a depth-ordered tile list, residuals
    const Camera& rc = scene.test.cameras[0];
    const auto rctx = render::prepare_camera(ref, rc);
    const auto ra = render::render_with_context(rctx);
    const auto rb = splatlm_b200::render::render_with_context(dev, rctx);
    const auto rf = splatlm_b200::render::render_full(dev, ref, rc);
    bool contrib_equal = ra.contrib_count == rb.contrib_count && ra.contrib_count == rf.contrib_count;
    double img_diff = 0.0, t_diff = 0.0;
    for (size_t i = 0; i < ra.image.data.size(); ++i)
        img_diff = std::max(img_diff, std::abs(ra.image.data[i] - rb.image.data[i]));
    for (size_t i = 0; i < ra.final_transmittance.size(); ++i)
        t_diff = std::max(t_diff, std::abs(ra.final_transmittance[i] - rb.final_transmittance[i]));
    const int tile = static_cast<int>(rctx.grid.lists.size() / 2);
    std::vector<render::SplatD> ordered;
    for (int idx : rctx.grid.lists[tile]) ordered.push_back(rctx.splats[idx]);
    const double ppx = (tile % rctx.grid.tiles_x) * 16 + 7.5, ppy = (tile / rctx.grid.tiles_x) * 16 + 7.5;
    const auto pa = render::render_pixel(ordered, ppx, ppy);
    const auto pb = splatlm_b200::render::render_pixel(dev, ordered, ppx, ppy);
    const double pix_diff = std::max({std::abs(pa.rgb[0] - pb.rgb[0]), std::abs(pa.rgb[1] - pb.rgb[1]),
                                      std::abs(pa.rgb[2] - pb.rgb[2]), std::abs(pa.transmittance - pb.transmittance)});
    contrib_equal = contrib_equal && pa.contrib == pb.contrib;
    const Image truth = io::widen(scene.test.images[0]);
    const bool resid_equal = render::residuals(ra.image, truth).data == splatlm_b200::render::residuals(ra.image, truth).data;
    bool resid_throws = false;
    try {
        splatlm_b200::render::residuals(ra.image, Image(3, 3));
    } catch (const std::invalid_argument&) {
        resid_throws = true;
    }
    // one-shot autodiff wrappers (jacobian.hpp:80-87)
    const auto oa = autodiff::gn_apply(ref, cams, plan, 0.1, p), ob = splatlm_b200::gn_apply(dev, ref, cams, plan, 0.1, p);
    double onum = 0, oden = 0;
    for (size_t i = 0; i < oa.size(); ++i) {
        onum += (oa[i] - ob[i]) * (oa[i] - ob[i]);
        oden += oa[i] * oa[i];
    }
    std::printf("{\"batches_equal\": %s, \"rng_equal\": %s, \"worst_loss_rel\": %.3e, \"gn_apply_rel\": %.3e, "
                "\"split_psnr_diff\": %.3e, \"split_ssim_diff\": %.3e, \"eval_ssim_diff\": %.3e, "
                "\"eval_mse_rel\": %.3e, \"full_gradient_rel\": %.3e, \"first_order_equal\": %s, "
                "\"render_contrib_equal\": %s, \"render_image_diff\": %.3e, \"render_t_diff\": %.3e, "
                "\"render_pixel_diff\": %.3e, \"residuals_equal\": %s, \"one_shot_gn_rel\": %.3e}\n",
                batches_equal ? "true" : "false", rng_equal ? "true" : "false", worst, std::sqrt(num / den),
                std::abs(er.psnr - eb.psnr), std::abs(er.ssim - eb.ssim), std::abs(ma.ssim - mb.ssim),
                std::abs(ma.mse - mb.mse) / ma.mse, std::sqrt(gnum / gden), fo_equal ? "true" : "false",
                contrib_equal ? "true" : "false", img_diff, t_diff, pix_diff,
                (resid_equal && resid_throws) ? "true" : "false", std::sqrt(onum / oden));
    return 0;
}
