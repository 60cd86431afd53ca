// oracle/ref_bench.cpp — TEST INFRASTRUCTURE ONLY: the CPU reference arm of bench.py.
//
// Times the UNMODIFIED reference (oracle/_ref objects, built from
// /root/reference/proj/src by oracle/Makefile) on the bench workload, with
// every input drawn by the reference itself -- nothing of libslm_b200 is
// linked or loaded:
//   * configs[2] inputs the way io::train_run seeds them (run.cpp:126-167):
//     io::random_init(G, [-1,1]^3, mt19937_64(1)), ring cameras W x H
//     (io::ring_camera, scene_gen.cpp:11-36, with height / cy set for the
//     non-square shape), sampling::kmeans_cameras (seed 1 ^ 0x9e37...),
//     sampling::sample_view_batch, sampling::build_sample_plan (uniform, N);
//   * gn_apply: autodiff::SampledJacobian over the WHOLE view batch
//     (jacobian.cpp:339-344), `warmup` untimed then `steps` timed calls;
//   * lm_step: solver::lm_step (lm.cpp:56-157) at the same shape, PCG 8,
//     on a ground truth of G/2 toy Gaussians (generate_toy_scene's
//     distributions, scales shrunk by (20/G)^(1/3) -- bench.py gt_scene);
//   * configs[0] time-to-PSNR: the toy scene run of
//     tests/golden/make_psnr_target.py (10 LM iterations, full pixels).
// Prints one JSON object.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <numeric>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "splatlm/autodiff/jacobian.hpp"
#include "splatlm/core/parallel.hpp"
#include "splatlm/core/types.hpp"
#include "splatlm/io/dataset.hpp"
#include "splatlm/io/image_io.hpp"
#include "splatlm/io/scene_gen.hpp"
#include "splatlm/metrics/image_metrics.hpp"
#include "splatlm/render/rasterizer.hpp"
#include "splatlm/sampling/sample_plan.hpp"
#include "splatlm/sampling/view_sampler.hpp"
#include "splatlm/solver/lm.hpp"

using namespace splatlm;
using clk = std::chrono::steady_clock;

namespace {

constexpr std::uint64_t kSalt = 0x9e3779b97f4a7c15ull;  // run.cpp:144

double secs(clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); }

struct Args {
    int gaussians = 1000000, views = 200, width = 1280, height = 720, batch = 8, spt = 32;
    int steps = 3, warmup = 1, lm_steps = 1, psnr = 1, threads = 0;
};

Camera ring_camera_wh(double angle, int w, int h) {
    Camera c = io::ring_camera(angle, 3.2, 1.1, w);
    c.height = h;
    c.cy = 0.5 * h;
    c.validate();
    return c;
}

std::string cpu_model() {
    std::ifstream f("/proc/cpuinfo");
    std::string line;
    while (std::getline(f, line))
        if (line.rfind("model name", 0) == 0) return line.substr(line.find(':') + 2);
    return "unknown";
}

int smt_active() {
    std::ifstream f("/sys/devices/system/cpu/smt/active");
    int v = -1;
    if (f >> v) return v;
    return -1;
}

std::string esc(const std::string& s) {
    std::string o;
    for (char c : s) o += (c == '"' || c == '\\') ? std::string("\\") + c : std::string(1, c);
    return o;
}

std::string arr(const std::vector<double>& v) {
    std::string s = "[";
    char b[64];
    for (size_t i = 0; i < v.size(); ++i) {
        std::snprintf(b, sizeof b, "%s%.6g", i ? ", " : "", v[i]);
        s += b;
    }
    return s + "]";
}

}  // namespace

int main(int argc, char** argv) {
    Args a;
    for (int i = 1; i + 1 < argc; i += 2) {
        const std::string k = argv[i];
        const int v = std::atoi(argv[i + 1]);
        if (k == "--gaussians") a.gaussians = v;
        else if (k == "--views") a.views = v;
        else if (k == "--width") a.width = v;
        else if (k == "--height") a.height = v;
        else if (k == "--batch") a.batch = v;
        else if (k == "--spt") a.spt = v;
        else if (k == "--steps") a.steps = v;
        else if (k == "--warmup") a.warmup = v;
        else if (k == "--lm-steps") a.lm_steps = v;
        else if (k == "--psnr") a.psnr = v;
        else if (k == "--threads") a.threads = v;
    }
    const int hw = static_cast<int>(std::thread::hardware_concurrency());
    set_thread_count(a.threads > 0 ? a.threads : hw);
    const auto t_start = clk::now();

    // ---- configs[2] inputs, drawn by the reference
    std::mt19937_64 rng(1);
    auto t0 = clk::now();
    const GaussianSet state = io::random_init(a.gaussians, {-1, -1, -1}, {1, 1, 1}, rng);
    std::vector<Camera> cams;
    for (int i = 0; i < a.views; ++i) cams.push_back(ring_camera_wh(2.0 * M_PI * i / a.views, a.width, a.height));
    const auto clusters = sampling::kmeans_cameras(sampling::camera_features(cams), a.batch, 1 ^ kSalt);
    const std::vector<int> batch = sampling::sample_view_batch(clusters, rng);
    std::vector<Camera> bcams;
    for (int i : batch) bcams.push_back(cams[i]);
    const sampling::SamplePlan plan =
        sampling::build_sample_plan(bcams, a.spt, sampling::ResidualDist::kUniform, {}, rng, 32);
    const double inputs_s = secs(t0, clk::now());

    // ---- gn_apply over the whole batch
    t0 = clk::now();
    autodiff::SampledJacobian jac(state, bcams, plan);
    const double ctor_s = secs(t0, clk::now());
    std::mt19937_64 prng(0);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    ParamVector p(jac.param_dim()), out(jac.param_dim());
    for (double& x : p) x = u(prng);
    for (int i = 0; i < a.warmup; ++i) jac.gn_apply(0.1, p, out);
    std::vector<double> times;
    for (int i = 0; i < a.steps; ++i) {
        t0 = clk::now();
        jac.gn_apply(0.1, p, out);
        times.push_back(secs(t0, clk::now()));
    }
    std::vector<double> sorted = times;
    std::sort(sorted.begin(), sorted.end());
    const double median = sorted.empty() ? 0.0 : sorted[sorted.size() / 2];
    const double mean = times.empty() ? 0.0 : std::accumulate(times.begin(), times.end(), 0.0) / times.size();

    // ---- lm_step at the same shape
    std::vector<double> lm_times;
    double lm_gt_s = 0.0;
    if (a.lm_steps > 0) {
        t0 = clk::now();
        const int gcount = std::max(1, a.gaussians / 2);
        io::ToySceneConfig tc;
        tc.gaussians = gcount;
        tc.train_cameras = 0;
        tc.test_cameras = 0;
        std::mt19937_64 grng(20214);
        GaussianSet gt = io::generate_toy_scene(tc, grng).ground_truth;
        const double shift = std::log(20.0 / gcount) / 3.0;  // scales x (20/G)^(1/3)
        for (double& v : gt.log_scales) v = v + shift;
        solver::TrainData data;
        data.cameras = cams;
        data.images.resize(cams.size());
        data.clusters = clusters;
        std::mt19937_64 lrng(1);
        GaussianSet lstate = io::random_init(a.gaussians, {-1, -1, -1}, {1, 1, 1}, lrng);
        solver::LmConfig cfg;
        cfg.pcg_iters_initial = cfg.pcg_iters_late = 8;
        cfg.batch_size_initial = cfg.batch_size_late = a.batch;
        cfg.samples_per_tile = a.spt;
        for (int it = 0; it < a.lm_steps; ++it) {
            // truth images of the views this step draws (the others are never read)
            std::mt19937_64 peek = lrng;
            for (int idx : sampling::sample_view_batch(data.clusters, peek))
                if (data.images[idx].width == 0)
                    data.images[idx] = io::widen(io::narrow(render::render_full(gt, cams[idx]).image));
            lm_gt_s += secs(t0, clk::now());
            t0 = clk::now();
            solver::lm_step(lstate, data, cfg, it, lrng);
            lm_times.push_back(secs(t0, clk::now()));
            t0 = clk::now();
        }
    }

    // ---- configs[0] time-to-PSNR (tests/golden/make_psnr_target.py)
    std::vector<double> psnr_curve, psnr_wall;
    if (a.psnr) {
        io::ToySceneConfig tc;
        tc.gaussians = 5000;
        tc.train_cameras = 8;
        tc.test_cameras = 4;
        tc.image_size = 256;
        std::mt19937_64 srng(20214);
        const io::ToyScene scene = io::generate_toy_scene(tc, srng);
        std::mt19937_64 prng1(1);
        GaussianSet s0 = io::random_init(10000, {-1, -1, -1}, {1, 1, 1}, prng1);
        solver::TrainData data;
        data.cameras = scene.train.cameras;
        for (const auto& im : scene.train.images) data.images.push_back(io::widen(im));
        data.rebuild_clusters(8, 1 ^ kSalt);
        solver::LmConfig cfg;
        cfg.pcg_iters_initial = cfg.pcg_iters_late = 8;
        cfg.batch_size_initial = cfg.batch_size_late = 8;
        cfg.samples_per_tile = 256;
        for (int it = 0; it < 10; ++it) {
            t0 = clk::now();
            solver::lm_step(s0, data, cfg, it, prng1);
            psnr_wall.push_back(secs(t0, clk::now()));
            double ps = 0.0;
            for (size_t i = 0; i < scene.test.cameras.size(); ++i)
                ps += metrics::psnr(render::render_full(s0, scene.test.cameras[i]).image,
                                    io::widen(scene.test.images[i]));
            psnr_curve.push_back(ps / scene.test.cameras.size());
        }
    }

    std::printf(
        "{\"kind\": \"reference\", \"threads\": %d, \"nproc\": %d, \"cpu_model\": \"%s\", \"smt_active\": %d, "
        "\"batch\": [",
        thread_count(), hw, esc(cpu_model()).c_str(), smt_active());
    for (size_t i = 0; i < batch.size(); ++i) std::printf("%s%d", i ? ", " : "", batch[i]);
    std::printf("], \"samples\": %zu, \"inputs_s\": %.3f, \"ctor_s\": %.3f, \"gn_apply_s\": %s, "
                "\"gn_apply_median_s\": %.6g, \"gn_apply_mean_s\": %.6g, \"lm_step_s\": %s, \"lm_gt_render_s\": %.3f, "
                "\"psnr_curve_db\": %s, \"psnr_wall_s\": %s, \"total_s\": %.3f}\n",
                static_cast<size_t>(plan.total_samples()), inputs_s, ctor_s, arr(times).c_str(), median, mean,
                arr(lm_times).c_str(), lm_gt_s, arr(psnr_curve).c_str(), arr(psnr_wall).c_str(),
                secs(t_start, clk::now()));
    return 0;
}
