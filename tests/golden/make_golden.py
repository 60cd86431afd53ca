"""Generate the golden fixtures in tests/golden/ from the REAL reference.

Run in the dev container (needs /root/reference, built by `make -C oracle`):

    python tests/golden/make_golden.py

Every array is produced by the unmodified reference library
(oracle/_ref/libsplatlm_ref.so, driven through oracle/ref_capi.cpp); the
inputs are seeded exactly like the reference's own tests
(tests/test_render.cpp, test_autodiff.cpp, test_sampling.cpp,
test_solver.cpp).  The fixtures travel with the repo; nothing on the GPU box
needs /root/reference.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle.cpu_bind import ref  # noqa: E402
from paper_2504_12905_b200.types import LmConfig, ring_camera  # noqa: E402
from support import MT64, random_scene, test_camera  # noqa: E402


def cam_arr(cams):
    return np.array([np.concatenate([c.world_to_cam, c.translation,
                                     [c.fx, c.fy, c.cx, c.cy, c.near_clip, c.width, c.height]])
                     for c in cams])


def set_arrs(prefix, g):
    g = g.copy()  # lm_step mutates in place
    return {f"{prefix}_means": g.means, f"{prefix}_log_scales": g.log_scales,
            f"{prefix}_rotations": g.rotations, f"{prefix}_opacity_logits": g.opacity_logits,
            f"{prefix}_colors": g.colors}


def plan_arrs(prefix, p):
    return {f"{prefix}_view_camera": p.view_camera, f"{prefix}_view_offset": p.view_offset,
            f"{prefix}_px": p.px, f"{prefix}_py": p.py, f"{prefix}_tile": p.tile,
            f"{prefix}_weight": p.weight}


def render_cases(R):
    """Tiled render + tile lists on the test_render.cpp:122 seeds, plus ring and
    non-square cameras over a random_init state."""
    out = {}
    rng = MT64(31)
    for t in range(20):
        size = 16 + rng() % 49
        cam = test_camera(size, 3.0)
        scene = random_scene(5 + rng() % 46, rng)
        off, idx = R.bin_and_sort(scene, cam)
        img, tr, cn = R.render_full(scene, cam)
        out.update(set_arrs(f"r{t}", scene))
        out[f"r{t}_cam"] = cam_arr([cam])
        out[f"r{t}_offsets"], out[f"r{t}_indices"] = off, idx
        out[f"r{t}_image"], out[f"r{t}_trans"], out[f"r{t}_contrib"] = img, tr, cn
    out["n_random"] = np.array(20)
    # random_init state seen from ring cameras, square and non-square
    st = R.random_init(400, [-1, -1, -1], [1, 1, 1], R.rng(1))
    cams = [ring_camera(0.0, 3.2, 1.1, 96), ring_camera(1.3, 3.2, 1.1, 80, 48),
            ring_camera(2.9, 3.2, 1.6, 72, 100)]
    out.update(set_arrs("ring", st))
    out["ring_cams"] = cam_arr(cams)
    for i, cam in enumerate(cams):
        off, idx = R.bin_and_sort(st, cam)
        img, tr, cn = R.render_full(st, cam)
        p = R.prepare(st, cam)
        out[f"ring{i}_offsets"], out[f"ring{i}_indices"] = off, idx
        out[f"ring{i}_image"], out[f"ring{i}_trans"], out[f"ring{i}_contrib"] = img, tr, cn
        for k, v in p.items():
            out[f"ring{i}_prep_{k}"] = v
    return out


def sampling_cases(R):
    out = {}
    cams40 = [test_camera(40, 3.0)]
    rng = R.rng(65)
    out.update(plan_arrs("u32", R.build_sample_plan(cams40, 32, 0, rng)))
    out.update(plan_arrs("u256", R.build_sample_plan([test_camera(32, 3.0)], 256, 0, R.rng(64))))
    out.update(plan_arrs("u13", R.build_sample_plan(cams40, 13, 0, R.rng(7), lane_width=1)))
    batch = [ring_camera(0.3, 3.2, 1.1, 80, 48), ring_camera(2.0, 3.2, 1.1, 64),
             ring_camera(4.0, 3.2, 1.1, 50, 70)]
    out["batch_cams"] = cam_arr(batch)
    out.update(plan_arrs("b64", R.build_sample_plan(batch, 64, 0, R.rng(123))))
    out["ex_cams"] = cam_arr(batch[:2])
    out.update(plan_arrs("ex", R.exhaustive_plan(batch[:2])))
    # k-means clusters and one batch draw over a 24-camera ring
    ring = [ring_camera(2 * np.pi * i / 24, 3.2, 1.1 + 0.1 * (i % 3), 64) for i in range(24)]
    out["km_cams"] = cam_arr(ring)
    out["km_features"] = R.camera_features(ring)
    assign = np.zeros(24, np.int32)
    for c, members in enumerate(R.kmeans_cameras(ring, 8, 1 ^ 0x9E3779B97F4A7C15)):
        assign[members] = c
    out["km_assign"] = assign
    # raw engine + distributions
    r = R.rng(2024)
    out["mt_first"] = np.array([r() for _ in range(1000)], np.uint64)
    return out


def jacobian_cases(R):
    out = {}
    cases = {
        # test_autodiff.cpp Fixture(5, 32, 48) exhaustive
        "jx": dict(scene=random_scene(5, MT64(48)), cams=[test_camera(32, 3.0)], plan="exhaustive"),
        # Fixture(12, 48, 140, 32) with lane width 1 (test_autodiff.cpp:326)
        "js": dict(seed=140, n=12, size=48, spt=32),
        # random_init state, 2 ring views, N = 32 lane 32 (lm_step shape)
        "jr": dict(ring=True),
    }
    for name, c in cases.items():
        if "scene" in c:
            scene, cams = c["scene"], c["cams"]
            plan = R.exhaustive_plan(cams)
        elif "seed" in c:
            rng = MT64(c["seed"])
            scene = random_scene(c["n"], rng)
            cams = [test_camera(c["size"], 3.0)]
            plan = R.build_sample_plan(cams, c["spt"], 0, R.rng(c["seed"] + 1), lane_width=1)
        else:
            scene = R.random_init(300, [-1, -1, -1], [1, 1, 1], R.rng(9))
            cams = [ring_camera(0.4, 3.2, 1.1, 64), ring_camera(2.2, 3.2, 1.1, 80, 48)]
            plan = R.build_sample_plan(cams, 32, 0, R.rng(10))
        jac = R.jacobian(scene, cams, plan)
        g = np.random.default_rng({"jx": 1, "js": 2, "jr": 3}[name])
        v = g.uniform(-1, 1, jac.param_dim())
        u = g.uniform(-1, 1, jac.residual_dim())
        p = g.uniform(-1, 1, jac.param_dim())
        out.update(set_arrs(name, scene))
        out[f"{name}_cams"] = cam_arr(cams)
        out.update(plan_arrs(name, plan))
        out[f"{name}_v"], out[f"{name}_u"], out[f"{name}_p"] = v, u, p
        out[f"{name}_jvp"] = jac.jvp(v)
        out[f"{name}_vjp"] = jac.vjp(u)
        out[f"{name}_diag"] = jac.jtj_diag()
        out[f"{name}_gn"] = jac.gn_apply(0.1, p)
        out[f"{name}_weights"] = jac.residual_weights()
        minv = 1.0 / (out[f"{name}_diag"] + 0.1)
        res = jac.pcg(0.1, out[f"{name}_vjp"], minv, 8)
        out[f"{name}_pcg_x"] = res.x
        out[f"{name}_pcg_meta"] = np.array([res.iterations, res.breakdown, res.rel_residual])
    return out


def lm_cases(R):
    """Free-running LM trajectory on the toy scene (run.cpp:120-196 shape)."""
    out = {}
    gt, tc, ti, sc, si = R.toy_scene(gaussians=20, train_cameras=8, test_cameras=4, image_size=64)
    out.update(set_arrs("toy_gt", gt))
    out["toy_train_cams"], out["toy_train_imgs"] = cam_arr(tc), ti
    out["toy_test_cams"], out["toy_test_imgs"] = cam_arr(sc), si
    rng = R.rng(1)
    st = R.random_init(40, [-1, -1, -1], [1, 1, 1], rng)
    out.update(set_arrs("lm_init", st))
    td = R.train_data(tc, ti)
    td.rebuild_clusters(8, 1 ^ 0x9E3779B97F4A7C15)
    cfg = LmConfig(pcg_iters_initial=8, pcg_iters_late=8)
    reps = []
    for it in range(12):
        r = R.lm_step(st, td, cfg, it, rng)
        reps.append([r.iteration, r.loss_before, r.loss_after, r.eta, r.pcg_iterations,
                     r.breakdown] + [int(b) for b in r.batch])
    out["lm_reports"] = np.array(reps, np.float64)
    out.update(set_arrs("lm_final", st))
    out["lm_rng_next"] = np.array([rng()], np.uint64)
    # test PSNR of the final state (evaluate_split, run.cpp:77-92)
    ps = []
    for cam, img in zip(sc, si):
        ren, _, _ = R.render_full(st, cam)
        ps.append(R.psnr(ren, img.astype(np.float64)))
    out["lm_test_psnr"] = np.array(ps)
    return out


def metrics_cases(R):
    """metrics::mse / psnr / ssim (image_metrics.cpp:108-139) on seeded image pairs, and the
    per-camera evaluate of the toy LM run's final state on its test split (run.cpp:77-92)."""
    out = {}
    rng = np.random.default_rng(2504)
    shapes = [(6, 6), (17, 33), (40, 24), (64, 64), (7, 90)]
    for i, (h, w) in enumerate(shapes):
        a = rng.random((h, w, 3))
        b = np.clip(a + rng.normal(0.0, 0.05 * (i + 1), a.shape), 0.0, 1.0)
        out[f"m{i}_a"], out[f"m{i}_b"] = a, b
        out[f"m{i}_ref"] = np.array([R.mse(a, b), R.psnr(a, b), R.ssim(a, b)])
        out[f"m{i}_self"] = np.array([R.mse(a, a), R.psnr(a, a), R.ssim(a, a)])
        out[f"m{i}_sres"], out[f"m{i}_sdc"] = R.ssim_diag_residuals(a, b)
    d = np.load(os.path.join(HERE, "lm.npz"))
    from support import g_cams, g_set
    st = g_set(d, "lm_final")
    rows = []
    for cam, img in zip(g_cams(d["toy_test_cams"]), d["toy_test_imgs"]):
        ren, _, _ = R.render_full(st, cam)
        gt = np.asarray(img, np.float64)
        rows.append([R.mse(ren, gt), R.psnr(ren, gt), R.ssim(ren, gt)])
    out["split_metrics"] = np.array(rows)
    return out


def lm_ssim_cases(R):
    """The same toy LM run with the mse+ssim loss (lm.cpp:86-119, ssim_weight 0.2)."""
    out = {}
    d = np.load(os.path.join(HERE, "lm.npz"))
    from support import g_cams
    tc, ti = g_cams(d["toy_train_cams"]), list(d["toy_train_imgs"])
    rng = R.rng(1)
    st = R.random_init(40, [-1, -1, -1], [1, 1, 1], rng)
    td = R.train_data(tc, ti)
    td.rebuild_clusters(8, 1 ^ 0x9E3779B97F4A7C15)
    cfg = LmConfig(pcg_iters_initial=8, pcg_iters_late=8, loss=1, ssim_weight=0.2)
    reps = []
    for it in range(8):
        r = R.lm_step(st, td, cfg, it, rng)
        reps.append([r.iteration, r.loss_before, r.loss_after, r.eta, r.pcg_iterations,
                     r.breakdown] + [int(b) for b in r.batch])
    out["lms_reports"] = np.array(reps, np.float64)
    out.update(set_arrs("lms_final", st))
    out["lms_rng_next"] = np.array([rng()], np.uint64)
    # batch_loss with the mse+ssim loss on the final state, all train views
    out["lms_batch_loss"] = np.array([R.batch_loss(st, tc, ti, loss=1, ssim_weight=0.2)])
    return out


def first_order_cases(R):
    """baselines::full_gradient and the Adam / RMSprop / SGD-momentum steps
    (first_order.cpp) on the toy LM scene, as train_run drives them (run.cpp:176-182)."""
    from paper_2504_12905_b200.types import FirstOrderConfig
    out = {}
    d = np.load(os.path.join(HERE, "lm.npz"))
    from support import g_cams, g_set
    tc, ti = g_cams(d["toy_train_cams"]), list(d["toy_train_imgs"])
    st0 = g_set(d, "lm_init")
    out["fo_grad_mse"] = R.full_gradient(st0, tc, ti, 0)
    out["fo_grad_ssim"] = R.full_gradient(st0, tc, ti, 1, 0.2)
    for kind in (0, 1, 2):
        extra = FirstOrderConfig.sgd_paper_lrs() if kind == 2 else {}
        cfg = FirstOrderConfig(kind=kind, decay_iterations=6, **extra)
        st = st0.copy()
        m1, m2, step = np.zeros(st.count * 14), np.zeros(st.count * 14), 0
        losses = []
        for it in range(6):
            grad = R.full_gradient(st, tc, ti, 0)
            step = R.first_order_step(st, m1, m2, step, grad, cfg)
            losses.append(R.batch_loss(st, tc, ti))
        out[f"fo{kind}_losses"] = np.array(losses)
        out.update(set_arrs(f"fo{kind}_final", st))
        out[f"fo{kind}_m1"], out[f"fo{kind}_m2"] = m1, m2
    return out


RUN_CASES = {  # io::train_run on the toy scene, deterministic mode
    "lm": dict(optimizer="lm", iterations=6, eval_every=3),
    "adam": dict(optimizer="adam", iterations=4, eval_every=2),
}


def run_cases(R):
    """io::train_run outputs (metrics.csv, summary.json, checkpoint.bin + .meta.txt) for the
    toy scene, stored as bytes (run.cpp:120-212, checkpoint.cpp:45-66)."""
    import tempfile

    from paper_2504_12905_b200.types import FirstOrderConfig
    out = {}
    for name, c in RUN_CASES.items():
        with tempfile.TemporaryDirectory() as d:
            R.train_run_toy(d, c["optimizer"], c["iterations"], LmConfig(pcg_iters_initial=8), FirstOrderConfig(),
                            eval_every=c["eval_every"], deterministic=True)
            for f in ("metrics.csv", "summary.json", "checkpoint.bin", "checkpoint.bin.meta.txt"):
                with open(os.path.join(d, f), "rb") as fh:
                    out[f"{name}_{f}"] = np.frombuffer(fh.read(), np.uint8)
    return out


def main():
    R = ref()
    groups = {"render": render_cases, "sampling": sampling_cases, "jacobian": jacobian_cases,
              "lm": lm_cases, "metrics": metrics_cases, "lm_ssim": lm_ssim_cases,
              "first_order": first_order_cases, "run": run_cases}
    only = sys.argv[1:]  # optional group names: regenerate just those
    for name, fn in groups.items():
        if only and name not in only:
            continue
        arrs = fn(R)
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **arrs)
        print(f"{path}: {os.path.getsize(path) / 1e6:.2f} MB, {len(arrs)} arrays")


if __name__ == "__main__":
    main()
