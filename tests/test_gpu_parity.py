"""GPU parity: the sm_100a path through the C ABI vs the reference.

Anchors: the golden fixtures made by the unmodified reference
(tests/golden/*.npz) and the C restatement (oracle/liboracle.so, pinned to the
reference bit for bit by tests/test_oracle.py) on fresh seeded inputs.

Bars (BASELINE.json north_star):
* bit-exact: tile/Gaussian lists, per-tile sort order, sampled pixel sets,
  view batches;
* norm-relative 1e-4: Jv, J^T u, diag(J^T W J), J^T W J p, the CG solution,
  per-iteration loss.  The sampled pixels' blend decisions (skip, clamp,
  termination) and final colours come from an FP64 replay of the reference's
  blend (k_masks), so the products differ from the reference only by FP32
  value rounding (~5e-6 at the full 1M-Gaussian size); the full-image render
  used for the losses is FP32, where a pixel within rounding of a gate may
  take the other branch.
"""
import math
import os

import numpy as np
import pytest

from paper_2504_12905_b200.types import GaussianSet, LmConfig, SamplePlan
from support import (MT64, g_cams, g_plan, g_set, golden, norm_rel, random_scene, rel_error)
from support import test_camera as tcam

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def gpu():
    from paper_2504_12905_b200 import splatlm
    return splatlm.lib()


# ----------------------------------------------------------------- K1/K3/K4
@pytest.mark.parametrize("t", range(20))
def test_tile_lists_bit_exact_random_scenes(gpu, t):
    d = golden("render")
    g = g_set(d, f"r{t}")
    cam = g_cams(d[f"r{t}_cam"])[0]
    off, idx = gpu.bin_and_sort(g, cam)
    assert np.array_equal(off, d[f"r{t}_offsets"])
    assert np.array_equal(idx, d[f"r{t}_indices"])


@pytest.mark.parametrize("i", range(3))
def test_tile_lists_bit_exact_ring_views(gpu, i):
    d = golden("render")
    g = g_set(d, "ring")
    cam = g_cams(d["ring_cams"])[i]
    off, idx = gpu.bin_and_sort(g, cam)
    assert np.array_equal(off, d[f"ring{i}_offsets"])
    assert np.array_equal(idx, d[f"ring{i}_indices"])
    p = gpu.prepare(g, cam)
    assert np.array_equal(p["valid"], d[f"ring{i}_prep_valid"])
    assert np.array_equal(p["depth"][p["valid"] == 1], d[f"ring{i}_prep_depth"][p["valid"] == 1])
    v = p["valid"] == 1
    assert np.allclose(p["mean2d"].reshape(-1, 2)[v], d[f"ring{i}_prep_mean2d"].reshape(-1, 2)[v], rtol=1e-6)


def test_bin_and_sort_known_answers(gpu):
    """test_render.cpp:89-120: empty scene, single-tile locality, depth order."""
    from paper_2504_12905_b200.types import GaussianSet
    cam = tcam(64, 3.0)
    off, idx = gpu.bin_and_sort(GaussianSet.zeros(0), cam)
    assert idx.size == 0 and np.all(off == 0)
    one = GaussianSet.zeros(1)
    one.means[:] = [-0.30, -0.30, 0.0]
    one.log_scales[:] = np.log(0.01)
    one.opacity_logits[:] = 0.5
    off, idx = gpu.bin_and_sort(one, cam)
    assert np.count_nonzero(np.diff(off)) == 1
    two = GaussianSet.zeros(2)
    two.means[:] = [0, 0, 1.0, 0, 0, 0.0]
    two.log_scales[:] = np.log(0.2)
    two.opacity_logits[:] = 0.5
    off, idx = gpu.bin_and_sort(two, cam)
    shared = [idx[off[t]:off[t + 1]] for t in range(off.size - 1) if off[t + 1] - off[t] == 2]
    assert shared and all(list(s) == [1, 0] for s in shared)


def test_permuted_storage_order(gpu):
    """test_render.cpp:137: the per-tile sort removes storage-order dependence."""
    rng = MT64(33)
    g = random_scene(12, rng)
    perm = np.random.default_rng(1).permutation(12)
    h = g.copy()
    h.means = g.means.reshape(-1, 3)[perm].reshape(-1).copy()
    h.log_scales = g.log_scales.reshape(-1, 3)[perm].reshape(-1).copy()
    h.colors = g.colors.reshape(-1, 3)[perm].reshape(-1).copy()
    h.rotations = g.rotations.reshape(-1, 4)[perm].reshape(-1).copy()
    h.opacity_logits = g.opacity_logits[perm].copy()
    a = gpu.render_full(g, tcam(32, 3.0))[0]
    b = gpu.render_full(h, tcam(32, 3.0))[0]
    assert np.max(np.abs(a - b)) < 1e-6


# ----------------------------------------------------------------- K6
@pytest.mark.parametrize("t", range(20))
def test_render_random_scenes(gpu, t):
    """render_full (the drop-in API replays blend_pixel in FP64): contributor counts
    bit-exact, image / transmittance to FP32-stored colours (1e-6)."""
    d = golden("render")
    g = g_set(d, f"r{t}")
    cam = g_cams(d[f"r{t}_cam"])[0]
    img, tr, cn = gpu.render_full(g, cam)
    assert np.array_equal(cn, d[f"r{t}_contrib"])
    assert norm_rel(img, d[f"r{t}_image"]) < 1e-6
    assert np.max(np.abs(img - d[f"r{t}_image"])) < 1e-6


@pytest.mark.parametrize("i", range(3))
def test_render_ring_views(gpu, i):
    d = golden("render")
    g = g_set(d, "ring")
    cam = g_cams(d["ring_cams"])[i]
    img, tr, cn = gpu.render_full(g, cam)
    assert np.array_equal(cn, d[f"ring{i}_contrib"])
    assert norm_rel(img, d[f"ring{i}_image"]) < 1e-6
    assert np.max(np.abs(tr - d[f"ring{i}_trans"])) < 1e-12


def test_fp32_render_matches_exact_render(gpu):
    """The FP32 k_render (the LM step's losses, slm_scene_render) against the exact
    render on the reference's ring scene: same image to FP32 tolerance."""
    from paper_2504_12905_b200 import splatlm
    d = golden("render")
    g = g_set(d, "ring")
    cam = g_cams(d["ring_cams"])[0]
    img32 = splatlm.Scene(gpu, g).render(cam)[0]
    assert norm_rel(img32.astype(np.float64), d["ring0_image"]) < TOL


def test_render_known_answers(gpu):
    """test_render.cpp:170-182: empty scene is background, T = 1."""
    from paper_2504_12905_b200.types import GaussianSet
    img, tr, cn = gpu.render_full(GaussianSet.zeros(0), tcam(32, 3.0))
    assert np.all(img == 0) and np.all(tr == 1) and np.all(cn == 0)


# ----------------------------------------------------------------- Jacobian products
@pytest.mark.parametrize("name", ["jx", "js", "jr"])
def test_jacobian_products_vs_reference(gpu, name):
    d = golden("jacobian")
    g = g_set(d, name)
    cams = g_cams(d[f"{name}_cams"])
    jac = gpu.jacobian(g, cams, g_plan(d, name))
    assert jac.residual_dim() == d[f"{name}_jvp"].size and jac.param_dim() == d[f"{name}_vjp"].size
    assert np.array_equal(jac.residual_weights(), d[f"{name}_weights"])
    errs = {
        "jvp": norm_rel(jac.jvp(d[f"{name}_v"]), d[f"{name}_jvp"]),
        "vjp": norm_rel(jac.vjp(d[f"{name}_u"]), d[f"{name}_vjp"]),
        "diag": norm_rel(jac.jtj_diag(), d[f"{name}_diag"]),
        "gn": norm_rel(jac.gn_apply(0.1, d[f"{name}_p"]), d[f"{name}_gn"]),
    }
    print(name, errs)
    assert all(e < TOL for e in errs.values()), errs
    minv = 1.0 / (d[f"{name}_diag"] + 0.1)
    res = jac.pcg(0.1, d[f"{name}_vjp"], minv, 8)
    meta = d[f"{name}_pcg_meta"]
    assert res.iterations == int(meta[0]) and res.breakdown == bool(meta[1])
    assert norm_rel(res.x, d[f"{name}_pcg_x"]) < TOL


def test_adjoint_identity(gpu):
    """test_autodiff.cpp:131: <Jv, u> == <v, J^T u> (FP32 raster: 1e-4)."""
    g = random_scene(5, MT64(48))
    cams = [tcam(32, 3.0)]
    host = gpu
    plan = host.exhaustive_plan(cams)
    jac = gpu.jacobian(g, cams, plan)
    r = np.random.default_rng(49)
    for _ in range(10):
        v = r.uniform(-1, 1, jac.param_dim())
        u = r.uniform(-1, 1, jac.residual_dim())
        lhs = float(np.dot(jac.jvp(v), u))
        rhs = float(np.dot(v, jac.vjp(u)))
        assert rel_error(lhs, rhs) < TOL


def test_gn_apply_symmetric_pd_and_linear(gpu):
    """test_autodiff.cpp:106,264: linearity, symmetry, positive definiteness."""
    rng = MT64(56)
    g = random_scene(5, rng)
    cams = [tcam(32, 3.0)]
    plan = gpu.build_sample_plan(cams, 8, 0, gpu.rng(57), lane_width=1)
    jac = gpu.jacobian(g, cams, plan)
    r = np.random.default_rng(57)
    assert np.all(jac.gn_apply(0.05, np.zeros(jac.param_dim())) == 0)
    for _ in range(5):
        p1, p2 = r.uniform(-1, 1, (2, jac.param_dim()))
        a1, a2 = jac.gn_apply(0.05, p1), jac.gn_apply(0.05, p2)
        assert rel_error(float(p1 @ a2), float(p2 @ a1)) < TOL
        assert float(p1 @ a1) >= 0.05 * float(p1 @ p1) * (1 - TOL)
        a12 = jac.gn_apply(0.05, 1.7 * p1 - 0.6 * p2)
        assert norm_rel(a12, 1.7 * a1 - 0.6 * a2) < TOL
    assert np.all(jac.jtj_diag() >= 0)


@pytest.mark.parametrize("seed,n,size,spt", [(140, 12, 48, 32), (77, 30, 64, 13), (5, 40, 80, 64)])
def test_products_vs_oracle_fresh_cases(gpu, port, seed, n, size, spt):
    rng = MT64(seed)
    g = random_scene(n, rng)
    cams = [tcam(size, 3.0), tcam(size // 2 + 8, 3.2)]
    plan = port.build_sample_plan(cams, spt, 0, port.rng(seed), lane_width=1)
    ja, jb = gpu.jacobian(g, cams, plan), port.jacobian(g, cams, plan)
    r = np.random.default_rng(seed)
    v, u, p = r.uniform(-1, 1, ja.param_dim()), r.uniform(-1, 1, ja.residual_dim()), r.uniform(-1, 1, ja.param_dim())
    assert norm_rel(ja.jvp(v), jb.jvp(v)) < TOL
    assert norm_rel(ja.vjp(u), jb.vjp(u)) < TOL
    assert norm_rel(ja.jtj_diag(), jb.jtj_diag()) < TOL
    assert norm_rel(ja.gn_apply(0.1, p), jb.gn_apply(0.1, p)) < TOL


def test_empty_plan_views(gpu):
    """test_autodiff.cpp:226: an empty plan gives zero products."""
    g = random_scene(6, MT64(52))
    cams = [tcam(32, 3.0)]
    plan = SamplePlan(np.array([0], np.int32), np.array([0, 0], np.int64), np.zeros(0, np.int32),
                      np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0))
    jac = gpu.jacobian(g, cams, plan)
    assert np.all(jac.jtj_diag() == 0)
    assert np.all(jac.gn_apply(0.1, np.zeros(jac.param_dim())) == 0)


def test_jacobian_errors(gpu):
    g = random_scene(3, MT64(47))
    cams = [tcam(32, 3.0)]
    plan = gpu.build_sample_plan(cams, 16, 0, gpu.rng(1), lane_width=1)
    jac = gpu.jacobian(g, cams, plan)
    with pytest.raises(ValueError):
        jac.vjp(np.ones(3))
    bad = SamplePlan(np.array([3], np.int32), plan.view_offset, plan.px, plan.py, plan.tile, plan.weight)
    with pytest.raises(ValueError):
        gpu.jacobian(g, cams, bad)


# ----------------------------------------------------------------- PCG / solver
def test_pcg_dense_operator(gpu):
    """test_solver.cpp:44-107 through the host-operator PCG."""
    b = np.arange(1.0, 8.0)
    res = gpu.pcg_dense(np.eye(7), b, np.ones(7), 5)
    assert res.iterations == 1 and not res.breakdown and np.allclose(res.x, b, rtol=1e-6)
    res = gpu.pcg_dense(np.eye(5), np.zeros(5), np.ones(5), 5)
    assert res.iterations == 0 and np.all(res.x == 0)
    r = np.random.default_rng(91)
    for _ in range(10):
        n = int(r.integers(2, 21))
        a = r.uniform(-1, 1, (n, n))
        m = a.T @ a + 0.1 * np.eye(n)
        bb = r.uniform(-1, 1, n)
        res = gpu.pcg_dense(m, bb, 1.0 / np.diag(m), n + 3)
        assert np.linalg.norm(m @ res.x - bb) / np.linalg.norm(bb) < 1e-3
    m = np.eye(4)
    m[2, 2] = -2.0
    assert gpu.pcg_dense(m, np.array([0, 0, 1.0, 0]), np.ones(4), 10).breakdown


def test_learning_rate(gpu):
    cfg = LmConfig()
    delta = np.zeros(28)
    delta[11] = 123.0
    assert gpu.learning_rate(delta, 5, cfg) == 0.05
    delta[11] = 10.0
    assert gpu.learning_rate(delta, 50, cfg) == pytest.approx(0.1)
    delta[:] = 0
    delta[0] = 99.0
    assert gpu.learning_rate(delta, 50, cfg) == pytest.approx(0.2)
    delta[14 + 13] = -10.0
    assert gpu.learning_rate(delta, 50, cfg) == pytest.approx(0.1)


def test_apply_update(gpu, port):
    g = random_scene(20, MT64(3))
    h = g.copy()
    delta = np.random.default_rng(0).uniform(-1, 1, 14 * 20)
    gpu.apply_update(g, delta, 0.2)
    port.apply_update(h, delta, 0.2)
    assert np.max(np.abs(g.pack() - h.pack())) < 1e-12


# ----------------------------------------------------------------- lm_step
def test_lm_trajectory_vs_reference(gpu):
    """12 free-running LM steps on the toy scene vs the reference's own run:
    identical view batches (RNG replay), losses within 1e-4 relative."""
    d = golden("lm")
    tc = g_cams(d["toy_train_cams"])
    rng = gpu.rng(1)
    st = gpu.random_init(40, [-1, -1, -1], [1, 1, 1], rng)
    assert st == g_set(d, "lm_init")
    td = gpu.train_data(tc, list(d["toy_train_imgs"]))
    td.rebuild_clusters(8, 1 ^ 0x9E3779B97F4A7C15)
    cfg = LmConfig(pcg_iters_initial=8, pcg_iters_late=8)
    worst = 0.0
    for it, row in enumerate(d["lm_reports"]):
        r = gpu.lm_step(st, td, cfg, it, rng)
        assert r.batch == [int(b) for b in row[6:]]
        assert r.pcg_iterations == int(row[4]) and r.breakdown == bool(row[5])
        assert r.eta == pytest.approx(row[3], rel=1e-6)
        worst = max(worst, rel_error(r.loss_before, row[1]), rel_error(r.loss_after, row[2]))
    print("worst per-iteration loss rel err", worst)
    assert worst < TOL
    assert rng() == int(d["lm_rng_next"][0])  # same RNG position: samplers replayed exactly
    assert norm_rel(st.pack(), g_set(d, "lm_final").pack()) < 1e-3


@pytest.mark.parametrize("dist", [0, 1])
def test_lm_speculation_discarded_when_inputs_change(gpu, port, dist):
    """lm_step draws the next step's batch + plan speculatively during its PCG; a
    caller that touches the RNG or rebuilds the clusters between steps must get
    exactly the reference's draws (the speculation is discarded)."""
    gt, tc, ti, _, _ = port.toy_scene(20, 8, 1, 64, 20214)
    rg, ro = gpu.rng(5), port.rng(5)
    sg = gpu.random_init(60, [-1, -1, -1], [1, 1, 1], rg)
    so = port.random_init(60, [-1, -1, -1], [1, 1, 1], ro)
    tdg, tdo = gpu.train_data(tc, list(ti)), port.train_data(tc, list(ti))
    for td in (tdg, tdo):
        td.rebuild_clusters(4, 7)
    cfg = LmConfig(batch_size_initial=4, pcg_iters_initial=4, dist=dist)
    for it in range(5):
        if it == 2:  # the caller consumes the RNG between steps
            assert rg() == ro()
        if it == 3:  # ... and rebuilds the clusters (batch size change, run.cpp:145-153)
            for td in (tdg, tdo):
                td.rebuild_clusters(3, 11)
            cfg = LmConfig(batch_size_initial=3, pcg_iters_initial=4, dist=dist)
        a, b = gpu.lm_step(sg, tdg, cfg, it, rg), port.lm_step(so, tdo, cfg, it, ro)
        assert a.batch == b.batch, f"step {it}: batch {a.batch} vs {b.batch}"
        assert rel_error(a.loss_after, b.loss_after) < TOL
    assert rg() == ro()  # same RNG position


def test_lm_step_fixed_point(gpu, port):
    """test_solver.cpp:132: at zero residual the step does not move the state."""
    gt, tc, ti, sc, si = port.toy_scene(8, 4, 1, 32, 93)
    imgs = [gpu.render_full(gt, c)[0].astype(np.float32) for c in tc]
    td = gpu.train_data(tc, imgs)
    td.rebuild_clusters(4, 1)
    st = gt.copy()
    r = gpu.lm_step(st, td, LmConfig(batch_size_initial=4), 0, gpu.rng(94))
    assert r.loss_before < 1e-10
    assert np.max(np.abs(st.pack() - gt.pack())) < 1e-5


@pytest.mark.parametrize("count", [3000, 20000])
def test_long_tile_lists_sorted_exactly(gpu, port, count):
    """Lists beyond the 2048-entry CTA sort (smem 16384 path) and beyond 16384
    (chunk + merge-path path) still match the reference order bit for bit."""
    from paper_2504_12905_b200.types import GaussianSet
    r = np.random.default_rng(count)
    g = GaussianSet(count)
    g.means = r.uniform(-0.3, 0.3, 3 * count)
    g.log_scales = np.full(3 * count, np.log(0.6))  # every splat covers the whole image
    g.rotations = r.uniform(-1, 1, 4 * count)
    g.renormalize_rotations()
    g.opacity_logits = r.uniform(-1, 2, count)
    g.colors = r.uniform(-1, 1, 3 * count)
    cam = tcam(48, 3.0)
    oo, io = port.bin_and_sort(g, cam)
    og, ig = gpu.bin_and_sort(g, cam)
    assert int(np.max(np.diff(oo))) > (2048 if count < 10000 else 16384)
    assert np.array_equal(oo, og) and np.array_equal(io, ig)


def test_cpp_adapter_drop_in(gpu):
    """The reference's own C++ caller code (tests/cpp/adapter_parity.cpp) run
    on the reference CPU path and through include/splatlm_b200.hpp: same view
    batches and RNG stream, losses and gn_apply within 1e-4."""
    import json
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                       "adapter_parity")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/adapter_parity not built (needs /root/reference at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    r = json.loads(out.stdout.strip().splitlines()[-1])
    print(r)
    assert r["batches_equal"] and r["rng_equal"]
    assert r["worst_loss_rel"] < TOL and r["gn_apply_rel"] < TOL
    assert r["split_psnr_diff"] < 1e-3 and r["split_ssim_diff"] < 1e-5
    assert r["eval_ssim_diff"] <= 1e-12 and r["eval_mse_rel"] <= 1e-12
    assert r["full_gradient_rel"] < TOL and r["first_order_equal"]
    # render:: surface (render_full / render_with_context / render_pixel / residuals) and
    # the one-shot autodiff wrappers through the adapter
    assert r["render_contrib_equal"] and r["residuals_equal"]
    assert r["render_image_diff"] < 1e-12 and r["render_t_diff"] < 1e-12 and r["render_pixel_diff"] < 1e-12
    assert r["one_shot_gn_rel"] < TOL


@pytest.mark.gpu
def test_cfg0_psnr_curve_matches_reference(gpu):
    """configs[0] (toy scene, 10k Gaussians, 8 x 256^2 full pixels, PCG 8): the test-split
    PSNR after each of the 10 LM iterations is within +-0.05 dB of the reference's own run
    (tests/golden/psnr_cfg0.json, made by tests/golden/make_psnr_target.py)."""
    import json

    import bench
    from paper_2504_12905_b200 import splatlm
    from paper_2504_12905_b200.types import LmConfig

    ref = json.load(open(bench.PSNR_TARGET))
    c = ref["config"]
    L = gpu
    train, timgs, test, simgs = bench.cfg0_scene(L, c)
    td = L.train_data(train, timgs)
    td.set_clusters(L.kmeans_cameras(train, c["batch"], c["seed"] ^ bench.KMEANS_SALT))
    rng = L.rng(c["seed"])
    scene = splatlm.Scene(L, L.random_init(c["gaussians"], [-1, -1, -1], [1, 1, 1], rng))
    cfg = LmConfig(pcg_iters_initial=c["pcg"], pcg_iters_late=c["pcg"], batch_size_initial=c["batch"],
                   batch_size_late=c["batch"], samples_per_tile=c["spt"])
    sd = L.train_data(test, simgs)
    for it, (rp, rl) in enumerate(zip(ref["psnr"], ref["loss_after"])):
        rep = scene.lm_step(td, cfg, it, rng)
        p = np.mean([bench.psnr(scene.render(cam)[0], im) for cam, im in zip(test, simgs)])
        ev = scene.evaluate_split(sd)  # device evaluate_split agrees with the host PSNR
        assert abs(ev.psnr - p) <= 1e-6
        assert abs(p - rp) <= 0.05, f"iteration {it}: PSNR {p:.4f} vs reference {rp:.4f}"
        assert abs(rep.loss_after - rl) <= 1e-3 * rl, f"iteration {it}: loss {rep.loss_after} vs {rl}"


@pytest.mark.gpu
@pytest.mark.parametrize("spread,n,levels", [(0.0, 300, 5), (1e-12, 300, 5), (1e-9, 300, 5), (1e-7, 300, 5),
                                             (1e-12, 300, 0), (1e-10, 6000, 0), (1e-11, 20000, 0), (1e-8, 20000, 9)])
def test_tile_lists_bit_exact_near_equal_depths(gpu, spread, n, levels):
    """Depth ties and near-ties (equal upper 32 key bits, distinct doubles): the
    radix tile-list construction sorts the upper halves, then fixes up runs -- short
    ones per thread, long ones (a near-planar scene: runs of thousands) per CTA
    (bitonic chunks + merge path); the order must still be the reference's
    (depth, index) order, bit for bit."""
    from oracle.cpu_bind import port

    rng = np.random.default_rng(11)
    g = GaussianSet.zeros(n)
    # levels > 0: that many distinct depths (exact ties); 0: n distinct depths within `spread`
    dz = spread * (rng.integers(0, levels, n) if levels else rng.uniform(0.0, 1.0, n))
    g.means = np.column_stack([rng.uniform(-0.6, 0.6, n), rng.uniform(-0.6, 0.6, n),
                               np.full(n, 0.25) + dz]).reshape(-1)
    g.log_scales = np.full(3 * n, math.log(0.2))
    g.rotations = np.tile([1.0, 0.0, 0.0, 0.0], n)
    g.opacity_logits = rng.uniform(-0.5, 1.0, n)
    g.colors = rng.uniform(-1, 1, 3 * n)
    cam = tcam(64)
    o_off, o_idx = port().bin_and_sort(g, cam)
    off, idx = gpu.bin_and_sort(g, cam)
    assert np.array_equal(off, o_off)
    assert np.array_equal(idx, o_idx)


# ----------------------------------------------------------------- metrics
@pytest.mark.parametrize("i", range(5))
def test_evaluate_matches_reference(gpu, i):
    """metrics::evaluate on the device (metrics.cu) vs the reference's own mse / psnr /
    ssim (tests/golden/metrics.npz).  Every filtered moment and local SSIM value is
    computed in the reference's f64 operation order; only the pixel sums are ordered
    differently, hence 1e-12."""
    d = golden("metrics")
    a, b = d[f"m{i}_a"], d[f"m{i}_b"]
    mse, psnr, ssim = d[f"m{i}_ref"]
    r = gpu.evaluate(a, b)
    assert abs(r.ssim - ssim) <= 1e-12
    assert r.mse == pytest.approx(mse, rel=1e-12)
    assert r.psnr == pytest.approx(psnr, rel=1e-12)
    s = gpu.evaluate(a, a)
    assert (s.mse, s.psnr, s.ssim) == tuple(d[f"m{i}_self"])


def test_evaluate_full_size_matches_oracle(gpu, port):
    """A 1280x720 pair (configs[2] view size; tile edges not multiples of 32) vs the C
    restatement, which is bitwise equal to the reference's ssim."""
    rng = np.random.default_rng(3)
    a = rng.random((720, 1280, 3))
    b = np.clip(a + rng.normal(0, 0.03, a.shape), 0, 1)
    r = gpu.evaluate(a, b)
    assert abs(r.ssim - port.ssim(a, b)) <= 1e-12
    assert r.mse == pytest.approx(port.mse(a, b), rel=1e-12)
    with pytest.raises(Exception):
        gpu.evaluate(a, b[:10])


def test_evaluate_split_matches_reference(gpu):
    """io::evaluate_split (run.cpp:77-92) of the toy LM run's final state on its 4 test
    views: device renders (f32) + device metrics vs the reference's f64 render_full +
    evaluate.  The render is f32, so the bars are 1e-3 dB PSNR and 1e-5 SSIM."""
    d = golden("lm")
    g = g_set(d, "lm_final")
    split = gpu.train_data(g_cams(d["toy_test_cams"]), list(d["toy_test_imgs"]))
    ref = golden("metrics")["split_metrics"].mean(axis=0)
    r = gpu.evaluate_split(g, split)
    print(r, ref)
    assert r.mse == pytest.approx(ref[0], rel=1e-4)
    assert abs(r.psnr - ref[1]) <= 1e-3
    assert abs(r.ssim - ref[2]) <= 1e-5


@pytest.mark.parametrize("i", range(5))
def test_ssim_diag_residuals_match_reference(gpu, i):
    """metrics::ssim_diag_residuals on the device vs the reference's outputs: every
    value is computed in the reference's f64 operation order, so bit for bit."""
    d = golden("metrics")
    r, dc = gpu.ssim_diag_residuals(d[f"m{i}_a"], d[f"m{i}_b"])
    print("max |dres|", np.abs(r - d[f"m{i}_sres"]).max(), "max |ddc|", np.abs(dc - d[f"m{i}_sdc"]).max())
    assert np.array_equal(r, d[f"m{i}_sres"])
    assert np.array_equal(dc, d[f"m{i}_sdc"])


def test_lm_trajectory_mse_ssim_vs_reference(gpu):
    """8 LM steps with the mse+ssim loss (lm.cpp:86-119: diagonal SSIM rows folded into
    the rhs and the per-channel weights) vs the reference's run: identical batches,
    losses within 1e-4, then batch_loss(mse+ssim) of the final state."""
    d = golden("lm_ssim")
    dl = golden("lm")
    tc = g_cams(dl["toy_train_cams"])
    imgs = list(dl["toy_train_imgs"])
    rng = gpu.rng(1)
    st = gpu.random_init(40, [-1, -1, -1], [1, 1, 1], rng)
    td = gpu.train_data(tc, imgs)
    td.rebuild_clusters(8, 1 ^ 0x9E3779B97F4A7C15)
    cfg = LmConfig(pcg_iters_initial=8, pcg_iters_late=8, loss=1, ssim_weight=0.2)
    worst = 0.0
    for it, row in enumerate(d["lms_reports"]):
        r = gpu.lm_step(st, td, cfg, it, rng)
        assert r.batch == [int(b) for b in row[6:]]
        assert r.pcg_iterations == int(row[4]) and r.breakdown == bool(row[5])
        assert r.eta == pytest.approx(row[3], rel=1e-6)
        worst = max(worst, rel_error(r.loss_before, row[1]), rel_error(r.loss_after, row[2]))
    print("worst per-iteration loss rel err", worst)
    assert worst < TOL
    assert rng() == int(d["lms_rng_next"][0])
    assert norm_rel(st.pack(), g_set(d, "lms_final").pack()) < 1e-3
    ref_final = g_set(d, "lms_final")
    bl = gpu.batch_loss(ref_final, td, list(range(len(tc))), loss=1, ssim_weight=0.2)
    assert rel_error(bl, float(d["lms_batch_loss"][0])) < TOL


@pytest.mark.parametrize("dist", [1, 2])
def test_lm_weighted_distributions_vs_oracle(gpu, port, dist):
    """lm_step with the weighted residual distributions (sample_plan.cpp:127-165:
    kResidual softmax, kGaussianCount): the host draws the uniforms from the caller's
    RNG in the reference's order, the device builds the per-tile CDFs from the render
    and picks the pixels.  Batches and the RNG position are exact; the pixel picks
    use the f32 render's CDF (the reference's is f64), so a draw landing within
    rounding of a CDF step may pick the neighbour -- losses agree to 1e-4."""
    gt, tc, ti, _, _ = port.toy_scene(20, 8, 1, 64, 20214)
    rg, ro = gpu.rng(3), port.rng(3)
    sg = gpu.random_init(60, [-1, -1, -1], [1, 1, 1], rg)
    so = port.random_init(60, [-1, -1, -1], [1, 1, 1], ro)
    tdg, tdo = gpu.train_data(tc, list(ti)), port.train_data(tc, list(ti))
    for td in (tdg, tdo):
        td.rebuild_clusters(8, 5)
    cfg = LmConfig(pcg_iters_initial=8, samples_per_tile=32, dist=dist)
    worst = 0.0
    for it in range(6):
        a, b = gpu.lm_step(sg, tdg, cfg, it, rg), port.lm_step(so, tdo, cfg, it, ro)
        assert a.batch == b.batch
        worst = max(worst, rel_error(a.loss_before, b.loss_before), rel_error(a.loss_after, b.loss_after))
    print("dist", dist, "worst loss rel err", worst)
    assert worst < TOL
    assert rg() == ro()


# ----------------------------------------------------------------- first-order baselines (§8f rank 4)
@pytest.mark.parametrize("loss", [0, 1])
def test_full_gradient_vs_reference(gpu, loss):
    """baselines::full_gradient on the device (exhaustive plan laid out tile-major,
    u = 2/M (r + w s s'), the LM path's J^T pass) vs the reference's gradient."""
    d = golden("first_order")
    dl = golden("lm")
    split = gpu.train_data(g_cams(dl["toy_train_cams"]), list(dl["toy_train_imgs"]))
    g = gpu.full_gradient(g_set(dl, "lm_init"), split, loss, 0.2)
    err = norm_rel(g, d["fo_grad_ssim" if loss else "fo_grad_mse"])
    print("full_gradient rel err", err)
    assert err < TOL


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_first_order_step_bitwise(gpu, port, kind):
    """first_order_step on the device on a given gradient: f64 state and moments, the
    reference's operation order, so state and moments are bitwise the C restatement's
    (which is bitwise the reference's, tests/test_oracle.py)."""
    from paper_2504_12905_b200.types import FirstOrderConfig
    d = golden("first_order")
    st0 = g_set(golden("lm"), "lm_init")
    cfg = FirstOrderConfig(kind=kind, decay_iterations=3)
    a, b = st0.copy(), st0.copy()
    n = 14 * st0.count
    ma1, ma2, mb1, mb2, sa, sb = np.zeros(n), np.zeros(n), np.zeros(n), np.zeros(n), 0, 0
    for it in range(4):
        grad = d["fo_grad_mse"] * (1.0 + 0.5 * it)
        sa = gpu.first_order_step(a, ma1, ma2, sa, grad, cfg)
        sb = port.first_order_step(b, mb1, mb2, sb, grad, cfg)
    assert sa == sb == 4
    assert np.array_equal(a.pack(), b.pack())
    assert np.array_equal(ma1, mb1) and np.array_equal(ma2, mb2)


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_first_order_training_vs_reference(gpu, kind):
    """Six train_run iterations of a first-order optimizer entirely on the device
    (full_gradient + step + batch_loss, run.cpp:176-182) vs the reference's losses."""
    from paper_2504_12905_b200 import splatlm
    from paper_2504_12905_b200.types import FirstOrderConfig
    d = golden("first_order")
    dl = golden("lm")
    data = gpu.train_data(g_cams(dl["toy_train_cams"]), list(dl["toy_train_imgs"]))
    scene = splatlm.Scene(gpu, g_set(dl, "lm_init"))
    fo = splatlm.FirstOrder(gpu, scene)
    extra = FirstOrderConfig.sgd_paper_lrs() if kind == 2 else {}
    cfg = FirstOrderConfig(kind=kind, decay_iterations=6, **extra)
    worst = 0.0
    for it in range(6):
        worst = max(worst, rel_error(fo.step(data, cfg), d[f"fo{kind}_losses"][it]))
    print("kind", kind, "worst loss rel err", worst)
    assert worst < TOL
    assert norm_rel(scene.download().pack(), g_set(d, f"fo{kind}_final").pack()) < 1e-3


# ----------------------------------------------------------------- run driver (§8f rank 3)
@pytest.mark.parametrize("case", ["lm", "adam"])
def test_train_run_matches_reference(gpu, tmp_path, case):
    """io::train_run on the toy scene, deterministic mode, every step on the device vs the
    reference's own run (tests/golden/run.npz): metrics.csv has the same header, rows and
    empty-field pattern with values within tolerance, summary.json the same keys and
    settings, checkpoint.bin the same header and .meta.txt with parameters close."""
    import json

    from paper_2504_12905_b200.run import RunConfig, train_run
    from paper_2504_12905_b200.types import GaussianSet
    iters, every = (6, 3) if case == "lm" else (4, 2)
    cfg = RunConfig(optimizer=case, iterations=iters, eval_every=every, out_dir=str(tmp_path),
                    deterministic=True, lm=LmConfig(pcg_iters_initial=8))
    res = train_run(gpu, cfg)
    g = golden("run")
    mine = (tmp_path / "metrics.csv").read_text().splitlines()
    ref = bytes(g[f"{case}_metrics.csv"]).decode().splitlines()
    assert mine[0] == ref[0] and len(mine) == len(ref)
    for a, b in zip(mine[1:], ref[1:]):
        fa, fb = a.split(","), b.split(",")
        assert [x == "" for x in fa] == [x == "" for x in fb], (a, b)
        assert fa[0] == fb[0] and fa[6:] == fb[6:]  # iter, pcg_iters, breakdown
        assert rel_error(float(fa[2]), float(fb[2])) < TOL  # train_loss
        if fb[3]:
            assert abs(float(fa[3]) - float(fb[3])) < 0.01 and abs(float(fa[4]) - float(fb[4])) < 1e-3
        if fb[5]:
            assert float(fa[5]) == pytest.approx(float(fb[5]), rel=1e-6)
    sm, sr = json.loads((tmp_path / "summary.json").read_text()), json.loads(bytes(g[f"{case}_summary.json"]))
    assert sm.keys() == sr.keys()
    for k, v in sr.items():
        if isinstance(v, float) and k not in ("damping",):
            assert abs(sm[k] - v) <= 1e-3 * max(1.0, abs(v)), k
        else:
            assert sm[k] == v, k
    ck = (tmp_path / "checkpoint.bin").read_bytes()
    ref_ck = bytes(g[f"{case}_checkpoint.bin"])
    assert ck[:20] == ref_ck[:20] and len(ck) == len(ref_ck)
    assert (tmp_path / "checkpoint.bin.meta.txt").read_bytes() == bytes(g[f"{case}_checkpoint.bin.meta.txt"])
    assert norm_rel(np.frombuffer(ck[20:], "<f8"), np.frombuffer(ref_ck[20:], "<f8")) < 1e-3
    assert res.final_train_loss == pytest.approx(sr["final_train_loss"], rel=TOL)
    # eval_run on the checkpoint reproduces the final test metrics
    from paper_2504_12905_b200.run import eval_run
    ev = eval_run(gpu, RunConfig(out_dir=str(tmp_path / "eval")), res.checkpoint)
    assert ev.psnr == pytest.approx(res.final_test.psnr, abs=1e-9)
    assert GaussianSet  # noqa


# ----------------------------------------------------------------- misc
def test_evaluate_edge_cases(gpu):
    """metrics::evaluate on identical, constant and empty images (test_metrics.cpp:88-99):
    ssim(a, a) == 1, psnr capped at 100 dB, empty images give mse 0 / ssim 1."""
    a = np.full((9, 13, 3), 0.25)
    r = gpu.evaluate(a, a)
    assert (r.mse, r.psnr, r.ssim) == (0.0, 100.0, 1.0)
    b = np.full((9, 13, 3), 0.75)
    c = gpu.evaluate(a, b)
    assert c.mse == pytest.approx(0.25) and c.psnr == pytest.approx(10 * math.log10(4.0))
    e = gpu.evaluate(np.zeros((0, 0, 3)), np.zeros((0, 0, 3)))
    assert (e.mse, e.psnr, e.ssim) == (0.0, 100.0, 1.0)


def test_train_run_wall_clock_column(gpu, tmp_path):
    """Non-deterministic mode fills wall_ms with %.3f (run.cpp:54-75)."""
    from paper_2504_12905_b200.run import METRICS_CSV_HEADER, RunConfig, train_run
    train_run(gpu, RunConfig(optimizer="sgd", iterations=2, eval_every=0, out_dir=str(tmp_path),
                             deterministic=False))
    rows = (tmp_path / "metrics.csv").read_text().splitlines()
    assert rows[0] == METRICS_CSV_HEADER and len(rows) == 3
    for row in rows[1:]:
        f = row.split(",")
        assert len(f) == 8 and f[1] and len(f[1].split(".")[1]) == 3 and f[5] == f[6] == f[7] == ""
    assert rows[-1].split(",")[3]  # the last iteration is always evaluated


# ----------------------------------------------------------------- §8f rows: exact weighted draws, weights API
@pytest.mark.parametrize("dist", [1, 2])
def test_weighted_sample_sets_bit_exact_vs_reference(gpu, reflib, dist):
    """kResidual / kGaussianCount (sample_plan.cpp:127-165): the device builds each tile's
    density and CDF from the FP64 render (k_render_exact) and picks with the host's
    uniforms; the reference builds them from its own render_full.  Two LM steps: the
    picked pixels of every sample equal the reference's plan, weights to f32 rounding."""
    gt, tc, ti, _, _ = reflib.toy_scene(20, 8, 1, 64, 20214)
    rg, rr = gpu.rng(3), reflib.rng(3)
    st = gpu.random_init(60, [-1, -1, -1], [1, 1, 1], rg)
    assert st == reflib.random_init(60, [-1, -1, -1], [1, 1, 1], rr)
    td = gpu.train_data(tc, list(ti))
    td.rebuild_clusters(8, 5)
    clusters = td.clusters()
    cfg = LmConfig(pcg_iters_initial=4, samples_per_tile=32, dist=dist)
    for it in range(2):
        batch = reflib.sample_view_batch(clusters, rr)
        aux = []
        for v in batch:
            img, _, cn = reflib.render_full(st, tc[v])
            aux.append((img, cn, np.asarray(ti[v], np.float64)))
        plan = reflib.build_sample_plan([tc[v] for v in batch], 32, dist, rr, 32, aux=aux)
        rep = gpu.lm_step(st, td, cfg, it, rg)
        assert rep.batch == batch
        px, py, w = gpu.last_samples()
        assert np.array_equal(px, plan.px) and np.array_equal(py, plan.py)
        want = (plan.weight / plan.total_samples()).astype(np.float32)
        assert np.max(np.abs(w - want) / want) <= 1e-6
        assert rg() == rr()  # same RNG position (one uniform per draw)
        rg, rr = gpu.rng(100 + it), reflib.rng(100 + it)


def test_set_residual_weights_vs_reference(gpu, reflib):
    """SampledJacobian::set_residual_weights (jacobian.cpp:121-125): custom per-residual
    weights round-trip through residual_weights() and change jtj_diag / gn_apply like
    the reference's; a wrong length raises std::invalid_argument (ValueError)."""
    d = golden("jacobian")
    st = g_set(d, "jx")
    cams = g_cams(d["jx_cams"])
    plan = g_plan(d, "jx")
    jg, jr = gpu.jacobian(st, cams, plan), reflib.jacobian(st, cams, plan)
    w = np.random.default_rng(4).uniform(0.1, 3.0, jg.residual_dim()) * jg.residual_weights()
    jg.set_residual_weights(w)
    jr.set_residual_weights(w)
    assert np.array_equal(jg.residual_weights(), w)
    p = np.random.default_rng(5).uniform(-1, 1, jg.param_dim())
    assert norm_rel(jg.gn_apply(0.1, p), jr.gn_apply(0.1, p)) < TOL
    assert norm_rel(jg.jtj_diag(), jr.jtj_diag()) < TOL
    with pytest.raises(ValueError):
        jg.set_residual_weights(w[:-1])


# ----------------------------------------------------------------- render:: surface
@pytest.mark.parametrize("t", range(4))
def test_render_with_context_and_pixel_vs_reference(gpu, reflib, t):
    """render::render_with_context on the reference's own prepared splats and tile grid
    (prepare_camera, rasterizer.cpp:10-50) equals its render_full: contributor counts
    exactly, colour and transmittance to 1e-12; render_pixel over one tile's ordered
    list equals the reference pixel; residuals is rendered - truth."""
    d = golden("render")
    g = g_set(d, f"r{t}")
    cam = g_cams(d[f"r{t}_cam"])[0]
    prep = reflib.prepare(g, cam)
    splats = gpu.pack_splats(prep)
    off, idx = reflib.bin_and_sort(g, cam)
    img, tr, cn = gpu.render_with_context(cam, splats, off, idx)
    ri, rt, rc = reflib.render_full(g, cam)
    assert np.array_equal(cn, rc)
    assert np.max(np.abs(img - ri)) < 1e-12 and np.max(np.abs(tr - rt)) < 1e-12
    tile = len(off) // 2
    order = idx[off[tile]:off[tile + 1]]
    x0, y0 = (tile % cam.tiles_x) * 16, (tile // cam.tiles_x) * 16
    x, y = x0 + min(7, cam.width - 1 - x0), y0 + min(7, cam.height - 1 - y0)
    rgb, T, c = gpu.render_pixel(splats[order], x + 0.5, y + 0.5)
    assert c == rc[y, x] and abs(T - rt[y, x]) < 1e-12 and np.max(np.abs(rgb - ri[y, x])) < 1e-12
    assert np.array_equal(gpu.residuals(img, ri), img - ri)
    with pytest.raises(ValueError):
        gpu.residuals(img, ri[:1])
