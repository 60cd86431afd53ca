"""Pin the C restatement (oracle/liboracle.so) against the real reference.

Two anchors, both CPU-only (no GPU):
* the committed golden fixtures (tests/golden/*.npz, produced by the
  unmodified reference through tests/golden/make_golden.py) — always run;
* the live reference (oracle/_ref) where it was built — extra cross-checks.

Integer / index outputs (tile lists, sample plans, clusters, RNG streams) must
be bit-exact; double outputs are compared bitwise where the restatement keeps
the reference operation order, else to 1e-12 relative.
"""
import numpy as np
import pytest

from paper_2504_12905_b200.types import LmConfig, SamplePlan
from support import MT64, g_cams, g_plan, g_set, golden, norm_rel, random_scene
from support import test_camera as tcam


def test_mt19937_64_stream(port):
    d = golden("sampling")
    r = port.rng(2024)
    got = np.array([r() for _ in range(1000)], np.uint64)
    assert np.array_equal(got, d["mt_first"])
    m = MT64(2024)
    assert [m() for _ in range(1000)] == [int(x) for x in d["mt_first"]]


@pytest.mark.parametrize("t", range(20))
def test_tile_lists_and_render_random_scenes(port, t):
    """test_render.cpp:122 seeds: tile lists bit-exact, render bitwise."""
    d = golden("render")
    g = g_set(d, f"r{t}")
    cam = g_cams(d[f"r{t}_cam"])[0]
    off, idx = port.bin_and_sort(g, cam)
    assert np.array_equal(off, d[f"r{t}_offsets"])
    assert np.array_equal(idx, d[f"r{t}_indices"])
    img, tr, cn = port.render_full(g, cam)
    assert np.array_equal(img, d[f"r{t}_image"])
    assert np.array_equal(tr, d[f"r{t}_trans"])
    assert np.array_equal(cn, d[f"r{t}_contrib"])


@pytest.mark.parametrize("i", range(3))
def test_ring_views_prepare_bin_render(port, i):
    d = golden("render")
    g = g_set(d, "ring")
    cam = g_cams(d["ring_cams"])[i]
    p = port.prepare(g, cam)
    for k, v in p.items():
        assert np.array_equal(v, d[f"ring{i}_prep_{k}"]), k
    off, idx = port.bin_and_sort(g, cam)
    assert np.array_equal(off, d[f"ring{i}_offsets"])
    assert np.array_equal(idx, d[f"ring{i}_indices"])
    img, tr, cn = port.render_full(g, cam)
    assert np.array_equal(img, d[f"ring{i}_image"])
    assert np.array_equal(cn, d[f"ring{i}_contrib"])


def _plan_eq(a: SamplePlan, d, prefix):
    for k in ("view_camera", "view_offset", "px", "py", "tile", "weight"):
        assert np.array_equal(getattr(a, k), d[f"{prefix}_{k}"]), k


def test_sample_plans_bit_exact(port):
    d = golden("sampling")
    _plan_eq(port.build_sample_plan([tcam(40, 3.0)], 32, 0, port.rng(65)), d, "u32")
    _plan_eq(port.build_sample_plan([tcam(32, 3.0)], 256, 0, port.rng(64)), d, "u256")
    _plan_eq(port.build_sample_plan([tcam(40, 3.0)], 13, 0, port.rng(7), lane_width=1), d, "u13")
    batch = g_cams(d["batch_cams"])
    _plan_eq(port.build_sample_plan(batch, 64, 0, port.rng(123)), d, "b64")
    _plan_eq(port.exhaustive_plan(g_cams(d["ex_cams"])), d, "ex")


def test_sample_plan_known_answers(port):
    """test_sampling.cpp:160-215: exhaustive weights, per-tile counts, validation."""
    plan = port.build_sample_plan([tcam(32, 3.0)], 256, 0, port.rng(64))
    assert len(set(zip(plan.px, plan.py))) == 32 * 32
    assert np.allclose(plan.weight, 1024.0)
    plan = port.build_sample_plan([tcam(40, 3.0)], 32, 0, port.rng(65))
    assert plan.total_samples() == 4 * 32 + 4 * 32 + 32
    with pytest.raises(ValueError):
        port.build_sample_plan([tcam(32, 3.0)], 257, 0, port.rng(1), lane_width=1)
    with pytest.raises(ValueError):
        port.build_sample_plan([tcam(32, 3.0)], 0, 0, port.rng(1))
    with pytest.raises(ValueError):
        port.build_sample_plan([tcam(32, 3.0)], 48, 0, port.rng(1))


def test_kmeans_and_features(port):
    d = golden("sampling")
    cams = g_cams(d["km_cams"])
    assert np.array_equal(port.camera_features(cams), d["km_features"])
    clusters = port.kmeans_cameras(cams, 8, 1 ^ 0x9E3779B97F4A7C15)
    assign = np.zeros(len(cams), np.int32)
    for c, m in enumerate(clusters):
        assign[m] = c
    assert np.array_equal(assign, d["km_assign"])


@pytest.mark.parametrize("name", ["jx", "js", "jr"])
def test_jacobian_products(port, name):
    d = golden("jacobian")
    g = g_set(d, name)
    cams = g_cams(d[f"{name}_cams"])
    jac = port.jacobian(g, cams, g_plan(d, name))
    assert np.array_equal(jac.residual_weights(), d[f"{name}_weights"])
    assert np.array_equal(jac.jvp(d[f"{name}_v"]), d[f"{name}_jvp"])
    assert np.array_equal(jac.vjp(d[f"{name}_u"]), d[f"{name}_vjp"])
    assert np.array_equal(jac.jtj_diag(), d[f"{name}_diag"])
    assert np.array_equal(jac.gn_apply(0.1, d[f"{name}_p"]), d[f"{name}_gn"])
    minv = 1.0 / (d[f"{name}_diag"] + 0.1)
    res = jac.pcg(0.1, d[f"{name}_vjp"], minv, 8)
    meta = d[f"{name}_pcg_meta"]
    assert res.iterations == int(meta[0]) and res.breakdown == bool(meta[1])
    assert norm_rel(res.x, d[f"{name}_pcg_x"]) < 1e-12


def test_lm_trajectory(port):
    """Free-running 12-step LM trajectory: batches exact, losses and state bitwise."""
    d = golden("lm")
    tc = g_cams(d["toy_train_cams"])
    rng = port.rng(1)
    st = port.random_init(40, [-1, -1, -1], [1, 1, 1], rng)
    assert st == g_set(d, "lm_init")
    td = port.train_data(tc, list(d["toy_train_imgs"]))
    td.rebuild_clusters(8, 1 ^ 0x9E3779B97F4A7C15)
    cfg = LmConfig(pcg_iters_initial=8, pcg_iters_late=8)
    for it, row in enumerate(d["lm_reports"]):
        r = port.lm_step(st, td, cfg, it, rng)
        assert r.batch == [int(b) for b in row[6:]]
        assert r.pcg_iterations == int(row[4]) and r.breakdown == bool(row[5])
        assert r.eta == row[3]
        assert abs(r.loss_before - row[1]) <= 1e-12 * row[1]
        assert abs(r.loss_after - row[2]) <= 1e-12 * row[2]
    assert np.max(np.abs(st.pack() - g_set(d, "lm_final").pack())) <= 1e-12
    assert rng() == int(d["lm_rng_next"][0])


def test_toy_scene_generator(port):
    d = golden("lm")
    gt, tc, ti, sc, si = port.toy_scene(20, 8, 4, 64, 20214)
    assert gt == g_set(d, "toy_gt")
    assert np.array_equal(ti, d["toy_train_imgs"])
    assert np.array_equal(si, d["toy_test_imgs"])


def test_pcg_dense_known_answers(port):
    """test_solver.cpp:44-107: identity in one step, zero rhs, dense SPD, breakdown."""
    b = np.arange(1.0, 8.0)
    res = port.pcg_dense(np.eye(7), b, np.ones(7), 5)
    assert res.iterations == 1 and not res.breakdown and np.allclose(res.x, b, rtol=1e-12)
    res = port.pcg_dense(np.eye(5) * 2, np.zeros(5), np.ones(5), 5)
    assert res.iterations == 0 and np.all(res.x == 0)
    g = np.random.default_rng(91)
    for _ in range(20):
        n = int(g.integers(2, 21))
        a = g.uniform(-1, 1, (n, n))
        m = a.T @ a + 0.1 * np.eye(n)
        bb = g.uniform(-1, 1, n)
        res = port.pcg_dense(m, bb, 1.0 / np.diag(m), n + 3)
        assert np.linalg.norm(m @ res.x - bb) / np.linalg.norm(bb) <= 1e-8
    m = np.eye(4)
    m[2, 2] = -2.0
    assert port.pcg_dense(m, np.array([0, 0, 1.0, 0]), np.ones(4), 10).breakdown


def test_learning_rate_known_answers(port):
    """test_solver.cpp:109-130."""
    cfg = LmConfig()
    delta = np.zeros(28)
    delta[11] = 123.0
    assert port.learning_rate(delta, 5, cfg) == 0.05
    delta[11] = 10.0
    assert port.learning_rate(delta, 50, cfg) == pytest.approx(0.1)
    delta[11] = 0.5
    assert port.learning_rate(delta, 50, cfg) == pytest.approx(0.2)
    delta[:] = 0
    delta[0] = 99.0
    assert port.learning_rate(delta, 50, cfg) == pytest.approx(0.2)
    delta[14 + 11 + 2] = -10.0
    assert port.learning_rate(delta, 50, cfg) == pytest.approx(0.1)


def test_live_reference_cross_check(port, reflib):
    """Where the reference is built: a fresh random case through both."""
    rng = MT64(777)
    g = random_scene(30, rng)
    cams = [tcam(48, 3.0)]
    plan = reflib.build_sample_plan(cams, 32, 0, reflib.rng(5), lane_width=1)
    plan2 = port.build_sample_plan(cams, 32, 0, port.rng(5), lane_width=1)
    assert np.array_equal(plan.px, plan2.px) and np.array_equal(plan.weight, plan2.weight)
    ja, jb = reflib.jacobian(g, cams, plan), port.jacobian(g, cams, plan)
    p = np.random.default_rng(0).uniform(-1, 1, ja.param_dim())
    assert np.array_equal(ja.gn_apply(0.1, p), jb.gn_apply(0.1, p))
    assert np.array_equal(ja.jtj_diag(), jb.jtj_diag())


@pytest.mark.parametrize("i", range(5))
def test_image_metrics_known_answers(port, i):
    """metrics::mse / psnr / ssim (image_metrics.cpp:108-139) on the reference's own
    outputs (tests/golden/metrics.npz): the SSIM restatement keeps the reference's
    operation order (bitwise); the MSE sum order differs from the AVX2 kernel (1e-12)."""
    d = golden("metrics")
    a, b = d[f"m{i}_a"], d[f"m{i}_b"]
    mse, psnr, ssim = d[f"m{i}_ref"]
    assert port.ssim(a, b) == ssim
    assert port.mse(a, b) == pytest.approx(mse, rel=1e-12)
    assert port.psnr(a, b) == pytest.approx(psnr, rel=1e-12)
    assert [port.mse(a, a), port.psnr(a, a), port.ssim(a, a)] == list(d[f"m{i}_self"])


def test_ssim_live_reference(port, reflib):
    rng = np.random.default_rng(9)
    for h, w in [(6, 11), (33, 20), (128, 96)]:
        a = rng.random((h, w, 3))
        b = np.clip(a + rng.normal(0, 0.1, a.shape), 0, 1)
        assert port.ssim(a, b) == reflib.ssim(a, b)


@pytest.mark.parametrize("i", range(5))
def test_ssim_diag_residuals_known_answers(port, i):
    """metrics::ssim_diag_residuals (image_metrics.cpp:141-178): residual s and centre
    derivative, bitwise against the reference's outputs."""
    d = golden("metrics")
    r, dc = port.ssim_diag_residuals(d[f"m{i}_a"], d[f"m{i}_b"])
    assert np.array_equal(r, d[f"m{i}_sres"])
    assert np.array_equal(dc, d[f"m{i}_sdc"])
    # identical images: zero residuals and derivatives (test_metrics.cpp:120-126)
    z, zd = port.ssim_diag_residuals(d[f"m{i}_a"], d[f"m{i}_a"])
    assert not z.any() and not zd.any()


def test_lm_trajectory_mse_ssim(port):
    """lm_step with the mse+ssim loss (lm.cpp:86-119): the diagonal SSIM rows fold into the
    rhs and the per-channel weights; losses and state against the reference's run."""
    d = golden("lm_ssim")
    dl = golden("lm")
    tc = g_cams(dl["toy_train_cams"])
    rng = port.rng(1)
    st = port.random_init(40, [-1, -1, -1], [1, 1, 1], rng)
    td = port.train_data(tc, list(dl["toy_train_imgs"]))
    td.rebuild_clusters(8, 1 ^ 0x9E3779B97F4A7C15)
    cfg = LmConfig(pcg_iters_initial=8, pcg_iters_late=8, loss=1, ssim_weight=0.2)
    for it, row in enumerate(d["lms_reports"]):
        r = port.lm_step(st, td, cfg, it, rng)
        assert r.batch == [int(b) for b in row[6:]]
        assert r.pcg_iterations == int(row[4]) and r.breakdown == bool(row[5])
        assert r.eta == row[3]
        assert abs(r.loss_before - row[1]) <= 1e-12 * row[1]
        assert abs(r.loss_after - row[2]) <= 1e-12 * row[2]
    assert np.max(np.abs(st.pack() - g_set(d, "lms_final").pack())) <= 1e-12
    assert rng() == int(d["lms_rng_next"][0])
    bl = port.batch_loss(st, tc, list(dl["toy_train_imgs"]), loss=1, ssim_weight=0.2)
    assert bl == pytest.approx(float(d["lms_batch_loss"][0]), rel=1e-12)


def test_first_order_baselines_vs_reference(port):
    """baselines::full_gradient and the Adam / RMSprop / SGD-momentum trajectories
    (first_order.cpp) on the toy scene vs the reference's outputs (golden)."""
    from paper_2504_12905_b200.types import FirstOrderConfig
    d = golden("first_order")
    dl = golden("lm")
    tc, ti = g_cams(dl["toy_train_cams"]), list(dl["toy_train_imgs"])
    st0 = g_set(dl, "lm_init")
    assert norm_rel(port.full_gradient(st0, tc, ti, 0), d["fo_grad_mse"]) < 1e-12
    assert norm_rel(port.full_gradient(st0, tc, ti, 1, 0.2), d["fo_grad_ssim"]) < 1e-12
    for kind in (0, 1, 2):
        extra = FirstOrderConfig.sgd_paper_lrs() if kind == 2 else {}
        cfg = FirstOrderConfig(kind=kind, decay_iterations=6, **extra)
        st = st0.copy()
        m1, m2, step = np.zeros(st.count * 14), np.zeros(st.count * 14), 0
        for it in range(6):
            step = port.first_order_step(st, m1, m2, step, port.full_gradient(st, tc, ti, 0), cfg)
            assert port.batch_loss(st, tc, ti) == pytest.approx(d[f"fo{kind}_losses"][it], rel=1e-12)
        assert norm_rel(st.pack(), g_set(d, f"fo{kind}_final").pack()) < 1e-12
        assert norm_rel(m1, d[f"fo{kind}_m1"]) < 1e-12 or not d[f"fo{kind}_m1"].any()


def test_first_order_default_config(reflib):
    """FirstOrderConfig defaults (first_order.hpp:12-37) match the reference's."""
    import ctypes as C
    from paper_2504_12905_b200.types import CFirstOrderConfig, FirstOrderConfig
    fn = reflib.lib.ref_default_first_order_config
    fn.argtypes = [C.POINTER(CFirstOrderConfig)]
    fn.restype = None
    c = CFirstOrderConfig()
    fn(C.byref(c))
    mine = FirstOrderConfig().to_c()
    for name, _ in CFirstOrderConfig._fields_:
        assert getattr(c, name) == getattr(mine, name), name
