"""Run-to-run reproducibility of the device path (GPU).

The reference's contract: every result is bitwise independent of scheduling
(jacobian.cpp:19-21,246-247 -- a fixed 16-chunk ordered merge), "same seed,
same trajectory" (test_solver.cpp:268-286), byte-identical CSV and checkpoint
on rerun (acceptance_main.cpp:436-468, cli_test.sh:21-25).  Here the J^T and
diag(J^T W J) accumulations run in a fixed per-plan slot order (DetOrder,
chain.cu det_gather) -- the default -- so products, PCG solutions, LM
trajectories and run-driver files are compared with ==, not a tolerance.
"""
import numpy as np
import pytest

from paper_2504_12905_b200.types import LmConfig
from support import g_cams, g_set, golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    from paper_2504_12905_b200 import splatlm
    L = splatlm.lib()
    L.set_deterministic(True)
    return L


def _products(jac, seed=0):
    r = np.random.default_rng(seed)
    p = r.uniform(-1, 1, jac.param_dim())
    u = r.uniform(-1, 1, jac.residual_dim())
    return [jac.gn_apply(0.1, p), jac.vjp(u), jac.jtj_diag(), jac.jvp(p)]


def _toy_inputs(port, n=400, views=4, size=96, spt=32, seed=3):
    gt, tc, ti, _, _ = port.toy_scene(20, views, 1, size, 20214)
    st = port.random_init(n, [-1, -1, -1], [1, 1, 1], port.rng(seed))
    plan = port.build_sample_plan(tc[:views], spt, 0, port.rng(seed + 1))
    return st, tc[:views], plan


def test_products_bitwise_reproducible(gpu, port):
    """gn_apply / vjp / jtj_diag / jvp: repeated on one Jacobian and on a freshly
    built one (new plan order, new buffers), results are bitwise equal."""
    st, cams, plan = _toy_inputs(port)
    ja = gpu.jacobian(st, cams, plan)
    first = _products(ja)
    again = _products(ja)
    jb = gpu.jacobian(st, cams, plan)
    fresh = _products(jb)
    for a, b, c in zip(first, again, fresh):
        assert np.array_equal(a, b)
        assert np.array_equal(a, c)


def test_slot_order_counting_equals_radix(gpu, port, monkeypatch):
    """The per-plan summation order built by counting placement + per-key segment
    sort (default) is the stable radix order: products bitwise equal."""
    st, cams, plan = _toy_inputs(port, n=600, seed=5)
    monkeypatch.setenv("SLM_SLOT_ORDER", "radix")
    radix = _products(gpu.jacobian(st, cams, plan))
    monkeypatch.setenv("SLM_SLOT_ORDER", "counting")
    counting = _products(gpu.jacobian(st, cams, plan))
    for a, b in zip(radix, counting):
        assert np.array_equal(a, b)


def test_slot_order_with_a_splat_in_every_group(gpu, port, monkeypatch):
    """One wide, faint splat at the origin is blended in nearly every group of the
    plan (one key with over 64 slots: the counting path's guard hands the plan to
    the radix passes); products still equal the radix order bitwise."""
    st, cams, plan = _toy_inputs(port, n=600, size=192, seed=7)
    st.means[0:3] = 0.0
    st.log_scales[0:3] = np.log(0.8)
    st.opacity_logits[0] = -2.0
    monkeypatch.setenv("SLM_SLOT_ORDER", "radix")
    radix = _products(gpu.jacobian(st, cams, plan))
    monkeypatch.setenv("SLM_SLOT_ORDER", "counting")
    counting = _products(gpu.jacobian(st, cams, plan))
    for a, b in zip(radix, counting):
        assert np.array_equal(a, b)


def test_pcg_bitwise_reproducible(gpu, port):
    st, cams, plan = _toy_inputs(port, n=300, seed=9)
    jac = gpu.jacobian(st, cams, plan)
    r = np.random.default_rng(1)
    b = r.uniform(-1, 1, jac.param_dim())
    minv = 1.0 / (jac.jtj_diag() + 0.1)
    x1, x2 = jac.pcg(0.1, b, minv, 8), jac.pcg(0.1, b, minv, 8)
    assert np.array_equal(x1.x, x2.x) and x1.iterations == x2.iterations


def _lm_run(gpu, cfg, steps=8):
    d = golden("lm")
    tc = g_cams(d["toy_train_cams"])
    rng = gpu.rng(1)
    st = gpu.random_init(40, [-1, -1, -1], [1, 1, 1], rng)
    td = gpu.train_data(tc, list(d["toy_train_imgs"]))
    td.rebuild_clusters(8, 1 ^ 0x9E3779B97F4A7C15)
    reps = [gpu.lm_step(st, td, cfg, it, rng) for it in range(steps)]
    return [(r.loss_before, r.loss_after, r.eta, r.pcg_iterations, r.breakdown, tuple(r.batch)) for r in reps], \
        st.pack(), rng()


@pytest.mark.parametrize("loss,dist", [(0, 0), (1, 0), (0, 1), (0, 2)])
def test_lm_trajectory_bitwise_reproducible(gpu, loss, dist):
    """test_solver.cpp:268-286 ("same seed, same trajectory"): two 8-step lm_step runs
    from the same seed give bitwise-equal reports, final state and RNG position --
    mse, mse+ssim and both weighted residual distributions."""
    cfg = LmConfig(pcg_iters_initial=8, pcg_iters_late=8, loss=loss, ssim_weight=0.2, dist=dist,
                   samples_per_tile=32 if dist else 256)
    a = _lm_run(gpu, cfg)
    b = _lm_run(gpu, cfg)
    assert a[0] == b[0]
    assert np.array_equal(a[1], b[1])
    assert a[2] == b[2]


def test_mse_ssim_trajectory_reproducible_vs_reference(gpu):
    """The mse+ssim trajectory that was flaky at 1e-4 with float atomics: three reruns,
    all bitwise equal to each other, and within 1e-4 of the reference's run."""
    from support import rel_error
    d = golden("lm_ssim")
    cfg = LmConfig(pcg_iters_initial=8, pcg_iters_late=8, loss=1, ssim_weight=0.2)
    runs = [_lm_run(gpu, cfg, steps=len(d["lms_reports"])) for _ in range(3)]
    for r in runs[1:]:
        assert r[0] == runs[0][0] and np.array_equal(r[1], runs[0][1])
    worst = max(max(rel_error(a[0], row[1]), rel_error(a[1], row[2]))
                for a, row in zip(runs[0][0], d["lms_reports"]))
    print("worst per-iteration loss rel err", worst)
    assert worst < 1e-4


def test_train_run_files_byte_identical(gpu, tmp_path):
    """acceptance_main.cpp:436-468 / cli_test.sh:21-25: two deterministic train_run
    invocations write byte-identical metrics.csv, summary.json and checkpoint."""
    from paper_2504_12905_b200.run import RunConfig, train_run
    outs = []
    for k in range(2):
        out = tmp_path / f"run{k}"
        train_run(gpu, RunConfig(optimizer="lm", iterations=5, eval_every=2, out_dir=str(out), deterministic=True,
                                 lm=LmConfig(pcg_iters_initial=8)))
        outs.append(out)
    for name in ("metrics.csv", "summary.json", "checkpoint.bin", "checkpoint.bin.meta.txt"):
        assert (outs[0] / name).read_bytes() == (outs[1] / name).read_bytes(), name


def test_atomic_mode_still_available(gpu, port):
    """set_deterministic(False) selects the float red.global.add accumulation: same
    products to FP32 rounding (the order-dependent last bits are the only difference)."""
    from support import norm_rel
    st, cams, plan = _toy_inputs(port, seed=5)
    det = _products(gpu.jacobian(st, cams, plan))
    gpu.set_deterministic(False)
    try:
        fast = _products(gpu.jacobian(st, cams, plan))
    finally:
        gpu.set_deterministic(True)
    for a, b in zip(det, fast):
        assert norm_rel(b, a) < 1e-5
