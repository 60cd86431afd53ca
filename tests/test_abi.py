"""CPU-side checks of the product library (no GPU needed).

* libslm_b200.so loads and exports every entry point include/slm_b200.h declares;
* the host samplers (build_sample_plan, exhaustive_plan, k-means view
  batching, random_init) reproduce the reference's sampled pixel sets and RNG
  stream bit for bit (north-star "bit-exact: sampled pixel sets");
* without a CUDA device the compute path refuses to run (no CPU fallback).
"""
import os
import re

import numpy as np
import pytest

from paper_2504_12905_b200 import splatlm
from support import g_cams, golden
from support import test_camera as tcam

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def host():
    from paper_2504_12905_b200.build import build
    build()
    return splatlm.HostSampler()


def test_exports_every_declared_symbol(host):
    hdr = open(os.path.join(ROOT, "include", "slm_b200.h")).read()
    names = set(re.findall(r"\b(slm_[a-z0-9_]+)\s*\(", hdr))
    names.discard("slm_apply_fn")
    assert len(names) > 50
    dll = splatlm.load_library()
    missing = [n for n in sorted(names) if not hasattr(dll, n)]
    assert not missing, missing


def _plan_eq(a, d, prefix):
    for k in ("view_camera", "view_offset", "px", "py", "tile", "weight"):
        assert np.array_equal(getattr(a, k), d[f"{prefix}_{k}"]), k


def test_sample_plans_bit_exact(host):
    d = golden("sampling")
    _plan_eq(host.build_sample_plan([tcam(40, 3.0)], 32, 0, host.rng(65)), d, "u32")
    _plan_eq(host.build_sample_plan([tcam(32, 3.0)], 256, 0, host.rng(64)), d, "u256")
    _plan_eq(host.build_sample_plan([tcam(40, 3.0)], 13, 0, host.rng(7), lane_width=1), d, "u13")
    _plan_eq(host.build_sample_plan(g_cams(d["batch_cams"]), 64, 0, host.rng(123)), d, "b64")
    _plan_eq(host.exhaustive_plan(g_cams(d["ex_cams"])), d, "ex")


def test_sample_plan_validation(host):
    """test_sampling.cpp:204-215: N>256, N=0, N % lane != 0 -> invalid_argument."""
    cams = [tcam(32, 3.0)]
    for n, lane in ((257, 1), (0, 32), (48, 32)):
        with pytest.raises(ValueError):
            host.build_sample_plan(cams, n, 0, host.rng(1), lane_width=lane)
    with pytest.raises(ValueError):
        host.build_sample_plan(cams, 32, 1, host.rng(1))  # residual dist without aux


def test_weighted_plans_match_port(host, port):
    """Residual / contributor-count distributions draw through the CDF."""
    rng = np.random.default_rng(5)
    cams = [tcam(40, 3.0), tcam(24, 3.0)]
    aux = []
    for c in cams:
        aux.append((rng.uniform(0, 1, (c.height, c.width, 3)),
                    rng.integers(0, 30, (c.height, c.width)).astype(np.int32),
                    rng.uniform(0, 1, (c.height, c.width, 3))))
    for dist in (1, 2):
        a = host.build_sample_plan(cams, 32, dist, host.rng(9), aux=aux)
        b = port.build_sample_plan(cams, 32, dist, port.rng(9), aux=aux)
        for k in ("px", "py", "tile", "weight", "view_offset"):
            assert np.array_equal(getattr(a, k), getattr(b, k)), (dist, k)


def test_random_init_and_rng_stream(host):
    d = golden("lm")
    from support import g_set
    g = host.random_init(40, [-1, -1, -1], [1, 1, 1], host.rng(1))
    assert g == g_set(d, "lm_init")
    r = host.rng(2024)
    assert np.array_equal(np.array([r() for _ in range(1000)], np.uint64), golden("sampling")["mt_first"])


def test_kmeans_features_and_batch(host, port):
    d = golden("sampling")
    cams = g_cams(d["km_cams"])
    assert np.array_equal(host.camera_features(cams), d["km_features"])
    cl = host.kmeans_cameras(cams, 8, 1 ^ 0x9E3779B97F4A7C15)
    assign = np.zeros(len(cams), np.int32)
    for c, m in enumerate(cl):
        assign[m] = c
    assert np.array_equal(assign, d["km_assign"])
    # sample_view_batch consumes the engine like the reference (view_sampler.cpp:173-184)
    a = host.sample_view_batch(cl, host.rng(77))
    r = port.rng(77)
    from support import MT64
    m = MT64(77)
    want = [members[m.uniform_int(0, len(members) - 1)] for members in cl]
    assert a == [int(x) for x in want]


def test_ring_camera_matches_reference_generator(host, port):
    a = host.ring_camera(1.234, 3.2, 1.1, 64)
    b = port.ring_camera(1.234, 3.2, 1.1, 64)
    assert np.array_equal(a.world_to_cam, b.world_to_cam)
    assert np.array_equal(a.translation, b.translation) and a.fx == b.fx


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(splatlm.CudaUnavailable):
        splatlm.Lib()


# ---- run-driver wire formats: host code, no GPU needed
def _golden_bytes(name):
    return bytes(golden("run")[name])


def test_checkpoint_bytes_match_reference(tmp_path):
    """io::save_checkpoint / load_checkpoint (checkpoint.cpp:12-82): a file written by the
    reference loads here bit for bit, and writing it back reproduces the reference's bytes
    and .meta.txt exactly."""
    import ctypes as C

    from paper_2504_12905_b200.types import CGaussians, GaussianSet
    dll = splatlm.load_library()
    src = tmp_path / "ref.bin"
    src.write_bytes(_golden_bytes("lm_checkpoint.bin"))
    n = C.c_int32()
    assert dll.slm_checkpoint_count(os.fsencode(str(src)), C.byref(n)) == 0 and n.value == 40
    g = GaussianSet(n.value)
    cg = g.to_c()
    assert dll.slm_load_checkpoint(os.fsencode(str(src)), C.byref(cg)) == 0
    raw = np.frombuffer(_golden_bytes("lm_checkpoint.bin")[20:], "<f8")
    assert np.array_equal(g.pack(), raw)
    out = tmp_path / "mine.bin"
    assert dll.slm_save_checkpoint(os.fsencode(str(out)), C.byref(cg)) == 0
    assert out.read_bytes() == _golden_bytes("lm_checkpoint.bin")
    assert (tmp_path / "mine.bin.meta.txt").read_bytes() == _golden_bytes("lm_checkpoint.bin.meta.txt")
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOTSPLAT" + bytes(12))
    assert dll.slm_checkpoint_count(os.fsencode(str(bad)), C.byref(n)) != 0
    assert b"not a splatlm checkpoint" in dll.slm_last_error()
    g2 = GaussianSet(3)
    cg2 = g2.to_c()
    assert dll.slm_load_checkpoint(os.fsencode(str(src)), C.byref(cg2)) != 0  # count mismatch


def test_summary_json_layout_matches_reference():
    """summary.json is nlohmann dump(2): sorted keys, shortest round-trip doubles; the
    driver's writer reproduces the reference's bytes from the same values."""
    import json

    from paper_2504_12905_b200.run import METRICS_CSV_HEADER, _json_dump
    for case in ("lm", "adam"):
        ref = _golden_bytes(f"{case}_summary.json").decode()
        assert _json_dump(json.loads(ref)) == ref
        assert _golden_bytes(f"{case}_metrics.csv").decode().splitlines()[0] == METRICS_CSV_HEADER


def test_estimate_loss_matches_reference(host, port):
    """sampling::estimate_loss (sample_plan.cpp:199-222): the library's host version is
    bitwise the reference's (same summation order) on uniform and weighted plans, and on
    the exhaustive plan it equals the MSE (test_sampling.cpp:171-174)."""
    import oracle
    from oracle.cpu_bind import ref
    libs = [port] + ([ref()] if oracle.have_ref() else [])
    rng = np.random.default_rng(12)
    cams = [tcam(40, 3.0), tcam(32, 2.5), tcam(48, 3.0)]
    fields = [rng.normal(0, 0.3, (c.height, c.width, 3)) for c in cams]
    plans = [host.build_sample_plan(cams, 32, 0, host.rng(7)), host.exhaustive_plan(cams)]
    aux = [(rng.random((c.height, c.width, 3)), rng.integers(0, 9, (c.height, c.width)).astype(np.int32),
            rng.random((c.height, c.width, 3))) for c in cams]
    plans.append(host.build_sample_plan(cams, 32, 1, host.rng(8), aux=aux))
    plans.append(host.build_sample_plan(cams, 16, 2, host.rng(9), 16, aux=aux))
    for plan in plans:
        mine = host.estimate_loss(cams, plan, fields)
        for lib in libs:
            assert mine == lib.estimate_loss(cams, plan, fields), lib.kind
    pixels = sum(c.width * c.height for c in cams)
    mse = sum(float(np.sum(f ** 2)) for f in fields) / (3 * pixels)
    assert host.estimate_loss(cams, plans[1], fields) == pytest.approx(mse, rel=1e-12)
    with pytest.raises(ValueError):
        host.estimate_loss(cams, plans[0], fields[:2])


def test_large_uniform_plans_parallel_path_bit_exact(host, port):
    """Uniform plans of >= 65536 samples take the parallel path (raw mt19937_64
    outputs drawn in order, per-tile shuffles on several threads): the sampled
    pixels, weights and the RNG position after the plan are the C restatement's
    (pinned bitwise to the reference) -- full-pixel 256x256 views (configs[0])
    and a 1280x720 view at 64 samples per tile, two plans in a row each."""
    from support import test_camera as tc
    for cams, spt in (([tc(256, 3.0 + 0.1 * i) for i in range(8)], 256), ([tc(1280, 3.0)], 64)):
        ra, rb = host.rng(31), port.rng(31)
        for _ in range(2):
            a = host.build_sample_plan(cams, spt, 0, ra)
            b = port.build_sample_plan(cams, spt, 0, rb)
            assert len(a.px) >= 65536
            for k in ("view_camera", "view_offset", "px", "py", "tile", "weight"):
                assert np.array_equal(getattr(a, k), getattr(b, k)), k
        assert ra() == rb(), "RNG position after the plans"
