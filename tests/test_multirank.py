"""Multi-rank view sharding on CPU (gloo, world_size 2).

The B200 lm_step shards the LM batch's views across ranks
(slm_view_slice), every rank replaying the host RNG for the whole batch, and
allreduces J^T W J p, b and diag(J^T W J) over ranks.  That is
correct iff those quantities are sums over views with the GLOBAL weights
(1/q)/N_total.  Here each gloo rank evaluates its slice with the oracle
(the C restatement, pinned to the reference), the partials are allreduced
over gloo, and the result must equal the single-process full-batch value.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_12905_b200 import splatlm


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _slice(n, rank, world):
    import ctypes as C
    lo, hi = C.c_int(), C.c_int()
    assert splatlm.dll().slm_view_slice(n, rank, world, C.byref(lo), C.byref(hi)) == 0
    return lo.value, hi.value


def _problem(port):
    from support import MT64, random_scene
    from paper_2504_12905_b200.types import ring_camera
    g = port.random_init(300, [-1, -1, -1], [1, 1, 1], port.rng(9))
    cams = [ring_camera(0.5 * i, 3.2, 1.1, 64, 48) for i in range(5)]
    plan = port.build_sample_plan(cams, 32, 0, port.rng(11))
    return g, cams, plan


def _worker(rank, world, master_port, out):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(master_port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from oracle.cpu_bind import port as P
    from paper_2504_12905_b200.types import SamplePlan
    lib = P()
    g, cams, plan = _problem(lib)
    lo, hi = _slice(plan.n_views, rank, world)
    a, b = int(plan.view_offset[lo]), int(plan.view_offset[hi])
    sub = SamplePlan(plan.view_camera[lo:hi].copy(), plan.view_offset[lo:hi + 1] - a, plan.px[a:b],
                     plan.py[a:b], plan.tile[a:b], plan.weight[a:b], plan.samples_per_tile)
    jac = lib.jacobian(g, cams, sub)
    inv_total = 1.0 / plan.total_samples()  # global N_total (sample_plan.cpp:86-94)
    jac.set_residual_weights(np.repeat(sub.weight * inv_total, 3))
    p = np.random.default_rng(0).uniform(-1, 1, jac.param_dim())
    u = np.random.default_rng(1).uniform(-1, 1, 3 * plan.total_samples())[3 * a:3 * b]
    parts = [jac.gn_apply(0.0, p), jac.vjp(u), jac.jtj_diag()]
    red = []
    for x in parts:
        t = torch.from_numpy(x.copy())
        dist.all_reduce(t)
        red.append(t.numpy())
    if rank == 0:
        np.save(out, np.stack(red))
    dist.destroy_process_group()


def test_view_slices_partition_the_batch():
    for n in (1, 5, 8, 32):
        for world in (1, 2, 3, 8):
            covered = []
            for r in range(world):
                lo, hi = _slice(n, r, world)
                assert lo <= hi
                covered.extend(range(lo, hi))
            assert covered == list(range(n))


def test_two_rank_sum_over_views_matches_full_batch(port, tmp_path):
    out = str(tmp_path / "reduced.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    reduced = np.load(out)
    g, cams, plan = _problem(port)
    jac = port.jacobian(g, cams, plan)
    p = np.random.default_rng(0).uniform(-1, 1, jac.param_dim())
    u = np.random.default_rng(1).uniform(-1, 1, jac.residual_dim())
    full = [jac.gn_apply(0.0, p), jac.vjp(u), jac.jtj_diag()]
    for got, want in zip(reduced, full):
        assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)
