"""The view-sharded multi-rank path on ONE GPU (GPU).

Two contexts of this process act as ranks 0 and 1 of an in-process group
(slm_local_group, the collective seam's single-process implementation; the
deployment uses NCCL with one process per GPU).  Each rank replays
the host RNG for the whole batch, owns its slice of the views, and the
J^T W J p products, the fused [b | diag] and the loss scalars are summed over
the ranks -- exactly the world > 1 code path of lm_step.  The world-2 run must
draw the same batches, end at the same RNG position, keep the ranks' states
bitwise identical, and match the world-1 run to the float tolerance (the sums
over views are associated differently).
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from paper_2504_12905_b200.types import LmConfig
from support import g_cams, golden, norm_rel, rel_error

pytestmark = pytest.mark.gpu
STEPS = 8


def _setup(L, n=40):
    d = golden("lm")
    tc = g_cams(d["toy_train_cams"])
    rng = L.rng(1)
    st = L.random_init(n, [-1, -1, -1], [1, 1, 1], rng)
    td = L.train_data(tc, list(d["toy_train_imgs"]))
    td.rebuild_clusters(8, 1 ^ 0x9E3779B97F4A7C15)
    return st, td, rng


def _run(L, cfg, n=40):
    st, td, rng = _setup(L, n)
    reps = [L.lm_step(st, td, cfg, it, rng) for it in range(STEPS)]
    return [(r.loss_before, r.loss_after, r.eta, r.pcg_iterations, tuple(r.batch)) for r in reps], st.pack(), rng()


def _world2(cfg, chunks=4, n=40):
    from paper_2504_12905_b200 import splatlm
    group = splatlm.LocalGroup(2)
    libs = [splatlm.Lib(0), splatlm.Lib(0)]
    for r, L in enumerate(libs):
        L.init_local(group, r)
        L.set_comm_chunks(chunks)
    with ThreadPoolExecutor(2) as ex:
        out = list(ex.map(lambda L: _run(L, cfg, n), libs))
    return out


@pytest.mark.parametrize("loss,chunks,n", [(0, 1, 40), (1, 3, 40), (0, 1, 2000), (0, 4, 2000), (1, 3, 2000)])
def test_two_ranks_match_one(loss, chunks, n):
    """chunks: the product's chain + allreduce pipeline depth (1 = one allreduce); with
    2000 Gaussians the chain runs in up to 4 chunks of 512."""
    from paper_2504_12905_b200 import splatlm
    cfg = LmConfig(pcg_iters_initial=8, pcg_iters_late=8, loss=loss, ssim_weight=0.2)
    one = _run(splatlm.Lib(0), cfg, n)
    r0, r1 = _world2(cfg, chunks, n)
    # the ranks agree bit for bit (replicated CG vectors, rank-order sums)
    assert r0[0] == r1[0] and np.array_equal(r0[1], r1[1]) and r0[2] == r1[2]
    # same batches and RNG position as one rank; losses and state to the float tolerance
    worst = 0.0
    for a, b in zip(r0[0], one[0]):
        assert a[4] == b[4] and a[3] == b[3]
        worst = max(worst, rel_error(a[0], b[0]), rel_error(a[1], b[1]))
    print("world 2 vs 1: worst loss rel err", worst, "state", norm_rel(r0[1], one[1]))
    assert worst < 1e-4
    assert r0[2] == one[2]
    assert norm_rel(r0[1], one[1]) < 1e-4


def test_two_ranks_bitwise_reproducible():
    cfg = LmConfig(pcg_iters_initial=8, pcg_iters_late=8)
    a, b = _world2(cfg), _world2(cfg)
    assert a[0][0] == b[0][0] and np.array_equal(a[0][1], b[0][1])


def test_nccl_seam_one_rank():
    """The NCCL implementation of the collective seam (the deployment's, one
    process per GPU) in one process: dlopen of the NCCL library (PyTorch's
    bundled one, as bench.py picks it), unique id, a one-rank communicator, and
    the product path's f32 / f64 allreduce and grouped row allreduce on known
    data -- the calls and enums the multi-GPU runs make, exercised on one B200."""
    import os
    try:
        import nvidia.nccl
        os.environ.setdefault("SLM_NCCL_LIB", os.path.join(os.path.dirname(nvidia.nccl.__file__), "lib",
                                                           "libnccl.so.2"))
    except Exception:
        pass
    from paper_2504_12905_b200 import splatlm
    err, n = splatlm.lib().nccl_selftest()
    assert n > 0 and err == 0.0
