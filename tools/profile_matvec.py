"""Driver for ncu captures of the configs[2] hot path (one GPU).

    ncu --set full -k regex:k_sample_raster -s 2 -c 1 -o prof python tools/profile_matvec.py

Builds the bench workload (1M Gaussians, 8 views 1280x720, N=32), runs a few
J^T W J p products, one diag and (with --lm) one LM step.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--products", type=int, default=3)
    ap.add_argument("--gaussians", type=int, default=1_000_000)
    ap.add_argument("--diag", action="store_true")
    ap.add_argument("--lm", action="store_true")
    ap.add_argument("--passes", action="store_true")
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_2504_12905_b200 import splatlm
    args = bench.parse_args_for(a.gaussians)
    L = splatlm.Lib(0)
    state, cams, clusters, batch, plan = bench.host_inputs(L, args, 1)
    scene = splatlm.Scene(L, state)
    jac = scene.jacobian([cams[i] for i in batch], plan)
    P = 14 * scene.padded
    p = torch.empty(P, device="cuda").uniform_(-1, 1)
    u = torch.zeros(P, device="cuda")
    L.synchronize()
    for _ in range(a.products):
        jac.gn_apply_dev(0.1, p.data_ptr(), u.data_ptr())
    L.synchronize()
    if a.diag:
        jac.jtj_diag()
    if a.passes:  # pass 1 alone (JVP) and pass 2 alone (VJP) through the host API
        v = np.random.default_rng(0).uniform(-1, 1, jac.param_dim())
        jv = jac.jvp(v)
        jac.vjp(jv)
    if a.lm:
        gt = splatlm.Scene(L, bench.gt_scene(a.gaussians // 2, H=L))
        imgs = [gt.render(c)[0] for c in cams]
        td = L.train_data(cams, imgs)
        td.set_clusters(clusters)
        rng = L.rng(1)
        L.random_init(a.gaussians, [-1, -1, -1], [1, 1, 1], rng)
        scene.lm_step(td, bench.LmConfig(pcg_iters_initial=8, pcg_iters_late=8), 0, rng)
        L.render_full(state, cams[batch[0]])  # the FP64 drop-in render (k_render_exact)
    L.synchronize()
    print("done", jac.stats())


if __name__ == "__main__":
    main()
