"""configs[3]: pixel-sampling ratio sweep at 500k Gaussians (convergence vs cost).

    python tools/spt_sweep.py [--steps 6]

800x800 views (configs[3] leaves the size unstated; SURVEY §8 uses 800^2), 64 ring
views, 8-view LM batch, PCG 8.  For N in {13, 32, 64, 128, 256} samples per
16x16 tile (5%..100%): J^T W J p products/s, LM iterations/s and the batch loss
after each LM step (random_init state vs a 250k-Gaussian ground truth).
Prints one JSON line per N.
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2504_12905_b200 import splatlm  # noqa: E402
from paper_2504_12905_b200.types import LmConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--gaussians", type=int, default=500_000)
    a = ap.parse_args()
    args = bench.parse_args_for(a.gaussians)
    args.views, args.width, args.height = 64, 800, 800
    L = splatlm.Lib(0)
    cams = bench.cameras(args)
    gt = splatlm.Scene(L, bench.gt_scene(a.gaussians // 2, H=L))
    imgs = [gt.render(c)[0] for c in cams]
    del gt
    td = L.train_data(cams, imgs)
    td.set_clusters(L.kmeans_cameras(cams, 8, 1 ^ bench.KMEANS_SALT))
    for n in (13, 32, 64, 128, 256):
        lane = 13 if n == 13 else 32
        rng = L.rng(1)
        scene = splatlm.Scene(L, L.random_init(a.gaussians, [-1, -1, -1], [1, 1, 1], rng))
        cfg = LmConfig(pcg_iters_initial=8, pcg_iters_late=8, samples_per_tile=n, sample_lane_width=lane)
        # products/s on this step's Jacobian
        H = splatlm.HostSampler()
        r2 = H.rng(7)
        batch = H.sample_view_batch(td.clusters if hasattr(td, "clusters") else list(range(8)), r2) \
            if False else list(range(0, 64, 8))
        plan = L.build_sample_plan([cams[i] for i in batch], n, 0, L.rng(3), lane)
        jac = scene.jacobian([cams[i] for i in batch], plan)
        P = 14 * scene.padded
        p = torch.empty(P, device="cuda").uniform_(-1, 1)
        u = torch.zeros(P, device="cuda")
        for _ in range(3):
            jac.gn_apply_dev(0.1, p.data_ptr(), u.data_ptr())
        L.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            jac.gn_apply_dev(0.1, p.data_ptr(), u.data_ptr())
        L.synchronize()
        prod_s = 10 / (time.perf_counter() - t0)
        del jac
        losses, t0 = [], time.perf_counter()
        for it in range(a.steps):
            rep = scene.lm_step(td, cfg, it, rng)
            losses.append(rep.loss_after)
        lm_s = a.steps / (time.perf_counter() - t0)
        print(json.dumps({"samples_per_tile": n, "ratio": round(n / 256, 3), "products_per_s": round(prod_s, 1),
                          "lm_iters_per_s": round(lm_s, 2), "loss_after": [round(x, 6) for x in losses]}), flush=True)


if __name__ == "__main__":
    main()
