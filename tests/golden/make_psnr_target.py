"""configs[0] reference run for the time-to-PSNR metric (TEST INFRASTRUCTURE).

    python tests/golden/make_psnr_target.py [--iterations 10] [--threads N]

Runs the UNMODIFIED reference (oracle/_ref, built from /root/reference by
`make -C oracle`) the way io::train_run does for the toy scene
(run.cpp:120-200): generate_toy_scene(5000 Gaussians, 8 train + 4 test views,
256x256, scene seed 20214), random_init(10000, [-1,1]^3, seed 1), k-means
clusters (seed 1 ^ 0x9e3779b97f4a7c15), then lm_step with batch 8, full pixels
(N = 256), PCG 8, and the test-split mean PSNR after every iteration
(evaluate_split, run.cpp:77-92).  Writes tests/golden/psnr_cfg0.json with the
per-iteration test PSNR, loss_after, eta and the CPU wall time per iteration.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.cpu_bind import ref  # noqa: E402
from paper_2504_12905_b200.types import LmConfig  # noqa: E402

KMEANS_SALT = 0x9E3779B97F4A7C15
CFG0 = dict(toy_gaussians=5000, train=8, test=4, size=256, scene_seed=20214, gaussians=10000, seed=1,
            batch=8, spt=256, pcg=8)


def run(lib, iterations, threads):
    c = CFG0
    if threads:
        lib.set_threads(threads)
    _, tc, ti, sc, si = lib.toy_scene(c["toy_gaussians"], c["train"], c["test"], c["size"], c["scene_seed"])
    rng = lib.rng(c["seed"])
    state = lib.random_init(c["gaussians"], [-1, -1, -1], [1, 1, 1], rng)
    td = lib.train_data(tc, list(ti))
    td.rebuild_clusters(min(c["batch"], len(tc)), c["seed"] ^ KMEANS_SALT)
    cfg = LmConfig(pcg_iters_initial=c["pcg"], pcg_iters_late=c["pcg"], batch_size_initial=c["batch"],
                   batch_size_late=c["batch"], samples_per_tile=c["spt"])
    out = dict(config=c, psnr=[], loss_after=[], eta=[], wall_s=[])
    for it in range(iterations):
        t0 = time.perf_counter()
        rep = lib.lm_step(state, td, cfg, it, rng)
        out["wall_s"].append(time.perf_counter() - t0)
        ps = [lib.psnr(lib.render_full(state, cam)[0], np.asarray(img, np.float64)) for cam, img in zip(sc, si)]
        out["psnr"].append(float(np.mean(ps)))
        out["loss_after"].append(rep.loss_after)
        out["eta"].append(rep.eta)
        print(f"iter {it}: loss_after {rep.loss_after:.6g} test psnr {out['psnr'][-1]:.4f} "
              f"({out['wall_s'][-1]:.1f} s)", flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iterations", type=int, default=10)
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    a = ap.parse_args()
    out = run(ref(), a.iterations, a.threads)
    out["threads"] = a.threads
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "psnr_cfg0.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
