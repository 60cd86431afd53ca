"""configs[0] (toy scene, 10k Gaussians, 8 x 256^2, N=256, PCG 8): per-step wall
time and CUDA-event stage timings of lm_step, ordered vs atomic accumulation."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2504_12905_b200 import splatlm  # noqa: E402


def run(L, det: bool, timing: bool):
    ref = json.load(open(bench.PSNR_TARGET))
    c = ref["config"]
    train, timgs, test, simgs = bench.cfg0_scene(L, c)
    td = L.train_data(train, timgs)
    td.set_clusters(L.kmeans_cameras(train, c["batch"], c["seed"] ^ bench.KMEANS_SALT))
    rng = L.rng(c["seed"])
    scene = splatlm.Scene(L, L.random_init(c["gaussians"], [-1, -1, -1], [1, 1, 1], rng))
    cfg = bench.LmConfig(pcg_iters_initial=8, pcg_iters_late=8, batch_size_initial=8, batch_size_late=8,
                         samples_per_tile=256)
    L.set_deterministic(det)
    L.set_timing(timing)
    walls = []
    for it in range(10):
        L.synchronize()
        t0 = time.perf_counter()
        scene.lm_step(td, cfg, it, rng)
        L.synchronize()
        walls.append(1000 * (time.perf_counter() - t0))
        if timing and it == 5:
            print("  stages", L.timings())
    print(f"det={det} timing={timing}: step ms {[round(w, 2) for w in walls]} total {sum(walls):.1f}")


if __name__ == "__main__":
    L = splatlm.Lib(0)
    for det in (True, False):
        run(L, det, False)
        run(L, det, True)
