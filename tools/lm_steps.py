"""Per-step wall times and stage timings of lm_step at the bench workload (GPU)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2504_12905_b200 import splatlm  # noqa: E402
from paper_2504_12905_b200.types import LmConfig  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    dist = int(sys.argv[2]) if len(sys.argv) > 2 else 0   # residual distribution
    loss = int(sys.argv[3]) if len(sys.argv) > 3 else 0   # 1 = mse+ssim
    args = bench.parse_args_for(1_000_000)
    L = splatlm.Lib(0)
    state, cams, clusters, batch, plan = bench.host_inputs(L, args, 1)
    gt = splatlm.Scene(L, bench.gt_scene(args.gaussians // 2, H=L))
    imgs = [gt.render(c)[0] for c in cams]
    del gt
    td = L.train_data(cams, imgs)
    td.set_clusters(clusters)
    scene = splatlm.Scene(L, state)
    cfg = LmConfig(pcg_iters_initial=8, pcg_iters_late=8, batch_size_initial=8, batch_size_late=8, samples_per_tile=32,
                   dist=dist, loss=loss)
    rng = L.rng(1)
    L.random_init(args.gaussians, [-1, -1, -1], [1, 1, 1], rng)
    L.set_timing(True)
    for i in range(n):
        t0 = time.perf_counter()
        scene.lm_step(td, cfg, i, rng)
        dt = (time.perf_counter() - t0) * 1000
        tm = L.timings()
        print(f"step {i}: wall {dt:.1f} ms, marks sum {sum(tm.values()):.1f} ms: {tm}", flush=True)


if __name__ == "__main__":
    main()
