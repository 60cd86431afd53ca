"""Per-parameter Jv of single blended Gaussians at one full-size pixel: ours vs the reference."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import oracle  # noqa: E402
from oracle.cpu_bind import port, ref  # noqa: E402
from paper_2504_12905_b200 import splatlm  # noqa: E402
from paper_2504_12905_b200.types import SamplePlan  # noqa: E402


def main():
    s_idx = int(sys.argv[1]) if len(sys.argv) > 1 else 108720
    gs = [int(a) for a in sys.argv[2:]] or [240279]
    lib = ref() if oracle.have_ref() else port()
    lib.set_threads(os.cpu_count() or 1)
    args = bench.parse_args_for(1_000_000)
    state, cams, clusters, batch, plan = bench.host_inputs(splatlm.HostSampler(), args, 1)
    cam = cams[batch[0]]
    x, y, tile = int(plan.px[s_idx]), int(plan.py[s_idx]), int(plan.tile[s_idx])
    one = SamplePlan(np.zeros(1, np.int32), np.array([0, 1], np.int64), np.array([x], np.int32),
                     np.array([y], np.int32), np.array([tile], np.int32), np.array([plan.weight[s_idx]]), 32)
    gpu = splatlm.lib()
    jr, jg = lib.jacobian(state, [cam], one), gpu.jacobian(state, [cam], one)
    print("cam", cam.world_to_cam.round(4), cam.translation.round(4), cam.fx, cam.fy, cam.cx, cam.cy)
    for g in gs:
        print("Gaussian", g, "params", state.pack()[14 * g:14 * g + 14].round(4))
        for comp in range(14):
            q = np.zeros(jr.param_dim())
            q[14 * g + comp] = 1.0
            ra, rb = jr.jvp(q), jg.jvp(q)
            rel = np.abs(ra - rb).max() / max(np.abs(ra).max(), 1e-30)
            print(f"  [{comp:2d}] ref {ra.round(7)} ours {rb.round(7)} rel {rel:.2e}")


if __name__ == "__main__":
    main()
