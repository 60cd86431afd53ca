"""Diagnose the largest full-size jvp differences: per-pixel contrib / T, ours vs the reference."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import oracle  # noqa: E402
from oracle.cpu_bind import port, ref  # noqa: E402
from paper_2504_12905_b200 import splatlm  # noqa: E402


def main():
    lib = ref() if oracle.have_ref() else port()
    lib.set_threads(os.cpu_count() or 1)
    args = bench.parse_args_for(1_000_000)
    state, cams, clusters, batch, plan = bench.host_inputs(splatlm.HostSampler(), args, 1)
    cam = cams[batch[0]]
    plan = bench.sub_plan(plan, 0, 1)
    g = splatlm.lib()
    jr, jg = lib.jacobian(state, [cam], plan), g.jacobian(state, [cam], plan)
    p = np.random.default_rng(0).uniform(-1, 1, jr.param_dim())
    a, b = jg.jvp(p), jr.jvp(p)
    d = np.abs(a - b).reshape(-1, 3).max(axis=1)
    print("samples", d.size, "diff>1e-2:", int((d > 1e-2).sum()), "diff>1e-1:", int((d > 1e-1).sum()),
          "diff>1e-3:", int((d > 1e-3).sum()))
    img_r, tr_r, cn_r = lib.render_full(state, cam)
    img_g, tr_g, cn_g = g.render_full(state, cam)
    print("render max |dimg|", float(np.abs(img_r - img_g).max()), "contrib mismatches",
          int((cn_r != cn_g).sum()), "of", cn_r.size)
    for s in np.argsort(-d)[:6]:
        x, y = int(plan.px[s]), int(plan.py[s])
        print(f"sample {s} px ({x},{y}) diff {d[s]:.4f} contrib ref {cn_r[y, x]} ours {cn_g[y, x]} "
              f"T ref {tr_r[y, x]:.3e} ours {tr_g[y, x]:.3e} jvp ref {b[3*s:3*s+3].round(4)} ours {a[3*s:3*s+3].round(4)}")


if __name__ == "__main__":
    main()
