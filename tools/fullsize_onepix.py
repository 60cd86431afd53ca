"""Isolate one full-size pixel whose Jv differs: blended set (FP64 replay of blend_pixel
from the reference's own prepare + tile list) and per-Gaussian Jv contributions."""
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
    lib = ref() if oracle.have_ref() else port()
    lib.set_threads(os.cpu_count() or 1)
    args = bench.parse_args_for(1_000_000)
    state, cams, clusters, batch, plan = bench.host_inputs(splatlm.HostSampler(), args, 1)
    cam = cams[batch[0]]
    x, y = int(plan.px[s_idx]), int(plan.py[s_idx])
    tile = int(plan.tile[s_idx])
    one = SamplePlan(np.zeros(1, np.int32), np.array([0, 1], np.int64), np.array([x], np.int32),
                     np.array([y], np.int32), np.array([tile], np.int32), np.array([plan.weight[s_idx]]), 32)
    pr = lib.prepare(state, cam)
    off, idx = lib.bin_and_sort(state, cam)
    lst = idx[off[tile]:off[tile + 1]]
    T, blended = 1.0, []
    for g in lst:
        mx, my = pr["mean2d"][2 * g], pr["mean2d"][2 * g + 1]
        a, b, c = pr["conic"][3 * g:3 * g + 3]
        dx, dy = mx - (x + 0.5), my - (y + 0.5)
        power = -0.5 * (a * dx * dx + c * dy * dy) - b * dx * dy
        if power > 0:
            continue
        al = min(pr["opacity"][g] * np.exp(power), 0.99)
        if al < 1 / 255:
            continue
        if T * (1 - al) < 1e-4:
            break
        blended.append((int(g), al, T))
        T *= 1 - al
    print(f"sample {s_idx} px ({x},{y}) tile {tile}: list {len(lst)}, blended {len(blended)}, T_end {T:.4e}")
    gpu = splatlm.lib()
    jr, jg = lib.jacobian(state, [cam], one), gpu.jacobian(state, [cam], one)
    p = np.random.default_rng(0).uniform(-1, 1, jr.param_dim())
    print("full p: jvp ref", jr.jvp(p).round(5), "ours", jg.jvp(p).round(5))
    # bisect the blended Gaussians' parameter blocks for the differing contribution
    groups = [g for g, _, _ in blended]
    def jv(mask_g):
        q = np.zeros_like(p)
        for g in mask_g:
            q[14 * g:14 * g + 14] = p[14 * g:14 * g + 14]
        return jr.jvp(q), jg.jvp(q)
    cand = groups
    while len(cand) > 1:
        half = cand[:len(cand) // 2]
        a, b = jv(half)
        if np.abs(a - b).max() > 1e-3:
            cand = half
        else:
            cand = cand[len(cand) // 2:]
    g = cand[0]
    a, b = jv([g])
    k = [i for i, (gg, _, _) in enumerate(blended) if gg == g][0]
    print(f"culprit Gaussian {g} (blend position {k}, alpha {blended[k][1]:.6f}, T {blended[k][2]:.4e}): "
          f"ref {a.round(6)} ours {b.round(6)}")
    print("its params", state.pack()[14 * g:14 * g + 14].round(5), "conic", pr["conic"][3 * g:3 * g + 3],
          "mean2d", pr["mean2d"][2 * g:2 * g + 2], "radius", pr["radius"][g])
    for comp in range(14):
        q = np.zeros_like(p)
        q[14 * g + comp] = 1.0
        ra, rb = jr.jvp(q), jg.jvp(q)
        if np.abs(ra - rb).max() > 1e-4 * max(1, np.abs(ra).max()):
            print(f"  d/dparam[{comp}]: ref {ra.round(6)} ours {rb.round(6)}")


if __name__ == "__main__":
    main()
