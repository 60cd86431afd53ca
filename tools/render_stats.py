"""k_render work counters at configs[2] (8 batch views, random_init state and the
LM ground truth scene): how much of the per-tile list the warps walk."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    from paper_2504_12905_b200 import splatlm
    from paper_2504_12905_b200.types import cameras_to_c
    args = bench.parse_args_for(1_000_000)
    L = splatlm.Lib(0)
    state, cams, clusters, batch, plan = bench.host_inputs(L, args, 1)
    bc = [cams[i] for i in batch]
    for name, g in (("random_init", state), ("gt_scene", bench.gt_scene(args.gaussians // 2, H=L))):
        sc = splatlm.Scene(L, g)
        out = np.zeros(10, np.uint64)
        rc = L.dll.slm_debug_render_stats(sc.h, cameras_to_c(bc), len(bc), out.ctypes.data_as(C.POINTER(C.c_uint64)))
        assert rc == 0, L.dll.slm_last_error()
        it, box, live, blend, staged, E, npix, nt, exact, useful = [int(x) for x in out]
        # per thread counters: 64 threads per tile
        print(f"{name}: entries {E} ({E / nt:.0f}/tile), staged/tile {staged / 64 / nt:.0f}, "
              f"iterated/warp {it / 64 / (2 * nt):.0f}... thread-iter {it / (64 * nt):.0f}, box-pass {box / (64 * nt):.0f}, "
              f"live gates/px {live / npix:.0f}, blends/px {blend / npix:.0f}, "
              f"warp-entries: box {box / 32:.0f}, exact {exact:.0f}, useful {useful:.0f}")


if __name__ == "__main__":
    main()
