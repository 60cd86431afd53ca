"""Products of two fixed cases (the fused-chain path at 200k Gaussians / 4 views,
and the record-parallel k_det_reduce path on the toy scene) saved to an .npz, to
compare two library builds bitwise:  SLM_LIB=a.so python tools/bitwise_ab.py a.npz"""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(out):
    from paper_2504_12905_b200 import splatlm
    from paper_2504_12905_b200.types import ring_camera
    L = splatlm.lib()
    L.set_deterministic(True)
    H = splatlm.HostSampler()
    res = {}
    for name, (G, nv, w, h, spt) in {"big": (200_000, 4, 640, 480, 32), "toy": (400, 4, 96, 96, 32)}.items():
        rng = H.rng(3)
        st = H.random_init(G, [-1, -1, -1], [1, 1, 1], rng)
        cams = [ring_camera(2.0 * math.pi * i / nv, 3.2, 1.1, w, h) for i in range(nv)]
        plan = H.build_sample_plan(cams, spt, 0, rng, 32)
        jac = L.jacobian(st, cams, plan)
        r = np.random.default_rng(0)
        p = r.uniform(-1, 1, jac.param_dim())
        u = r.uniform(-1, 1, jac.residual_dim())
        res[name + "_gn"] = jac.gn_apply(0.1, p)
        res[name + "_vjp"] = jac.vjp(u)
        res[name + "_diag"] = jac.jtj_diag()
        res[name + "_jvp"] = jac.jvp(p)
    np.savez(out, **res)


if __name__ == "__main__":
    if len(sys.argv) > 2:
        a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
        for k in a.files:
            print(k, "bitwise equal" if np.array_equal(a[k], b[k]) else f"DIFF max {np.max(np.abs(a[k] - b[k]))}")
    else:
        main(sys.argv[1])
