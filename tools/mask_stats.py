"""Blend-mask density and lane-balance statistics at the bench workload (GPU).

    python tools/mask_stats.py [--gaussians N] [--spt N]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gaussians", type=int, default=1_000_000)
    a = ap.parse_args()
    from paper_2504_12905_b200 import splatlm
    args = bench.parse_args_for(a.gaussians)
    L = splatlm.Lib(0)
    state, cams, clusters, batch, plan = bench.host_inputs(L, args, 1)
    scene = splatlm.Scene(L, state)
    jac = scene.jacobian([cams[i] for i in batch], plan)
    s = jac.mask_stats()
    s.update(jac.stats())
    w = s["windows"]
    s["pairs_per_window"] = s["pairs"] / w
    s["density"] = s["pairs"] / (32 * 32 * w)
    s["walk_lane_eff"] = s["pairs"] / (32 * s["it_walk"])
    s["walk64_lane_eff"] = s["pairs"] / (32 * s["it_walk64"])
    print(json.dumps(s, indent=1))


if __name__ == "__main__":
    main()
