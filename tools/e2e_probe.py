"""Wall time of the host-vector gn_apply (the e2e path) at configs[2], per call."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    import torch
    from paper_2504_12905_b200 import splatlm
    args = bench.parse_args_for(1_000_000)
    L = splatlm.Lib(0)
    state, cams, clusters, batch, plan = bench.host_inputs(L, args, 1)
    jac = L.jacobian(state, [cams[i] for i in batch], plan)
    n = jac.param_dim()
    ph = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    ph[:] = np.random.default_rng(0).uniform(-1, 1, n)
    oh = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    for pinned in (True, False):
        pv = ph if pinned else ph.copy()
        ov = oh if pinned else oh.copy()
        jac.gn_apply(0.1, pv, out=ov)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            jac.gn_apply(0.1, pv, out=ov)
            ts.append(1000 * (time.perf_counter() - t0))
        print(f"pipeline={os.environ.get('SLM_HOST_PIPELINE', '1')} pinned={pinned}: ms {[round(t, 2) for t in ts]}")


if __name__ == "__main__":
    main()
