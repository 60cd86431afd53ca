"""Full-size (configs[2], 1 view) product errors vs the reference: jvp, vjp, gn_apply, diag."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import bench  # noqa: E402
import oracle  # noqa: E402
from oracle.cpu_bind import port, ref  # noqa: E402
from paper_2504_12905_b200 import splatlm  # noqa: E402


def nr(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    views = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    lib = ref() if oracle.have_ref() else port()
    lib.set_threads(os.cpu_count() or 1)
    args = bench.parse_args_for(1_000_000)
    state, cams, clusters, batch, plan = bench.host_inputs(splatlm.HostSampler(), args, 1)
    cams = [cams[i] for i in batch[:views]]
    plan = bench.sub_plan(plan, 0, views)
    g = splatlm.lib()
    jr, jg = lib.jacobian(state, cams, plan), g.jacobian(state, cams, plan)
    r = np.random.default_rng(0)
    p = r.uniform(-1, 1, jr.param_dim())
    u = r.uniform(-1, 1, jr.residual_dim())
    a, b = jg.jvp(p), jr.jvp(p)
    print("jvp", nr(a, b), "vjp", nr(jg.vjp(u), jr.vjp(u)), "gn", nr(jg.gn_apply(0.1, p), jr.gn_apply(0.1, p)),
          "diag", nr(jg.jtj_diag(), jr.jtj_diag()))
    d = np.abs(a - b)
    i = np.argsort(-d)[:5]
    print("largest jvp residual diffs", list(zip(i.tolist(), a[i].round(5).tolist(), b[i].round(5).tolist())))


if __name__ == "__main__":
    main()
