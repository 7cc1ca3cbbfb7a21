"""Debug aid: heat IPM solve with the level-8 time-block hierarchies run whole
in the cluster kernel (cluster_top8=1) against the tiled level 8 + cluster
bottom (cluster_top8=0), same inputs.

    python tools/check_top8.py [nt=8]
"""
import dataclasses
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_05896_b200 import _lib, configs, optcon as oc  # noqa: E402

nt = int(sys.argv[1]) if len(sys.argv) > 1 else 8
c = dataclasses.replace(configs.C5, horizon=nt * configs.C5.tau)
lib = _lib.load()
ctx = oc.Context(0)
res = {}
for top8 in (0, 1):
    _lib.check(lib.oc_set_tuning(b"cluster_top8", top8))
    qp = oc.QpProblem(oc.ControlProblem(pde="heat", alpha=c.alpha, beta=c.beta, y_d=c.y_d(), u_a=c.u_a,
                                        u_b=c.u_b, tau=c.tau, horizon=c.horizon), oc.Grid(c.level), ctx)
    t0 = time.perf_counter()
    r = oc.ipm_solve(qp, oc.IpmParams(sigma=c.sigma, solver=c.solver))
    res[top8] = r
    print(f"top8={top8}: nt={nt} nli={r.stats.nli} lin={[i.lin_iters for i in r.stats.iterations[1:]]} "
          f"solve_ms={r.solve_ms:.1f} wall={time.perf_counter() - t0:.2f}s", flush=True)
a, b = res[0], res[1]
ru = np.linalg.norm(a.u - b.u) / np.linalg.norm(a.u)
ry = np.linalg.norm(a.state.y - b.state.y) / np.linalg.norm(a.state.y)
print(f"rel u {ru:.3e} rel y {ry:.3e} dJ {abs(a.objective - b.objective) / abs(a.objective):.3e}")
_lib.check(lib.oc_set_tuning(b"cluster_top8", 1))
