"""C3 (capped GMRES, default auto smoother -> lexicographic fallback) with the
pipelined lexicographic batches off and on: bitwise comparison of u, y, Krylov
counts and the solve times.

    python tools/lex_pipe_c3.py [level=8]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_05896_b200 import _lib, configs, optcon as oc  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 8
c = configs.C3.with_level(level)
lib = _lib.load()
ctx = oc.Context(0)
res = {}
for v in ([int(a) for a in sys.argv[2:]] or [0, 1]):
    _lib.check(lib.oc_set_tuning(b"lex_pipeline", v))
    qp = oc.QpProblem(oc.ControlProblem(pde=c.pde, alpha=c.alpha, beta=c.beta, y_d=c.y_d(), u_a=c.u_a,
                                        u_b=c.u_b, y_a=c.y_a, y_b=c.y_b, observation=c.obs),
                      oc.Grid(c.level), ctx)
    r = oc.ipm_solve(qp, oc.IpmParams(sigma=c.sigma, solver=c.solver))
    res[v] = r
    print(f"lex_pipeline {v}: solve {r.solve_ms / 1e3:.2f} s, nli {r.stats.nli}, lin "
          f"{[i.lin_iters for i in r.stats.iterations[1:]]}, J {r.objective!r}", flush=True)
    qp.close()
if len(res) == 2:
    a, b = res[0], res[1]
    print("u bitwise", np.array_equal(a.u, b.u), "y bitwise", np.array_equal(a.state.y, b.state.y))
