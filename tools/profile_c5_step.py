"""Workload for an ncu launch list of whole C5 Newton steps (preconditioner
setup + Krylov solve), on a shortened horizon: `nt` time blocks, `its` IPM
iterations.

    python tools/profile_c5_step.py [nt=16] [its=2] [solver=minres-pd]
"""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_05896_b200 import configs, optcon as oc  # noqa: E402

nt = int(sys.argv[1]) if len(sys.argv) > 1 else 16
its = int(sys.argv[2]) if len(sys.argv) > 2 else 2
solver = sys.argv[3] if len(sys.argv) > 3 else "minres-pd"
c = dataclasses.replace(configs.ALL["C5"], horizon=nt * configs.ALL["C5"].tau)
ctx = oc.Context(0)
qp = oc.QpProblem(oc.ControlProblem(pde="heat", alpha=c.alpha, beta=c.beta, y_d=c.y_d(), u_a=c.u_a,
                                    u_b=c.u_b, tau=c.tau, horizon=c.horizon), oc.Grid(c.level), ctx)
r = oc.ipm_solve(qp, oc.IpmParams(sigma=c.sigma, solver=solver, max_iterations=its))
print("nli", r.stats.nli, "lin", list(r.stats.lin_iters) if hasattr(r.stats, "lin_iters") else r.stats.av_li,
      "device_ms", round(r.solve_ms, 2), flush=True)
