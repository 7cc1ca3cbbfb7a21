"""Workload for an ncu launch list of the persistent GMRES orthogonalisation:
the first Newton step of C3 (one capped 200-iteration GMRES solve).

    python tools/mgs_probe.py [level]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_1806_05896_b200 import configs, optcon as oc  # noqa: E402
from parity_full import problem_kwargs  # noqa: E402

lvl = int(sys.argv[1]) if len(sys.argv) > 1 else 10
c = configs.ALL["C3"].with_level(lvl)
kw = problem_kwargs(c)
kw["pde"] = c.pde
kw["observation"] = c.obs
ctx = oc.Context(0)
qp = oc.QpProblem(oc.ControlProblem(**kw), oc.Grid(c.level), ctx)
r = oc.ipm_solve(qp, oc.IpmParams(sigma=c.sigma, solver=c.solver, max_iterations=1))
print("newton steps", r.stats.nli)
