"""Device solve of one BASELINE config (optionally at another level / with the
lexicographic smoother) saved for a later comparison with a reference run
(tools/compare_saved.py --device), e.g. when the reference needs hours.

    python tools/device_solve_save.py C3 out.npz [level] [smoother]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_1806_05896_b200 import configs, optcon as oc  # noqa: E402
from parity_full import problem_kwargs  # noqa: E402

name, out = sys.argv[1], sys.argv[2]
c = configs.ALL[name]
if len(sys.argv) > 3:
    c = c.with_level(int(sys.argv[3]))
smoother = sys.argv[4] if len(sys.argv) > 4 else "color4"
kw = problem_kwargs(c)
kw["pde"] = c.pde
if c.obs is not None:
    kw["observation"] = c.obs
ctx = oc.Context(0)
qp = oc.QpProblem(oc.ControlProblem(**kw), oc.Grid(c.level), ctx)
r = oc.ipm_solve(qp, oc.IpmParams(sigma=c.sigma, solver=c.solver, gmres_restart=c.gmres_restart,
                                  smoother=smoother))
np.savez(out, u=r.u, y=r.state.y, z=r.state.z, objective=r.objective, nli=r.stats.nli,
         av_li=r.stats.av_li, lin=np.array([i.lin_iters for i in r.stats.iterations[1:]]),
         lin_converged=all(i.lin_converged for i in r.stats.iterations[1:]), ms=r.solve_ms,
         level=c.level, smoother=smoother)
print(f"{name} level {c.level} {smoother}: nli {r.stats.nli} av_li {r.stats.av_li:.3f} "
      f"J {r.objective:.15g} in {r.solve_ms / 1e3:.1f} s")
