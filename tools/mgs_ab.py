"""Same-box A/B of the GMRES orthogonalisation paths on C3 (full solve, twice
each, alternating): mgs_persistent = 0 (launch per step) vs 8 (default).

    python tools/mgs_ab.py [level]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_1806_05896_b200 import _lib, configs, optcon as oc  # noqa: E402
from parity_full import problem_kwargs  # noqa: E402

lvl = int(sys.argv[1]) if len(sys.argv) > 1 else 10
c = configs.ALL["C3"].with_level(lvl)
kw = problem_kwargs(c)
kw["pde"] = c.pde
kw["observation"] = c.obs
ctx = oc.Context(0)
L = _lib.load()
res = {}
for rep in range(2):
    for knob in (0, 8):
        _lib.check(L.oc_set_tuning(b"mgs_persistent", knob))
        qp = oc.QpProblem(oc.ControlProblem(**kw), oc.Grid(c.level), ctx)
        r = oc.ipm_solve(qp, oc.IpmParams(sigma=c.sigma, solver=c.solver))
        res.setdefault(knob, []).append((r.solve_ms, r.u.copy()))
        qp.close()
        print(f"mgs_persistent={knob}: {r.solve_ms / 1e3:.2f} s, av_li {r.stats.av_li:.3f}", flush=True)
_lib.check(L.oc_set_tuning(b"mgs_persistent", 8))
print("bitwise equal:", all(np.array_equal(res[0][0][1], u) for _, u in res[0] + res[8]))
