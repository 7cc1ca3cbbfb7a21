"""Debug aid: IPM solves (C2, C4, C5 with 4 time blocks) with a tuning knob
off and on: the solutions should be bitwise equal; prints the P apply times.

    python tools/check_knob.py cheb_block
"""
import os, sys
knob = sys.argv[1].encode() if len(sys.argv) > 1 else b"cheb_block"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1806_05896_b200 import _lib, configs, optcon as oc
lib = _lib.load(); ctx = oc.Context(0)
for name in ("C2", "C4", "C5"):
    c = configs.ALL[name]
    if name == "C5":
        import dataclasses
        c = dataclasses.replace(c, horizon=4 * c.tau)
    res = {}
    for v in (0, 1):
        _lib.check(lib.oc_set_tuning(knob, v))
        kw = dict(pde=c.pde, alpha=c.alpha, beta=c.beta, y_d=c.y_d(), u_a=c.u_a, u_b=c.u_b)
        if c.pde == "convdiff": kw["eps"] = c.eps
        if c.pde == "heat": kw.update(tau=c.tau, horizon=c.horizon)
        qp = oc.QpProblem(oc.ControlProblem(**kw), oc.Grid(c.level), ctx)
        r = oc.ipm_solve(qp, oc.IpmParams(sigma=c.sigma, solver=c.solver, gmres_restart=c.gmres_restart))
        k, p = qp.time_applies("pt", 20)
        res[v] = (r, p)
    print(name, "max|du|", float(np.abs(res[0][0].u - res[1][0].u).max()), "prec_ms off/on", round(res[0][1], 4), round(res[1][1], 4), flush=True)
