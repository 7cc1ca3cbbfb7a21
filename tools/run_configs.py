"""Run the BASELINE configs C1..C5 at full size on the device and print
time-to-tolerance and iteration statistics (one JSON line per config).

    python tools/run_configs.py [--smoother lex] [C1 C2 C3 C4 C5]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_05896_b200 import _lib, configs, optcon as oc  # noqa: E402

args = sys.argv[1:]
smoother = "color4"
solver = None
while args[:1] and args[0].startswith("--"):
    flag, val, args = args[0], args[1], args[2:]
    if flag == "--smoother":
        smoother = val
    elif flag == "--solver":
        solver = val
    elif flag == "--tune":  # name=value, any oc_set_tuning knob
        key, v = val.split("=")
        _lib.check(_lib.load().oc_set_tuning(key.encode(), int(v)))
    elif flag in ("--fuse", "--tile"):
        key = b"sweep_fuse" if flag == "--fuse" else b"sweep_tile"
        _lib.check(_lib.load().oc_set_tuning(key, int(val)))
names = args or ["C1", "C2", "C3", "C4", "C5"]
ctx = oc.Context(0)
for name in names:
    c = configs.ALL[name]
    kw = dict(pde=c.pde, alpha=c.alpha, beta=c.beta, y_d=c.y_d(), u_a=c.u_a, u_b=c.u_b)
    if c.pde == "convdiff":
        kw["eps"] = c.eps
    if c.pde == "heat":
        kw["tau"] = c.tau
    if c.y_a is not None:
        kw.update(y_a=c.y_a, y_b=c.y_b)
    if c.obs is not None:
        kw["observation"] = c.obs
    t0 = time.perf_counter()
    qp = oc.QpProblem(oc.ControlProblem(**kw), oc.Grid(c.level), ctx)
    t_setup = time.perf_counter() - t0
    params = oc.IpmParams(sigma=c.sigma, solver=solver or c.solver, gmres_restart=c.gmres_restart,
                          smoother=smoother)
    t0 = time.perf_counter()
    try:
        r = oc.ipm_solve(qp, params)
    except Exception as e:  # report and continue
        print(json.dumps({"config": name, "error": f"{type(e).__name__}: {e}"}), flush=True)
        continue
    wall = time.perf_counter() - t0
    print(json.dumps({
        "config": name, "level": c.level, "solver": solver or c.solver, "smoother": smoother, "setup_s": round(t_setup, 3),
        "solve_ms": round(r.solve_ms, 2), "wall_s": round(wall, 3), "nli": r.stats.nli,
        "av_li": round(r.stats.av_li, 3), "converged": r.stats.converged,
        "lin_iters": [i.lin_iters for i in r.stats.iterations[1:]],
        "lin_converged": all(i.lin_converged for i in r.stats.iterations[1:]),
        "objective": r.objective, "zeros": int((np.abs(r.u) < 1e-2).sum()),
        "krylov_its_per_s": round(r.total_lin / (r.solve_ms / 1e3), 2),
    }), flush=True)
