"""A/B of two builds of the library on the same box: for each config solves the
IPM, times the KKT + preconditioner applies (oc_time_applies) and saves u, so
two runs (OPTCON_B200_LIB=<other .so>) can be compared bit for bit.

    python tools/ab_lib.py out.npz [C2 C3 C4 ...]
    OPTCON_B200_LIB=.../liboptcon_b200_base.so python tools/ab_lib.py base.npz ...
    python tools/ab_lib.py --diff out.npz base.npz
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if sys.argv[1] == "--diff":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    for k in a.files:
        if k in b.files:
            d = float(np.abs(a[k] - b[k]).max()) if a[k].shape == b[k].shape else float("nan")
            print(k, "max|diff|", d, "bitwise" if d == 0.0 else "")
    sys.exit(0)

from paper_1806_05896_b200 import _lib, bytes_model, configs, optcon as oc  # noqa: E402

KIND = {"gmres-pt": "pt", "minres-pd": "pd", "gmres-ppi": "ppi"}
out = sys.argv[1]
names = sys.argv[2:] or ["C2", "C4", "C3"]
ctx = oc.Context(0)
save = {}
for name in names:
    import dataclasses
    c = configs.ALL[name.split("@")[0]]
    if "@" in name:  # C5@8: 8 time blocks
        c = dataclasses.replace(c, horizon=int(name.split("@")[1]) * c.tau)
    kw = dict(pde=c.pde, alpha=c.alpha, beta=c.beta, y_d=c.y_d(), u_a=c.u_a, u_b=c.u_b)
    if c.pde == "convdiff":
        kw["eps"] = c.eps
    if c.pde == "heat":
        kw.update(tau=c.tau, horizon=c.horizon)
    if c.y_a is not None:
        kw.update(y_a=c.y_a, y_b=c.y_b)
    if c.obs is not None:
        kw["observation"] = c.obs
    qp = oc.QpProblem(oc.ControlProblem(**kw), oc.Grid(c.level), ctx)
    r = oc.ipm_solve(qp, oc.IpmParams(sigma=c.sigma, solver=c.solver, gmres_restart=c.gmres_restart,
                                      smoother="color4"))
    kind = KIND[c.solver]
    kkt_ms, prec_ms = qp.time_applies(kind, 20)
    kb, pb = bytes_model.apply_bytes(kind, c.level, qp.ny, pde=c.pde, state_bounds=c.y_a is not None)
    print(json.dumps({"config": name, "lib": os.path.basename(_lib.LIB_PATH), "solve_ms": round(r.solve_ms, 1),
                      "nli": r.stats.nli, "av_li": round(r.stats.av_li, 3), "kkt_ms": round(kkt_ms, 4),
                      "prec_ms": round(prec_ms, 4),
                      "gbs": round((kb + pb) / ((kkt_ms + prec_ms) / 1e3) / 1e9, 1)}), flush=True)
    save[name + "_u"] = r.u
    save[name + "_y"] = r.state.y
    qp.close()
np.savez(out, **save)
