"""KKT + preconditioner apply bandwidth per BASELINE config (north_star:
">= 60% of peak HBM at the 1025^2 and 257^2 x 128 sizes"). Solves each config
once (so Theta and the preconditioner are the final Newton step's), then times
one KKT apply and one preconditioner apply with CUDA events (oc_time_applies)
and divides the SURVEY §8d algorithmic bytes (bytes_model) by that time.

    python tools/apply_bw.py [--smoother lex] [C1 C2 C3 C4 C5]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_05896_b200 import _lib, bytes_model, configs, optcon as oc  # noqa: E402

KIND = {"gmres-pt": "pt", "minres-pd": "pd", "gmres-ppi": "ppi"}

args = sys.argv[1:]
smoother = "color4"
while args[:1] and args[0].startswith("--"):
    flag, val, args = args[0], args[1], args[2:]
    if flag == "--smoother":
        smoother = val
    elif flag == "--tune":  # name=value, any oc_set_tuning knob
        key, v = val.split("=")
        _lib.check(_lib.load().oc_set_tuning(key.encode(), int(v)))
    elif flag in ("--fuse", "--tile"):
        key = b"sweep_fuse" if flag == "--fuse" else b"sweep_tile"
        _lib.check(_lib.load().oc_set_tuning(key, int(val)))
names = args or ["C1", "C2", "C4", "C5", "C3"]
peak = None
try:
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json"))).get("hbm_gbs")
except Exception:
    pass
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
    qp = oc.QpProblem(oc.ControlProblem(**kw), oc.Grid(c.level), ctx)
    r = oc.ipm_solve(qp, oc.IpmParams(sigma=c.sigma, solver=c.solver,
                                      gmres_restart=c.gmres_restart, smoother=smoother))
    kind = KIND[c.solver]
    kkt_ms, prec_ms = qp.time_applies(kind, 5)
    ny = qp.ny
    kb, pb = bytes_model.apply_bytes(kind, c.level, ny, pde=c.pde, state_bounds=c.y_a is not None)
    gbs = (kb + pb) / ((kkt_ms + prec_ms) / 1e3) / 1e9
    print(json.dumps({"config": name, "smoother": smoother, "solve_ms": round(r.solve_ms, 1),
                      "kkt_ms": round(kkt_ms, 4), "prec_ms": round(prec_ms, 3),
                      "kkt_gbs": round(kb / (kkt_ms / 1e3) / 1e9, 1),
                      "prec_gbs": round(pb / (prec_ms / 1e3) / 1e9, 1),
                      "apply_gbs": round(gbs, 1),
                      "frac_of_peak": round(gbs / peak, 4) if peak else None,
                      "peak_gbs": peak, "bytes_per_apply": kb + pb}), flush=True)
    qp.close()
