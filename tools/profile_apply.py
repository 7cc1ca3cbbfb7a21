"""Workload for ncu launch lists of ONE KKT + preconditioner apply at a
BASELINE config: one Newton step to set the preconditioner up, then
oc_time_applies (warm-ups + `reps` timed applies).

    python tools/profile_apply.py C4 [reps=1] [smoother=color4]

A config name may carry a level, e.g. C3@8.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_05896_b200 import configs, optcon as oc  # noqa: E402

KIND = {"gmres-pt": "pt", "minres-pd": "pd", "gmres-ppi": "ppi"}
args = sys.argv[1:]
while args[:1] and args[0] == "--tune":  # --tune name=value (oc_set_tuning knob)
    from paper_1806_05896_b200 import _lib

    key, v = args[1].split("=")
    _lib.check(_lib.load().oc_set_tuning(key.encode(), int(v)))
    args = args[2:]
sys.argv = sys.argv[:1] + args
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
smoother = sys.argv[3] if len(sys.argv) > 3 else "color4"
base, _, lvl = name.partition("@")
c = configs.ALL[base].with_level(int(lvl)) if lvl else configs.ALL[base]
kw = dict(pde=c.pde, alpha=c.alpha, beta=c.beta, y_d=c.y_d(), u_a=c.u_a, u_b=c.u_b)
if c.pde == "convdiff":
    kw["eps"] = c.eps
if c.pde == "heat":
    kw["tau"] = c.tau
if c.y_a is not None:
    kw.update(y_a=c.y_a, y_b=c.y_b)
if c.obs is not None:
    kw["observation"] = c.obs
ctx = oc.Context(0)
qp = oc.QpProblem(oc.ControlProblem(**kw), oc.Grid(c.level), ctx)
try:
    oc.ipm_solve(qp, oc.IpmParams(sigma=c.sigma, solver=c.solver, max_iterations=1,
                                  gmres_restart=c.gmres_restart, smoother=smoother))
except Exception as e:  # one IPM iteration does not converge: expected
    print("solve:", type(e).__name__, e)
print("MARK apply start", flush=True)
k, p = qp.time_applies(KIND[c.solver], reps)
print(f"{name}: kkt {k:.4f} ms, precond {p:.3f} ms")
