"""Launch-list workload for ONE KKT + preconditioner apply in a chosen smoother
mode, cheap to set up: one IPM iteration with linear_maxit=2 builds the
preconditioner, then the apply runs between cudaProfilerStart/Stop (use
`ncu --profile-from-start off`).

    python tools/profile_lex.py C3 [smoother=lex] [reps=1] [solver]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_05896_b200 import configs, optcon as oc  # noqa: E402

KIND = {"gmres-pt": "pt", "minres-pd": "pd", "gmres-ppi": "ppi"}
args = sys.argv[1:]
while args[:1] == ["--tune"]:  # --tune name=value (oc_set_tuning knob)
    from paper_1806_05896_b200 import _lib

    key, v = args[1].split("=")
    _lib.check(_lib.load().oc_set_tuning(key.encode(), int(v)))
    args = args[2:]
sys.argv = sys.argv[:1] + args
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
smoother = sys.argv[2] if len(sys.argv) > 2 else "lex"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
base, _, lvl = name.partition("@")
c = configs.ALL[base].with_level(int(lvl)) if lvl else configs.ALL[base]
if len(sys.argv) > 4:
    c = c.with_level(c.level, solver=sys.argv[4])
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
    oc.ipm_solve(qp, oc.IpmParams(sigma=c.sigma, solver=c.solver, max_iterations=1, linear_maxit=2,
                                  gmres_restart=c.gmres_restart, smoother=smoother))
except Exception as e:  # one IPM iteration does not converge: expected
    print("solve:", type(e).__name__, e)
qp.time_applies(KIND[c.solver], 2)  # warm (graph capture)
import torch  # noqa: E402

torch.cuda.profiler.start()
k, p = qp.time_applies(KIND[c.solver], reps)
torch.cuda.profiler.stop()
print(f"{name} {smoother}: kkt {k:.4f} ms, precond {p:.3f} ms")
