"""In-situ spans of a C5 step with R solves in flight: CUDA-event time of the
KKT applies, the P_D applies and the chained block solves on each replica's
stream, against the per-solve device time (where a Krylov iteration's time goes
when the GPU is shared).

    python tools/c5_insitu.py [--tune name=value] [R=8]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401

from paper_1806_05896_b200 import configs, optcon as oc, replicas  # noqa: E402

args = sys.argv[1:]
while args[:1] == ["--tune"]:
    from paper_1806_05896_b200 import _lib

    key, v = args[1].split("=")
    _lib.check(_lib.load().oc_set_tuning(key.encode(), int(v)))
    args = args[2:]
R = int(args[0]) if args else 8
c = configs.C5
ctxs = [oc.Context(0) for _ in range(R)]
qps = []
for i in range(R):
    yd = configs.sine_modes_spacetime(c.level, c.nt, c.tau, seed=42 + i)
    qps.append(oc.assemble_spacetime(oc.ControlProblem(pde="heat", tau=c.tau, alpha=c.alpha, beta=c.beta,
                                                       y_d=yd, u_a=c.u_a, u_b=c.u_b), oc.Grid(c.level), ctxs[i]))
params = oc.IpmParams(sigma=c.sigma, solver="minres-pd")


def solve(i):
    return oc.ipm_solve(qps[i], params)


replicas.run_concurrent(solve, range(R))  # warm
for cx in ctxs:
    cx.profile(True)
res = replicas.run_concurrent(solve, range(R))
for i, cx in enumerate(ctxs):
    pr = cx.profile_read()
    cx.profile(False)
    r = res[i]
    its = r.total_lin
    print(f"replica {i}: solve {r.solve_ms:8.1f} ms, {its} its -> {r.solve_ms / its:6.1f} ms/it | "
          f"kkt {pr['kkt'][0] / max(pr['kkt'][1], 1):6.3f} ms x {pr['kkt'][1]} | "
          f"prec {pr['prec'][0] / max(pr['prec'][1], 1):7.2f} ms x {pr['prec'][1]} | "
          f"chain {pr['block'][0] / max(pr['block'][1], 1):7.2f} ms x {pr['block'][1]}", flush=True)
