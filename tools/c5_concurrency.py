"""Throughput of R independent C5 solves in flight on one GPU (one context,
stream and host thread each; y_d seeds 42..42+R-1), R from the command line.

    python tools/c5_concurrency.py [--tune name=value] 1 2 4 8
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1806_05896_b200 import configs, optcon as oc, replicas  # noqa: E402

args = sys.argv[1:]
while args[:1] == ["--tune"]:  # --tune name=value (oc_set_tuning knob)
    from paper_1806_05896_b200 import _lib

    key, v = args[1].split("=")
    _lib.check(_lib.load().oc_set_tuning(key.encode(), int(v)))
    args = args[2:]
c = configs.C5
for R in [int(a) for a in args] or [1, 2, 4, 8]:
    ctxs = [oc.Context(0) for _ in range(R)]
    qps = []
    for i in range(R):
        yd = configs.sine_modes_spacetime(c.level, c.nt, c.tau, seed=42 + i)
        qps.append(oc.assemble_spacetime(oc.ControlProblem(pde="heat", tau=c.tau, alpha=c.alpha,
                                                           beta=c.beta, y_d=yd, u_a=c.u_a,
                                                           u_b=c.u_b), oc.Grid(c.level), ctxs[i]))
    params = oc.IpmParams(sigma=c.sigma, solver="minres-pd")

    def solve(i):
        return oc.ipm_solve(qps[i], params)

    replicas.run_concurrent(solve, range(R))  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = replicas.run_concurrent(solve, range(R))
    wall = time.perf_counter() - t0
    it = sum(r.total_lin for r in res.values())
    free, tot = torch.cuda.mem_get_info()
    print(f"R={R}: wall {wall:.2f} s, {it} Krylov its, {it / wall:.2f} it/s, per-solve ms "
          f"{[round(r.solve_ms) for r in res.values()]}, nli {[r.stats.nli for r in res.values()]}, "
          f"used {(tot - free) / 2**30:.1f} GiB", flush=True)
    for q in qps:
        q.close()
    for x in ctxs:
        x.close()
