"""How the C2 sweep scales with the number of cells in flight on one GPU: k cells
(each its own context/stream and host thread, as in bench.py) solved
concurrently, k = 1, 2, 3, 5, 9. Prints device step ms, wall ms, host CPU
seconds used by the process during the step and Krylov it/s.

    python tools/concurrency.py [--level 9] [--reps 3]
"""
import argparse
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_05896_b200 import configs, optcon as oc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--level", type=int, default=9)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--ks", default="1,2,3,5,9")
a = ap.parse_args()

print(f"host cpus: {os.cpu_count()}, affinity {len(os.sched_getaffinity(0))}", flush=True)
cells = [c.with_level(a.level) for c in configs.C2_CELLS]
params = oc.IpmParams(sigma=0.2, solver="gmres-pt")
grid = oc.Grid(a.level)
ctxs = [oc.Context(0) for _ in cells]
probs = [oc.build_qp(oc.ControlProblem(alpha=c.alpha, beta=c.beta, y_d=c.y_d(), u_a=c.u_a, u_b=c.u_b),
                     grid, cx) for c, cx in zip(cells, ctxs)]


def run(k):
    res = [None] * k

    def body(i):
        res[i] = oc.ipm_solve(probs[i], params)
        ctxs[i].record(1)

    for cx in ctxs[:k]:
        cx.synchronize()
        cx.record(0)
    t0, c0 = time.perf_counter(), os.times()
    th = [threading.Thread(target=body, args=(i,)) for i in range(k)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    wall = (time.perf_counter() - t0) * 1e3
    c1 = os.times()
    cpu = (c1.user - c0.user) + (c1.system - c0.system)
    dev = max(ctxs[0].elapsed_ms_to(0, cx, 1) for cx in ctxs[:k])
    its = sum(r.total_lin for r in res)
    return dev, wall, cpu, its


for k in [int(s) for s in a.ks.split(",")]:
    run(k)  # warm-up (graphs, pools)
    rows = [run(k) for _ in range(a.reps)]
    dev = min(r[0] for r in rows)
    wall = min(r[1] for r in rows)
    cpu = min(r[2] for r in rows)
    its = rows[0][3]
    print(f"k={k}: device {dev:.1f} ms, wall {wall:.1f} ms, host cpu {cpu:.2f} s "
          f"({cpu * 1e3 / wall:.1f} cores busy), {its} Krylov its, {its / dev * 1e3:.0f} it/s", flush=True)

for p in probs:  # problems before their contexts
    p.close()
for cx in ctxs:
    cx.close()
