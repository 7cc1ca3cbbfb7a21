"""Where the end-to-end (build_qp from host arrays -> ipm_solve -> host results)
time of the bench workload goes, per phase, for one cell alone and for the nine
C2 cells concurrently (one context + host thread each, as bench.py).

    python tools/e2e_probe.py [--reps 3]
"""
import argparse
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
from paper_1806_05896_b200 import configs, optcon as oc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()

cs = configs.C2_CELLS
grid = oc.Grid(9)
params = oc.IpmParams(sigma=0.2, solver="gmres-pt")
ctxs = [oc.Context(0) for _ in cs]
ny = 511 * 511
pinned = [dict(y_d=torch.from_numpy(c.y_d()).pin_memory(),
               u_a=torch.full((ny,), c.u_a, dtype=torch.float64).pin_memory(),
               u_b=torch.full((ny,), c.u_b, dtype=torch.float64).pin_memory()) for c in cs]
host_out = [dict(u=torch.zeros(ny, dtype=torch.float64).pin_memory().numpy(),
                 y=torch.zeros(ny, dtype=torch.float64).pin_memory().numpy(),
                 z=torch.zeros(2 * ny, dtype=torch.float64).pin_memory().numpy(),
                 p=torch.zeros(ny, dtype=torch.float64).pin_memory().numpy()) for _ in cs]
pageable_out = [dict(u=np.zeros(ny), y=np.zeros(ny), z=np.zeros(2 * ny), p=np.zeros(ny))
                for _ in cs]


def cell(i, out, resolve=False):
    c, hp = cs[i], pinned[i]
    t0 = time.perf_counter()
    qp = oc.build_qp(oc.ControlProblem(alpha=c.alpha, beta=c.beta, y_d=hp["y_d"].numpy(),
                                       u_a=hp["u_a"].numpy(), u_b=hp["u_b"].numpy()), grid, ctxs[i])
    ctxs[i].synchronize()
    t1 = time.perf_counter()
    r = oc.ipm_solve(qp, params, outputs=out[i])
    t2 = time.perf_counter()
    t3 = t2
    if resolve:
        oc.ipm_solve(qp, params, outputs=out[i])
        t3 = time.perf_counter()
    qp.close()
    t4 = time.perf_counter()
    return dict(build=1e3 * (t1 - t0), solve=1e3 * (t2 - t1), dev=r.solve_ms,
                resolve=1e3 * (t3 - t2), close=1e3 * (t4 - t3), it=r.total_lin)


def run_all(fn):
    res = [None] * len(cs)
    th = [threading.Thread(target=lambda i=i: res.__setitem__(i, fn(i))) for i in range(len(cs))]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    return res, 1e3 * (time.perf_counter() - t0)


def show(tag, rs, wall=None):
    keys = ["build", "solve", "dev", "resolve", "close"]
    m = {k: np.mean([r[k] for r in rs]) for k in keys}
    it = sum(r["it"] for r in rs)
    s = " ".join(f"{k} {m[k]:7.1f}" for k in keys)
    extra = f"  wall {wall:7.1f} ms  {it / wall * 1e3:7.1f} it/s" if wall else ""
    print(f"{tag:28s} {s}{extra}", flush=True)


for rep in range(a.reps):
    show("alone pinned (+resolve)", [cell(4, host_out, resolve=True)])
for rep in range(a.reps):
    rs, w = run_all(lambda i: cell(i, host_out))
    show("9 concurrent pinned out", rs, w)
for rep in range(a.reps):
    rs, w = run_all(lambda i: cell(i, pageable_out))
    show("9 concurrent pageable out", rs, w)
for rep in range(a.reps):
    rs, w = run_all(lambda i: cell(i, host_out, resolve=True))
    show("9 concurrent + resolve", rs, w)
