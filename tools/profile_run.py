"""Workload for ncu captures: one C2 cell (level 9 by default) solved twice;
the second solve is the one to profile (skip the first solve's launches).

    python tools/profile_run.py [--level 9] [--solver gmres-pt] [--cell 4]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1806_05896_b200 import _lib, configs, optcon as oc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--level", type=int, default=9)
ap.add_argument("--solver", default="gmres-pt")
ap.add_argument("--cell", type=int, default=4)
ap.add_argument("--repeat", type=int, default=2)
ap.add_argument("--tile", type=int, default=None, help="sweep_tile knob (bench under concurrency: 0)")
ap.add_argument("--fuse", type=int, default=None)
a = ap.parse_args()

if a.tile is not None:
    _lib.check(_lib.load().oc_set_tuning(b"sweep_tile", a.tile))
if a.fuse is not None:
    _lib.check(_lib.load().oc_set_tuning(b"sweep_fuse", a.fuse))
c = configs.C2_CELLS[a.cell].with_level(a.level, solver=a.solver)
ctx = oc.Context(0)
qp = oc.build_qp(oc.ControlProblem(alpha=c.alpha, beta=c.beta, y_d=c.y_d(), u_a=c.u_a, u_b=c.u_b),
                 oc.Grid(a.level), ctx)
for i in range(a.repeat):
    l0 = oc.Context.launch_count()
    t0 = time.perf_counter()
    r = oc.ipm_solve(qp, oc.IpmParams(sigma=0.2, solver=a.solver))
    dt = time.perf_counter() - t0
    print(f"solve {i}: nli={r.stats.nli} av_li={r.stats.av_li:.2f} device_ms={r.solve_ms:.2f} "
          f"wall_ms={dt * 1e3:.2f} launches={oc.Context.launch_count() - l0}", flush=True)
