"""Run the reference (oracle/_ref) on one BASELINE config on this machine's CPU
and save its outputs for a later device comparison (tools/compare_saved.py).

    python tools/ref_solve_save.py C3 out.npz [level]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
from paper_1806_05896_b200 import configs  # noqa: E402

name, out = sys.argv[1], sys.argv[2]
c = configs.ALL[name]
if len(sys.argv) > 3:
    c = c.with_level(int(sys.argv[3]))
kw = dict(alpha=c.alpha, beta=c.beta, y_d=c.y_d(), u_a=c.u_a, u_b=c.u_b)
if c.pde == "convdiff":
    kw["eps"] = c.eps
if c.pde == "heat":
    kw["tau"] = c.tau
if c.y_a is not None:
    kw.update(y_a=c.y_a, y_b=c.y_b)
if c.obs is not None:
    kw["obs"] = c.obs
t0 = time.perf_counter()
r = ref.RefProblem(c.pde, c.level, **kw).solve(c.solver, sigma=c.sigma)
dt = time.perf_counter() - t0
np.savez(out, u=r.u, y=r.y, z=r.z, objective=r.objective, nli=r.nli, av_li=r.av_li,
         lin=np.array([d["lin_iters"] for d in r.records[1:]]), seconds=dt, level=c.level)
print(f"{name} level {c.level}: nli {r.nli} av_li {r.av_li:.3f} J {r.objective:.15g} in {dt:.1f} s")
