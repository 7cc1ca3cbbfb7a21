"""Profiling aid: a few multigrid solves at one level (default 7), e.g. for
ncu capture of the cluster bottom kernel.

    python tools/mg_once.py [level=7] [reps=3] [smoother=color4]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_05896_b200 import optcon as oc  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 7
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
smoother = sys.argv[3] if len(sys.argv) > 3 else "color4"
ctx = oc.Context(0)
L = oc.assemble9("poisson", level)
L[4] += 1.0
mg = oc.MgHierarchy(L, level, ctx=ctx, smoother=smoother)
b = np.random.default_rng(0).uniform(-1, 1, L.shape[1])
import time  # noqa: E402

for _ in range(reps):
    t0 = time.perf_counter()
    x = mg.solve(b, 1, 5, 5)
    print(f"solve {1e3 * (time.perf_counter() - t0):.2f} ms")
print("ok", float(np.linalg.norm(x)))
