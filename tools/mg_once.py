"""Profiling aid: a few multigrid solves at one level (default 7), e.g. for
ncu capture of the cluster bottom kernel.

    python tools/mg_once.py [level=7] [reps=3]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_05896_b200 import optcon as oc  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 7
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = oc.Context(0)
L = oc.assemble9("poisson", level)
L[4] += 1.0
mg = oc.MgHierarchy(L, level, ctx=ctx)
b = np.random.default_rng(0).uniform(-1, 1, L.shape[1])
for _ in range(reps):
    x = mg.solve(b, 1, 5, 5)
print("ok", float(np.linalg.norm(x)))
