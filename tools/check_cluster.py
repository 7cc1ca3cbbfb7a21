"""Debug aid: multigrid solve with the cluster bottom (levels <= 7 in one
16-CTA cluster, levels <= 4 as the dense coarse-cycle operator) against the
single-CTA bottom on the same hierarchy data.

    python tools/check_cluster.py [levels=6,7,8]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_05896_b200 import _lib, optcon as oc  # noqa: E402

levels = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "6,7,8").split(",")]
lib = _lib.load()
ctx = oc.Context(0)
for level in levels:
    L = oc.assemble9("poisson", level)
    L[4] += 1.0
    b = np.random.default_rng(0).uniform(-1, 1, L.shape[1])
    out = {}
    for cb in (0, 1):
        _lib.check(lib.oc_set_tuning(b"cluster_bottom", cb))
        mg = oc.MgHierarchy(L, level, ctx=ctx)
        if cb:
            B = np.zeros((225, 225))
            _lib.check(lib.oc_debug_coarse_op(mg.h, 5, 5, B.ctypes.data))
            print(f"level {level}: B4 nan {int(np.isnan(B).sum())}, |B4| {np.abs(B).max():.3e}, "
                  f"asym {np.abs(B - B.T).max() / np.abs(B).max():.3e}", flush=True)
        out[cb] = {cyc: mg.solve(b, cyc, 5, 5) for cyc in (1, 3)}
        print(f"  cluster_bottom={cb}: nan {[int(np.isnan(v).sum()) for v in out[cb].values()]}", flush=True)
        del mg
    for cyc in (1, 3):
        d = np.linalg.norm(out[1][cyc] - out[0][cyc]) / np.linalg.norm(out[0][cyc])
        print(f"level {level} cycles {cyc}: rel diff cluster vs single-CTA {d:.3e}", flush=True)
_lib.check(lib.oc_set_tuning(b"cluster_bottom", 1))
