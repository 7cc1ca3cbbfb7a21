"""Tuning aid: phase timeline (us) of the cluster multigrid bottom kernel.

    python tools/cluster_probe.py [level=7]
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_05896_b200 import _lib, optcon as oc  # noqa: E402

NAMES = {0: "start", 1: "loaded", 2: "top pre+resid", 3: "l6 restrict+pre+resid",
         4: "c0 restrict", 5: "c0 levels", 6: "prolong+l6 post", 7: "top post"}

level = int(sys.argv[1]) if len(sys.argv) > 1 else 7
ctx = oc.Context(0)
L = oc.assemble9("poisson", level)
L[4] += 1.0
mg = oc.MgHierarchy(L, level, ctx=ctx)
b = np.random.default_rng(0).uniform(-1, 1, L.shape[1])
lib = _lib.load()
lib.oc_debug_cluster_probes.argtypes = [C.c_int, C.c_void_p]
lib.oc_debug_cluster_probes(1, None)
for _ in range(3):
    mg.solve(b, 1, 5, 5)
buf = (C.c_ulonglong * 64)()
import time  # noqa: E402

lib.oc_debug_cluster_probes(0, None)
for cyc in (1, 3):
    mg.solve(b, cyc, 5, 5)
    t0 = time.perf_counter()
    for _ in range(50):
        mg.solve(b, cyc, 5, 5)
    print(f"level {level} solve cycles={cyc}: {(time.perf_counter() - t0) / 50 * 1e6:.1f} us/call (host-timed)")
lib.oc_debug_cluster_probes(1, None)
mg.solve(b, 1, 5, 5)
lib.oc_debug_cluster_probes(0, buf)
t = np.array(buf[:], dtype=np.int64)
for r in range(2):
    base = t[r * 32]
    row = [(NAMES.get(i, i), round((t[r * 32 + i] - base) / 1e3, 2)) for i in range(32)
           if t[r * 32 + i]]
    print("CTA", r, row)
