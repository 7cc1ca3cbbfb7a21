"""%globaltimer stamps of one lexicographic sweep per band (tuning aid).

    python tools/lex_probe.py [level=10] [var=0]
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_05896_b200 import _lib, optcon as oc  # noqa: E402

ell = int(sys.argv[1]) if len(sys.argv) > 1 else 10
var = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ctx = oc.Context(0)
A = oc.assemble9("convdiff" if var else "poisson", ell, eps=0.02)
if not var:
    A = A.copy()
mg = oc.MgHierarchy(A, ell, ctx=ctx, smoother="lex")
b = np.random.default_rng(0).uniform(-1, 1, A.shape[1])
x0 = np.zeros_like(b)
L = _lib.load()
buf = (C.c_ulonglong * 512)()
mg.smooth(b, x0, True)
L.oc_debug_cluster_probes(3, buf)  # lex probes on
mg.smooth(b, x0, True)
L.oc_debug_cluster_probes(2, buf)  # read + off
t = np.array(buf, dtype=np.float64).reshape(64, 8)
nb = ((1 << ell) - 1 + 31) // 32
t0 = t[:nb, 0].min()
print("band  start  spun  c8end  end")
for w in range(nb):
    print(w, " ".join(f"{(t[w, s] - t0) / 1e3:8.1f}" for s in (0, 1, 2, 5)))
