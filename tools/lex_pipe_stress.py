"""Race stress for the pipelined lexicographic sweep batches: repeated multigrid
solves (2 V-cycles, 5 + 5 sweeps) at levels 10, 9, 8, 7 with the batches on,
each compared bit for bit with one sequential-launch solve.

    python tools/lex_pipe_stress.py
"""
import os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_1806_05896_b200 import _lib, optcon as oc
lib = _lib.load(); ctx = oc.Context(0)
bad = 0
for ell, kind in ((10, "convdiff"), (9, "poisson"), (8, "convdiff"), (7, "poisson")):
    L = oc.assemble9(kind, ell, eps=0.02) if kind == "convdiff" else oc.assemble9(kind, ell)
    L[4] += 1.0
    b = np.random.default_rng(ell).uniform(-1, 1, L.shape[1])
    _lib.check(lib.oc_set_tuning(b"lex_pipeline", 0))
    mg = oc.MgHierarchy(L, ell, ctx=ctx, smoother="lex"); ref = mg.solve(b, 2, 5, 5); mg.close()
    _lib.check(lib.oc_set_tuning(b"lex_pipeline", 1))
    mg = oc.MgHierarchy(L, ell, ctx=ctx, smoother="lex")
    n = 60 if ell < 10 else 25
    for i in range(n):
        x = mg.solve(b, 2, 5, 5)
        if not np.array_equal(x, ref):
            bad += 1
            print("MISMATCH", ell, kind, i, float(np.abs(x - ref).max()), flush=True)
    mg.close()
    print("level", ell, kind, "runs", n, "mismatches so far", bad, flush=True)
print("TOTAL MISMATCHES", bad)
