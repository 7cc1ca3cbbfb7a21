"""A/B of the pipelined lexicographic sweep batches (knob lex_pipeline): one
multigrid solve (3 V-cycles, 5 + 5 sweeps) of a variable operator per level,
off and on: bitwise comparison and wall time per solve.

    python tools/lex_pipe_ab.py [levels...=8 9 10]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_05896_b200 import _lib, optcon as oc  # noqa: E402

lib = _lib.load()
ctx = oc.Context(0)
for ell in [int(a) for a in sys.argv[1:]] or [8, 9, 10]:
    for kind in ("convdiff", "poisson"):
        L = oc.assemble9(kind, ell, eps=0.02) if kind == "convdiff" else oc.assemble9(kind, ell)
        L[4] += 1.0
        b = np.random.default_rng(5).uniform(-1, 1, L.shape[1])
        out, ms = {}, {}
        for v in (0, 1):
            _lib.check(lib.oc_set_tuning(b"lex_pipeline", v))
            mg = oc.MgHierarchy(L, ell, ctx=ctx, smoother="lex")
            mg.solve(b, 1, 5, 5)  # warm
            t0 = time.perf_counter()
            for _ in range(3):
                out[v] = mg.solve(b, 3, 5, 5)
            ms[v] = (time.perf_counter() - t0) / 3 * 1e3
            mg.close()
        d = float(np.abs(out[0] - out[1]).max())
        print(f"level {ell} {kind}: max|diff| {d} {'bitwise' if d == 0 else 'DIFFERENT'}; "
              f"solve ms off/on {ms[0]:.2f} / {ms[1]:.2f}", flush=True)
