"""Tuning aid: time one C2-style cell solve under each sweep launch shape.

    python tools/tune.py [level=9] [solver=gmres-pt]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_05896_b200 import _lib, configs, optcon as oc  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 9
solver = sys.argv[2] if len(sys.argv) > 2 else "gmres-pt"
L = _lib.load()
c = configs.C2_CELLS[4].with_level(level, solver=solver)
ctx = oc.Context(0)
qp = oc.build_qp(oc.ControlProblem(alpha=c.alpha, beta=c.beta, y_d=c.y_d(), u_a=c.u_a, u_b=c.u_b),
                 oc.Grid(level), ctx)
params = oc.IpmParams(sigma=0.2, solver=solver)
oc.ipm_solve(qp, params)
ref_u = None
for fuse in (1, 2, 3, 5):
    for tile in (0, 1, 2, 3):
        L.oc_set_tuning(b"sweep_tile", tile)
        L.oc_set_tuning(b"sweep_fuse", fuse)
        oc.ipm_solve(qp, params)
        best = min(oc.ipm_solve(qp, params).solve_ms for _ in range(2))
        r = oc.ipm_solve(qp, params)
        import numpy as np

        if ref_u is None:
            ref_u = r.u.copy()
        d = float(np.linalg.norm(r.u - ref_u) / np.linalg.norm(ref_u))
        print(f"level {level} fuse {fuse} tile {tile}: {best:8.2f} ms  nli {r.stats.nli} "
              f"av_li {r.stats.av_li:.2f} drift {d:.1e}", flush=True)
