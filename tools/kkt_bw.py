"""Steady KKT apply at 1025^2 for the three variants (kkt_tiled knob: 0 one
node per thread through L1, 1 shared-memory halo tiles, 2 TMA-staged tiles):
device time per apply (oc_time_applies) and the bytes it must move (fields,
Theta, outputs and the variable operators' coefficient arrays), plus a
bit-for-bit comparison of the applies.

    python tools/kkt_bw.py
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_05896_b200 import _lib, configs, optcon as oc  # noqa: E402

L = _lib.load()
peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json"))).get("hbm_gbs", 6442.2) \
    if os.path.exists(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")) else 6442.2
ctx = oc.Context(0)
cases = {"C2-type poisson 1025^2": configs.C2_CELLS[4].with_level(10), "C3": configs.C3, "C4": configs.C4}
for name, c in cases.items():
    kw = dict(pde=c.pde, alpha=c.alpha, beta=c.beta, y_d=c.y_d(), u_a=c.u_a, u_b=c.u_b)
    if c.pde == "convdiff":
        kw["eps"] = c.eps
    if c.y_a is not None:
        kw.update(y_a=c.y_a, y_b=c.y_b)
    if c.obs is not None:
        kw["observation"] = c.obs
    qp = oc.QpProblem(oc.ControlProblem(**kw), oc.Grid(c.level), ctx)
    try:
        oc.ipm_solve(qp, oc.IpmParams(sigma=c.sigma, solver=c.solver, max_iterations=1,
                                      linear_maxit=2, smoother="color4"))
    except Exception:
        pass
    n = qp.ny
    words = 4 + 2 + 4 + (1 if c.y_a is not None else 0) + (18 if c.pde == "convdiff" else 0) + \
        (9 if c.obs is not None else 0)
    rng = np.random.default_rng(1)
    th = oc.ThetaBlocks(rng.uniform(0.1, 1, n) if c.y_a is not None else None, rng.uniform(0.1, 1, n),
                        rng.uniform(0.1, 1, n))
    x = rng.uniform(-1, 1, 4 * n)
    ref = None
    for v in (0, 1, 2):
        _lib.check(L.oc_set_tuning(b"kkt_tiled", v))
        kind = {"gmres-pt": "pt", "gmres-ppi": "ppi", "minres-pd": "pd"}[c.solver]
        k_ms, _ = qp.time_applies(kind, 50)
        ax = qp.kkt_apply(th, x)
        if ref is None:
            ref = ax
        same = bool(np.array_equal(ax, ref))
        gbs = words * 8.0 * n / (k_ms / 1e3) / 1e9
        print(json.dumps({"case": name, "kkt_tiled": v, "kkt_ms": round(k_ms, 4), "words_per_node": words,
                          "gbs": round(gbs, 1), "frac": round(gbs / peak, 3), "bitwise_equal_to_v0": same}),
              flush=True)
    qp.close()
_lib.check(L.oc_set_tuning(b"kkt_tiled", 1))
