"""A/B of the heat KKT apply (knob kkt_tiled off/on): bitwise comparison of
A x on random x and theta at the C5 size, apply time from oc_time_applies.

    python tools/kkt_heat_ab.py [nt=128]
"""
import dataclasses
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_05896_b200 import _lib, configs, optcon as oc  # noqa: E402

nt = int(sys.argv[1]) if len(sys.argv) > 1 else 128
c = dataclasses.replace(configs.C5, horizon=nt * configs.C5.tau)
lib = _lib.load()
ctx = oc.Context(0)
qp = oc.QpProblem(oc.ControlProblem(pde="heat", alpha=c.alpha, beta=c.beta, y_d=c.y_d(), u_a=c.u_a,
                                    u_b=c.u_b, tau=c.tau, horizon=c.horizon), oc.Grid(c.level), ctx)
rng = np.random.default_rng(1)
ny = qp.ny
x = rng.standard_normal(4 * ny)
th = oc.ThetaBlocks(theta_y=None, theta_w=rng.random(ny) + 0.1, theta_v=rng.random(ny) + 0.1)
out = {}
for v in (0, 1):
    _lib.check(lib.oc_set_tuning(b"kkt_tiled", v))
    out[v] = np.array(qp.kkt_apply(th, x))
print("max|diff|", float(np.abs(out[0] - out[1]).max()), "rel", float(np.abs(out[0] - out[1]).max() / np.abs(out[0]).max()))
r = oc.ipm_solve(qp, oc.IpmParams(sigma=c.sigma, solver="minres-pd", max_iterations=1))
for v in (0, 1):
    _lib.check(lib.oc_set_tuning(b"kkt_tiled", v))
    k, p = qp.time_applies("pd", 5)
    print("kkt_tiled", v, "kkt_ms", round(k, 4), "prec_ms", round(p, 3))
