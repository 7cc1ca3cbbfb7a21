"""Tuning aid: phase timeline (us) of the level-8 cluster kernel (heat time
block solve, 3 V-cycles) from its %globaltimer probes.

    python tools/probe_top8.py
"""
import ctypes as C
import dataclasses
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_05896_b200 import _lib, configs, optcon as oc  # noqa: E402

c = dataclasses.replace(configs.C5, horizon=2 * configs.C5.tau)
lib = _lib.load()
ctx = oc.Context(0)
qp = oc.QpProblem(oc.ControlProblem(pde="heat", alpha=c.alpha, beta=c.beta, y_d=c.y_d(), u_a=c.u_a,
                                    u_b=c.u_b, tau=c.tau, horizon=c.horizon), oc.Grid(c.level), ctx)
oc.ipm_solve(qp, oc.IpmParams(sigma=c.sigma, solver=c.solver))
NAMES = {0: "start", 1: "loaded", 20: "cycle", 21: "l8 pre", 22: "l8 resid", 23: "l8 restrict",
         2: "l7 pre+resid", 3: "l6 restrict+pre+resid", 4: "c0 restrict", 5: "c0 levels",
         6: "prolong+l6 post", 7: "l7 post", 24: "l7 done", 25: "l8 prolong", 26: "l8 post"}
kk, pp = C.c_double(), C.c_double()
lib.oc_debug_cluster_probes(1, None)
_lib.check(lib.oc_time_applies(qp.h, 1, 1, C.byref(kk), C.byref(pp)))
buf = (C.c_ulonglong * 64)()
lib.oc_debug_cluster_probes(0, buf)
t = np.array(buf[:], dtype=np.int64)
base = t[0]
print("apply ms", pp.value)
print("CTA 0", [(NAMES.get(i, i), round((t[i] - base) / 1e3, 2)) for i in range(32) if t[i]])
