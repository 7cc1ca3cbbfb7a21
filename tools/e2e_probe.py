import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
from paper_1806_05896_b200 import configs, optcon as oc
ctx = oc.Context(0)
c = configs.C2_CELLS[4]
yd = c.y_d()
for rep in range(3):
    t0 = time.perf_counter()
    qp = oc.build_qp(oc.ControlProblem(alpha=c.alpha, beta=c.beta, y_d=yd, u_a=c.u_a, u_b=c.u_b), oc.Grid(9), ctx)
    t1 = time.perf_counter()
    r = oc.ipm_solve(qp, oc.IpmParams(sigma=0.2, solver="gmres-pt"))
    t2 = time.perf_counter()
    u = r.u.copy()
    t3 = time.perf_counter()
    qp.close()
    t4 = time.perf_counter()
    print(f"build {1e3*(t1-t0):.1f} ms  solve wall {1e3*(t2-t1):.1f} ms (device {r.solve_ms:.1f})  close {1e3*(t4-t3):.1f} ms")
