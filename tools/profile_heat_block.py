"""ncu workload: a C5-like heat problem with few time blocks, one Newton step,
then one timed preconditioner apply (the block solves of the time
substitution dominate C5).

    python tools/profile_heat_block.py [nt=8]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_05896_b200 import configs, optcon as oc  # noqa: E402

nt = int(sys.argv[1]) if len(sys.argv) > 1 else 8
c = configs.C5
tau = 1.0 / nt
yd = configs.sine_modes_spacetime(c.level, nt, tau, 42)
ctx = oc.Context(0)
qp = oc.assemble_spacetime(oc.ControlProblem(pde="heat", alpha=c.alpha, beta=c.beta, y_d=yd,
                                             u_a=c.u_a, u_b=c.u_b, tau=tau), oc.Grid(c.level), ctx)
oc.ipm_solve(qp, oc.IpmParams(sigma=c.sigma, solver="gmres-pt", max_iterations=1))
print("MARK", flush=True)
k, p = qp.time_applies("pt", 1)
print(f"heat nt={nt}: kkt {k:.3f} ms precond {p:.3f} ms")
