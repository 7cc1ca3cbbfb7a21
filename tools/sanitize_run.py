"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
every hand-written inter-CTA / intra-CTA protocol of the library runs once.

* C1-style solve at level 6 (the 16-CTA cluster bottom with st.async /
  mbarrier halo exchange, tiled sweeps, Chebyshev blocks, tiled KKT);
* lexicographic sweeps and V-cycle at level 7 (4 wavefront bands: the
  staging / compute warps, the sentinel mailbox between CTAs);
* C3-style capped GMRES at level 5 (columns j+1 >= 8 run the cooperative
  persistent Gram-Schmidt with its software grid barrier);
* a heat solve at level 4 x 4 steps (level-8-style batched time blocks).

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_05896_b200 import configs, optcon as oc  # noqa: E402

ctx = oc.Context(0)
c = configs.C1
qp = oc.build_qp(oc.ControlProblem(alpha=c.alpha, beta=c.beta, y_d=c.y_d(), u_a=c.u_a, u_b=c.u_b),
                 oc.Grid(c.level), ctx)
r = oc.ipm_solve(qp, oc.IpmParams(sigma=0.2, solver="gmres-pt", max_iterations=2))
print("C1 l6 gmres-pt 2 IPM iterations:", [i.lin_iters for i in r.stats.iterations[1:]], flush=True)

A = oc.assemble9("convdiff", 7, eps=0.02)
mg = oc.MgHierarchy(A, 7, ctx=ctx, smoother="lex")
b = np.random.default_rng(0).uniform(-1, 1, A.shape[1])
x = mg.smooth(b, np.zeros_like(b), True)
x = mg.smooth(b, x, False)
x = mg.solve(b, 1, 2, 2)
print("lex level 7 sweeps + V-cycle:", float(np.linalg.norm(x)), flush=True)

c3 = configs.C3.with_level(5)
q3 = oc.build_qp(oc.ControlProblem(alpha=c3.alpha, beta=c3.beta, y_d=c3.y_d(), u_a=c3.u_a,
                                   u_b=c3.u_b, y_a=c3.y_a, y_b=c3.y_b, observation=c3.obs),
                 oc.Grid(5), ctx)
r3 = oc.ipm_solve(q3, oc.IpmParams(sigma=0.2, solver="gmres-ppi", max_iterations=1,
                                   linear_maxit=12, smoother="color4"))
print("C3 l5 capped GMRES (persistent MGS from j+1 = 8):", r3.stats.iterations[1].lin_iters, flush=True)

c5 = configs.C5.with_level(4, tau=0.25)
q5 = oc.assemble_spacetime(oc.ControlProblem(pde="heat", tau=c5.tau, alpha=c5.alpha, beta=c5.beta,
                                             y_d=c5.y_d(), u_a=c5.u_a, u_b=c5.u_b),
                           oc.Grid(4), ctx)
r5 = oc.ipm_solve(q5, oc.IpmParams(sigma=0.2, solver="minres-pd", max_iterations=2))
print("heat l4 x 4 minres-pd:", [i.lin_iters for i in r5.stats.iterations[1:]], flush=True)
print("SANITIZE WORKLOAD DONE")
