"""Device objects left alive at interpreter exit (module globals, several
contexts and problems) are closed in a safe order by the atexit hook: the
process exits cleanly instead of tearing a context down after the CUDA
runtime."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = """
import sys, threading
sys.path.insert(0, {root!r})
from paper_1806_05896_b200 import configs, optcon as oc
# nine C2 cells on their own contexts and host threads, left alive as globals
# (without the atexit hook this exits with SIGSEGV)
ctxs = [oc.Context(0) for _ in configs.C2_CELLS]
probs = [oc.build_qp(oc.ControlProblem(alpha=c.alpha, beta=c.beta, y_d=c.y_d(), u_a=c.u_a,
                                       u_b=c.u_b), oc.Grid(c.level), cx)
         for c, cx in zip(configs.C2_CELLS, ctxs)]
res = [None] * len(probs)
def body(i):
    res[i] = oc.ipm_solve(probs[i], oc.IpmParams(sigma=0.2, solver="gmres-pt"))
th = [threading.Thread(target=body, args=(i,)) for i in range(len(probs))]
for t in th: t.start()
for t in th: t.join()
mg = oc.MgHierarchy(oc.assemble9("poisson", 5), 5, ctx=ctxs[0])
print("solved", [r.stats.nli for r in res])
"""


def test_objects_alive_at_exit_close_cleanly():
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, (r.returncode, r.stderr[-2000:])
    assert "solved" in r.stdout


SCRIPT_CLOSE_FIRST = """
import sys
sys.path.insert(0, {root!r})
from paper_1806_05896_b200 import configs, optcon as oc
# the context is closed while its problem and hierarchy are alive (the C++
# façade's thread-local default context dying first): the problem still
# solves, and the context is released with its last child
ctx = oc.Context(0)
c = configs.C1
qp = oc.build_qp(oc.ControlProblem(alpha=c.alpha, beta=c.beta, y_d=c.y_d(), u_a=c.u_a, u_b=c.u_b),
                 oc.Grid(c.level), ctx)
mg = oc.MgHierarchy(oc.assemble9("poisson", 5), 5, ctx=ctx)
ctx.close()
r = oc.ipm_solve(qp, oc.IpmParams(sigma=0.2, solver="minres-pd"))
x = mg.solve(configs.sine_modes(5))
qp.close()
mg.close()
print("ok", r.stats.nli, r.stats.converged)
"""


def test_context_closed_before_its_problems():
    r = subprocess.run([sys.executable, "-c", SCRIPT_CLOSE_FIRST.format(root=ROOT)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.returncode, r.stderr[-2000:])
    assert "ok 9 True" in r.stdout
