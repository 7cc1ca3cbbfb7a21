"""Device solve of one BASELINE config compared with reference outputs saved by
tools/ref_solve_save.py (for configs whose reference run is too long to repeat
on the GPU box).

    python tools/compare_saved.py C3 saved.npz [--smoother lex] [--out report.json]
    python tools/compare_saved.py C3 saved.npz --device device.npz   (no GPU needed)
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from paper_1806_05896_b200 import configs, optcon as oc  # noqa: E402
from parity_full import compare, problem_kwargs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("saved")
ap.add_argument("--smoother", default="color4")
ap.add_argument("--out", default=None)
ap.add_argument("--device", default=None, help="device results saved by tools/device_solve_save.py")
a = ap.parse_args()
s = np.load(a.saved)
c = configs.ALL[a.config].with_level(int(s["level"]))
kw = problem_kwargs(c)
kw["pde"] = c.pde
if c.obs is not None:
    kw["observation"] = c.obs
if a.device:
    d = np.load(a.device)
    a.smoother = str(d["smoother"])
    g = dict(u=d["u"], y=d["y"], z=d["z"], nli=int(d["nli"]), av_li=float(d["av_li"]),
             objective=float(d["objective"]), ms=float(d["ms"]), lin_converged=bool(d["lin_converged"]))
    dev_lin = [int(v) for v in d["lin"]]
else:
    ctx = oc.Context(0)
    qp = oc.QpProblem(oc.ControlProblem(**kw), oc.Grid(c.level), ctx)
    r = oc.ipm_solve(qp, oc.IpmParams(sigma=c.sigma, solver=c.solver, gmres_restart=c.gmres_restart,
                                      smoother=a.smoother))
    g = dict(u=r.u, y=r.state.y, z=r.state.z, nli=r.stats.nli, av_li=r.stats.av_li,
             objective=r.objective, ms=r.solve_ms,
             lin_converged=all(i.lin_converged for i in r.stats.iterations[1:]))
    dev_lin = [i.lin_iters for i in r.stats.iterations[1:]]
ref = dict(u=s["u"], y=s["y"], z=s["z"], nli=int(s["nli"]), av_li=float(s["av_li"]),
           objective=float(s["objective"]), seconds=float(s["seconds"]), lin_converged=None)
rep = compare(c, g, ref)
rep.update(smoother=a.smoother, level=c.level,
           lin_iters=(dev_lin, [int(v) for v in s["lin"]]))
print(json.dumps(rep))
if a.out:
    json.dump(rep, open(a.out, "w"), indent=1)
