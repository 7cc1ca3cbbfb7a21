"""Full-size parity: device solve vs the reference compiled from its sources
(oracle/_ref) on identical seeded inputs, for the BASELINE configs. The
reference runs on the host cores (one process per case, in parallel).

    python tools/parity_full.py [--out gpurun_out/parity_full.json] [cases...]

Cases: C1, C2 (9 cells), C4, C5 (gmres-pt, reference-native), C5m (C5 with
block-diagonal MINRES against the reference-class composition), C3@8 (C3 at
level 8: the reference needs ~1.4 h at 1025^2). Bar (north_star): u, y, J to rel 1e-8, NLI +-1, zero-count
and active sets exact.
"""
import argparse
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def case_list(names):
    from paper_1806_05896_b200 import configs

    out = []
    for nm in names:
        if nm == "C2":
            out += [(f"C2[{i}]", c) for i, c in enumerate(configs.C2_CELLS)]
        elif nm == "C5m":  # C5 with the solver BASELINE names (block-diagonal MINRES)
            out.append((nm, configs.C5.with_level(8, solver="minres-pd")))
        elif "@" in nm:
            base, lvl = nm.split("@")
            out.append((nm, configs.ALL[base].with_level(int(lvl))))
        else:
            out.append((nm, configs.ALL[nm]))
    return out


def problem_kwargs(c):
    kw = dict(alpha=c.alpha, beta=c.beta, y_d=c.y_d(), u_a=c.u_a, u_b=c.u_b)
    if c.pde == "convdiff":
        kw["eps"] = c.eps
    if c.pde == "heat":
        kw["tau"] = c.tau
    if c.y_a is not None:
        kw.update(y_a=c.y_a, y_b=c.y_b)
    return kw


def run_ref(args):
    name, c = args
    from oracle import ref

    kw = problem_kwargs(c)
    if c.obs is not None:
        kw["obs"] = c.obs
    t0 = time.perf_counter()
    P = ref.RefProblem(c.pde, c.level, **kw)
    # heat MINRES-P_D: the reference-class composition
    solver = "heat-minres-pd" if c.pde == "heat" and c.solver == "minres-pd" else c.solver
    r = P.solve(solver, sigma=c.sigma)
    return name, dict(u=r.u, y=r.y, z=r.z, nli=r.nli, av_li=r.av_li, objective=r.objective,
                      converged=r.converged, seconds=time.perf_counter() - t0,
                      lin=[d["lin_iters"] for d in r.records[1:]],
                      lin_converged=all(d["lin_converged"] for d in r.records[1:]))


def run_gpu(cases, smoother="color4"):
    from paper_1806_05896_b200 import optcon as oc

    ctx = oc.Context(0)
    out = {}
    for name, c in cases:
        kw = problem_kwargs(c)
        kw["pde"] = c.pde
        if c.obs is not None:
            kw["observation"] = c.obs
        qp = oc.QpProblem(oc.ControlProblem(**kw), oc.Grid(c.level), ctx)
        r = oc.ipm_solve(qp, oc.IpmParams(sigma=c.sigma, solver=c.solver,
                                          gmres_restart=c.gmres_restart, smoother=smoother))
        out[name] = dict(u=r.u.copy(), y=r.state.y.copy(), z=r.state.z.copy(), nli=r.stats.nli,
                         av_li=r.stats.av_li, objective=r.objective, converged=r.stats.converged,
                         ms=r.solve_ms, lin=[i.lin_iters for i in r.stats.iterations[1:]],
                         lin_converged=all(i.lin_converged for i in r.stats.iterations[1:]))
        qp.close()
    return out


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def compare(c, g, r):
    res = dict(rel_u=rel(g["u"], r["u"]), rel_y=rel(g["y"], r["y"]), rel_z=rel(g["z"], r["z"]),
               rel_J=abs(g["objective"] - r["objective"]) / abs(r["objective"]),
               nli=(g["nli"], r["nli"]), av_li=(round(g["av_li"], 3), round(r["av_li"], 3)),
               zeros=(int((np.abs(g["u"]) < 1e-2).sum()), int((np.abs(r["u"]) < 1e-2).sum())),
               gpu_ms=round(g["ms"], 2), ref_s=round(r["seconds"], 2),
               lin_converged=(g["lin_converged"], r["lin_converged"]))
    ua, ub = c.u_a, c.u_b
    act = [np.array_equal(g["u"] - ua < 1e-2, r["u"] - ua < 1e-2),
           np.array_equal(ub - g["u"] < 1e-2, ub - r["u"] < 1e-2)]
    if c.y_a is not None:
        span = c.y_b - c.y_a
        act += [np.array_equal(g["y"] - c.y_a < 1e-2 * span, r["y"] - c.y_a < 1e-2 * span),
                np.array_equal(c.y_b - g["y"] < 1e-2 * span, c.y_b - r["y"] < 1e-2 * span)]
    res["active_sets_equal"] = bool(all(act))
    res["pass"] = bool(res["rel_u"] <= 1e-8 and res["rel_y"] <= 1e-8 and res["rel_J"] <= 1e-8
                       and abs(g["nli"] - r["nli"]) <= 1 and res["zeros"][0] == res["zeros"][1]
                       and res["active_sets_equal"])
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cases", nargs="*", default=["C1", "C2", "C4", "C5", "C3@8"])
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "parity_full.json"))
    ap.add_argument("--procs", type=int, default=os.cpu_count() or 4)
    ap.add_argument("--smoother", default="auto", help="auto (default) | color4 | lex (faithful mode)")
    a = ap.parse_args()
    cases = case_list(a.cases)
    gpu = run_gpu(cases, a.smoother)
    print("gpu done", {k: round(v["ms"], 1) for k, v in gpu.items()}, flush=True)
    report = {}
    ctx = mp.get_context("fork")
    with ctx.Pool(min(a.procs, len(cases))) as pool:
        for name, r in pool.imap_unordered(run_ref, cases):
            c = dict(cases)[name]
            report[name] = compare(c, gpu[name], r)
            report[name]["smoother"] = a.smoother
            report[name]["lin_iters"] = (gpu[name]["lin"], r["lin"])
            print(name, json.dumps(report[name]), flush=True)
            os.makedirs(os.path.dirname(a.out), exist_ok=True)
            json.dump(report, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
