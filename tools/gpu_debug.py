"""Quick on-device parity probe (dev tool): GPU path vs the CPU reference oracle."""
import sys, time, traceback
import numpy as np
sys.path.insert(0, '/root/repo')
from oracle import ref
from paper_1806_05896_b200 import optcon as oc, configs

def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))

rng = np.random.default_rng(7)
for lvl in [4, 6]:
    n = ((1 << lvl) - 1) ** 2
    # KKT apply parity
    yd = configs.sine_modes(lvl)
    for pde, extra in [("poisson", {}), ("convdiff", dict(eps=0.02))]:
        try:
            R = ref.RefProblem(pde, lvl, alpha=1e-2, beta=1e-3, y_d=yd, u_a=-2, u_b=2, **extra)
            qp = oc.build_qp(oc.ControlProblem(pde=pde, alpha=1e-2, beta=1e-3, y_d=yd, u_a=-2.0, u_b=2.0, **extra), oc.Grid(lvl))
            tw = 10 ** rng.uniform(-2, 2, n); tv = 10 ** rng.uniform(-2, 2, n); ty = np.zeros(n)
            x = rng.uniform(-1, 1, 4 * n)
            a = R.kkt_apply(ty, tw, tv, x)
            b = qp.kkt_apply(oc.ThetaBlocks(None, tw, tv), x)
            print("KKT", lvl, pde, rel(b, a), flush=True)
            R.precond_setup(ty, tw, tv)
            for kind in ["pd", "pt"]:
                qp.precond_setup(oc.ThetaBlocks(None, tw, tv), oc.IpmParams(solver="gmres-pt" if kind == "pt" else "minres-pd"))
                r = rng.uniform(-1, 1, 4 * n)
                pa = R.precond_apply(kind, r); pb = qp.precond_apply(kind, r)
                blocks = [rel(pb[i*n:(i+1)*n], pa[i*n:(i+1)*n]) for i in range(4)]
                print("P", kind, lvl, pde, blocks, flush=True)
        except Exception:
            traceback.print_exc()

for cfg in [configs.C1, configs.C1.with_level(6, solver="gmres-pt")]:
    try:
        yd = cfg.y_d()
        R = ref.RefProblem(cfg.pde, cfg.level, alpha=cfg.alpha, beta=cfg.beta, y_d=yd, u_a=cfg.u_a, u_b=cfg.u_b)
        t = time.time(); rr = R.solve(cfg.solver, sigma=cfg.sigma); tr = time.time() - t
        qp = oc.build_qp(oc.ControlProblem(pde=cfg.pde, alpha=cfg.alpha, beta=cfg.beta, y_d=yd, u_a=cfg.u_a, u_b=cfg.u_b), oc.Grid(cfg.level))
        t = time.time(); rg = oc.ipm_solve(qp, oc.IpmParams(sigma=cfg.sigma, solver=cfg.solver)); tg = time.time() - t
        print("IPM", cfg.solver, "ref nli", rr.nli, "av", rr.av_li, "t", tr, "| gpu nli", rg.stats.nli, "av", rg.stats.av_li, "t", tg, rg.solve_ms)
        print("  rel u", rel(rg.u, rr.u), "rel y", rel(rg.state.y, rr.y), "J", rg.objective, rr.objective, "zeros", (np.abs(rg.u) < 1e-2).sum(), (np.abs(rr.u) < 1e-2).sum())
        for a, b in zip(rr.records, rg.stats.iterations):
            print("   ", a["k"], a["lin_iters"], b.lin_iters, a["norm_xd"], b.norm_xd, b.newton_ms)
    except Exception:
        traceback.print_exc()
