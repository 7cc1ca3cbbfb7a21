"""Generate the committed golden fixtures from the reference itself.

Runs the reference optcon library compiled from /root/reference (oracle/_ref,
built by `make -C oracle`) on seeded inputs and stores inputs + outputs as
small .npz files. GPU tests compare against these when the oracle library is
not available on the box; CPU tests check the numpy restatement against them.

    python tests/golden/make_golden.py            # everything
    python tests/golden/make_golden.py NAME ...   # only these IPM cases
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_1806_05896_b200 import configs  # noqa: E402

# (name, problem kwargs, solve kwargs); levels kept small so fixtures stay tiny
IPM_CASES = [
    ("known_answer_l6", dict(pde="poisson", level=6, alpha=1e-4, beta=1e-2, yd="sinsin",
                             u_a=-2.0, u_b=1.5), dict(solver="gmres-pt", sigma=0.2)),
    ("c1_l6_minres", dict(pde="poisson", level=6, alpha=1e-2, beta=1e-3, u_a=-2.0, u_b=2.0),
     dict(solver="minres-pd", sigma=0.2)),
    ("c1_l6_gmres", dict(pde="poisson", level=6, alpha=1e-2, beta=1e-3, u_a=-2.0, u_b=2.0),
     dict(solver="gmres-pt", sigma=0.2)),
    ("c2_l7_a1e-4_b1e-4", dict(pde="poisson", level=7, alpha=1e-4, beta=1e-4, u_a=-2.0,
                               u_b=2.0), dict(solver="gmres-pt", sigma=0.2)),
    ("c3_l5", dict(pde="poisson", level=5, alpha=1e-4, beta=1e-3, u_a=-2.0, u_b=2.0,
                   y_a=-0.2, y_b=0.3, obs=(0.0, 0.5, 0.0, 1.0)),
     dict(solver="gmres-ppi", sigma=0.2, linear_maxit=3000)),
    ("c3_l4", dict(pde="poisson", level=4, alpha=1e-4, beta=1e-3, u_a=-2.0, u_b=2.0,
                   y_a=-0.2, y_b=0.3, obs=(0.0, 0.5, 0.0, 1.0)),
     dict(solver="gmres-ppi", sigma=0.2, linear_maxit=3000)),
    ("c4_l6", dict(pde="convdiff", level=6, alpha=1e-4, beta=1e-3, u_a=-2.0, u_b=2.0, eps=0.02),
     dict(solver="gmres-pt", sigma=0.2)),
    ("c5_l5_nt16", dict(pde="heat", level=5, alpha=1e-3, beta=1e-4, u_a=-1.0, u_b=1.0,
                        tau=1.0 / 16), dict(solver="gmres-pt", sigma=0.2)),
    ("smoke_l5", dict(pde="poisson", level=5, alpha=1e-2, beta=1e-3, u_a=-2.0, u_b=2.0),
     dict(solver="gmres-pt", sigma=0.2)),
    # C3 in the capped-Krylov regime (every GMRES solve stops at linear_maxit,
    # as C3 does at 1025^2 with maxit 200): the solution depends on the exact
    # preconditioner, i.e. on the lexicographic smoother
    ("c3_l6_capped", dict(pde="poisson", level=6, alpha=1e-4, beta=1e-3, u_a=-2.0, u_b=2.0,
                          y_a=-0.2, y_b=0.3, obs=(0.0, 0.5, 0.0, 1.0)),
     dict(solver="gmres-ppi", sigma=0.2, linear_maxit=15)),
    # C3 with the reference's own cap (linear_maxit 200, ipm.hpp:27)
    ("c3_l6_maxit200", dict(pde="poisson", level=6, alpha=1e-4, beta=1e-3, u_a=-2.0, u_b=2.0,
                            y_a=-0.2, y_b=0.3, obs=(0.0, 0.5, 0.0, 1.0)),
     dict(solver="gmres-ppi", sigma=0.2, linear_maxit=200)),
]


def desired(kw):
    level = kw["level"]
    if kw.get("yd") == "sinsin":
        return configs.sin_sin(level)
    if kw["pde"] == "heat":
        nt = int(round(1.0 / kw["tau"]))
        return configs.sine_modes_spacetime(level, nt, kw["tau"], 42)
    return configs.sine_modes(level, 42)


def ref_problem(kw):
    k = dict(kw)
    k.pop("yd", None)
    pde = k.pop("pde")
    level = k.pop("level")
    return ref.RefProblem(pde, level, y_d=desired(kw), **k)


def make_ipm(only=()):
    for name, pkw, skw in IPM_CASES:
        if only and name not in only:
            continue
        P = ref_problem(pkw)
        r = P.solve(**skw)
        rec = np.array([[d["k"], d["mu"], d["norm_xp"], d["norm_xd"], d["norm_xc"],
                         d["lin_iters"], d["lin_relres"], d["lin_converged"]] for d in r.records])
        meta = dict(problem={k: v for k, v in pkw.items()}, solve=skw)
        out = dict(meta=json.dumps(meta), y_d=desired(pkw), y=r.y, z=r.z, p=r.p, u=r.u,
                   lam_za=r.lam_za, lam_zb=r.lam_zb, nli=r.nli, av_li=r.av_li, mu=r.mu,
                   objective=r.objective, converged=int(r.converged),
                   sparsity_pct=r.sparsity_pct, l1=r.l1, records=rec)
        if r.lam_ya is not None:
            out.update(lam_ya=r.lam_ya, lam_yb=r.lam_yb)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(f"{name}: nli={r.nli} av_li={r.av_li:.3f} converged={r.converged} "
              f"J={r.objective:.12g}")


def make_kkt():
    """Seeded KKT applies (make_saddle_operator) for each operator family."""
    rng = np.random.default_rng(7)
    cases = [
        ("kkt_poisson_l5", dict(pde="poisson", level=5, alpha=1e-2, beta=1e-3, u_a=-2.0, u_b=2.0)),
        ("kkt_convdiff_l5", dict(pde="convdiff", level=5, alpha=1e-4, beta=1e-3, u_a=-2.0,
                                 u_b=2.0, eps=0.02)),
        ("kkt_partial_l5", dict(pde="poisson", level=5, alpha=1e-4, beta=1e-3, u_a=-2.0, u_b=2.0,
                                y_a=-0.2, y_b=0.3, obs=(0.0, 0.5, 0.0, 1.0))),
        ("kkt_heat_l4", dict(pde="heat", level=4, alpha=1e-3, beta=1e-4, u_a=-1.0, u_b=1.0,
                             tau=0.125)),
    ]
    for name, pkw in cases:
        P = ref_problem(pkw)
        ny = P.ny
        tw = 10 ** rng.uniform(-2, 2, ny)
        tv = 10 ** rng.uniform(-2, 2, ny)
        ty = 10 ** rng.uniform(-3, 0, ny) if P.has_state_bounds else np.zeros(ny)
        x = rng.uniform(-1, 1, 4 * ny)
        ax = P.kkt_apply(ty, tw, tv, x)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"),
                            meta=json.dumps(dict(problem=pkw)), y_d=desired(pkw), theta_y=ty,
                            theta_w=tw, theta_v=tv, x=x, ax=ax)
        print(f"{name}: |Ax|={np.linalg.norm(ax):.6g}")


def make_assembly():
    out = {}
    for lvl in (3, 4):
        for what in ("mass", "poisson", "convdiff", "partial_mass", "lumped"):
            kw = dict(eps=0.02) if what == "convdiff" else {}
            obs = (0.0, 0.5, 0.0, 1.0) if what == "partial_mass" else None
            out[f"{what}_l{lvl}"] = ref.assemble9(what, lvl, obs=obs, **kw)
    np.savez_compressed(os.path.join(HERE, "assembly.npz"), **out)
    print("assembly: ", len(out), "operators")


if __name__ == "__main__":
    if len(sys.argv) > 1:
        make_ipm(tuple(sys.argv[1:]))
    else:
        make_assembly()
        make_kkt()
        make_ipm()
