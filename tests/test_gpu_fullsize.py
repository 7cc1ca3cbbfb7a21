"""Parity at BASELINE-scale sizes against the live reference (oracle/_ref, run
on the GPU box's CPU in the same test), bar of BASELINE.json's north_star:
u, y and J to 1e-8, Newton count +-1, zero count and active sets exact.

* C2: one (alpha, beta) cell at the full 513^2 size, gmres-pt (the reference
  default) and minres-pd (BASELINE's "same problem as C1");
* C4 convection-diffusion at 257^2 (GMRES(30));
* C5 heat with block-diagonal MINRES at 65^2 x 64 steps against the
  reference-class composition;
* C3 with the reference's cap (linear_maxit 200) at 129^2 through the default
  smoother (colour sweeps until the first capped solve, lexicographic after),
  Krylov counts equal to the reference's;
* the faithful preconditioners (lexicographic smoother) P_D, P_T, P_Pi
  applied once against the reference classes at 1e-11;
* GMRES(m) restarts: the device solve against a numpy restatement of
  restarted right-preconditioned GMRES (krylov.cpp:133-212 per cycle) over the
  device's own operator and preconditioner."""
import numpy as np
import pytest

from conftest import rel
from test_gpu_parity import active_sets

pytestmark = pytest.mark.gpu


def _kw(c, y_d=None):
    kw = dict(alpha=c.alpha, beta=c.beta, y_d=c.y_d() if y_d is None else y_d, u_a=c.u_a,
              u_b=c.u_b)
    if c.pde == "convdiff":
        kw["eps"] = c.eps
    if c.pde == "heat":
        kw["tau"] = c.tau
    if c.y_a is not None:
        kw.update(y_a=c.y_a, y_b=c.y_b)
    return kw


def _solve_both(oc, ctx, refmod, c, solver, ref_solver=None, **params):
    kw = _kw(c)
    rkw = dict(kw)
    okw = dict(kw)
    if c.obs is not None:
        rkw["obs"] = c.obs
        okw["observation"] = c.obs
    R = refmod.RefProblem(c.pde, c.level, **rkw)
    rr = R.solve(ref_solver or solver, sigma=c.sigma, **params)
    qp = oc.QpProblem(oc.ControlProblem(pde=c.pde, **okw), oc.Grid(c.level), ctx)
    r = oc.ipm_solve(qp, oc.IpmParams(sigma=c.sigma, solver=solver,
                                      gmres_restart=c.gmres_restart, **params))
    return r, rr


def _check(r, rr, c, counts=False):
    assert r.stats.converged
    assert abs(r.stats.nli - rr.nli) <= 1
    assert rel(r.u, rr.u) <= 1e-8, rel(r.u, rr.u)
    assert rel(r.state.y, rr.y) <= 1e-8, rel(r.state.y, rr.y)
    assert abs(r.objective - rr.objective) <= 1e-8 * abs(rr.objective)
    assert int((np.abs(r.u) < 1e-2).sum()) == int((np.abs(rr.u) < 1e-2).sum())
    for a, b in zip(active_sets(r.u, c.u_a, c.u_b), active_sets(rr.u, c.u_a, c.u_b)):
        assert np.array_equal(a, b)
    if c.y_a is not None:
        span = c.y_b - c.y_a
        assert np.array_equal(r.state.y - c.y_a < 1e-2 * span, rr.y - c.y_a < 1e-2 * span)
        assert np.array_equal(c.y_b - r.state.y < 1e-2 * span, c.y_b - rr.y < 1e-2 * span)
    if counts:
        assert [i.lin_iters for i in r.stats.iterations[1:]] == \
            [d["lin_iters"] for d in rr.records[1:]]


@pytest.mark.parametrize("solver", ["gmres-pt", "minres-pd"])
def test_c2_cell_full_size(oc, ctx, refmod, solver):
    from paper_1806_05896_b200 import configs

    c = configs.C2_CELLS[4]  # alpha 1e-4, beta 1e-3 at 513^2
    r, rr = _solve_both(oc, ctx, refmod, c, solver)
    _check(r, rr, c)


def test_c4_level8(oc, ctx, refmod):
    from paper_1806_05896_b200 import configs

    c = configs.C4.with_level(8)
    r, rr = _solve_both(oc, ctx, refmod, c, "gmres-pt")
    _check(r, rr, c)


def test_c5_minres_level6_nt64(oc, ctx, refmod):
    from paper_1806_05896_b200 import configs

    c = configs.C5.with_level(6, tau=1.0 / 64)
    r, rr = _solve_both(oc, ctx, refmod, c, "minres-pd", ref_solver="heat-minres-pd")
    _check(r, rr, c)


def test_c3_capped_level7_default_smoother(oc, ctx, refmod):
    from paper_1806_05896_b200 import configs

    c = configs.C3.with_level(7)
    r, rr = _solve_both(oc, ctx, refmod, c, "gmres-ppi", linear_maxit=200)
    assert any(d["lin_iters"] == 200 for d in rr.records[1:])  # the capped regime
    assert r.lex_from >= 1
    _check(r, rr, c, counts=True)


@pytest.mark.parametrize("kind", ["pd", "pt", "ppi"])
def test_lex_preconditioner_apply_matches_reference(oc, ctx, refmod, kind):
    from paper_1806_05896_b200 import configs

    level = 6
    n = ((1 << level) - 1) ** 2
    rng = np.random.default_rng(5)
    if kind == "ppi":
        c = configs.C3.with_level(level)
        kw = _kw(c)
        rkw = dict(kw, obs=c.obs)
        okw = dict(kw, observation=c.obs)
        ty = rng.uniform(0.1, 10.0, n)
    else:
        c = configs.C1
        kw = _kw(c)
        rkw, okw = kw, kw
        ty = None
    tw, tv = rng.uniform(0.01, 100.0, (2, n))
    R = refmod.RefProblem("poisson", level, **rkw)
    R.precond_setup(ty if ty is not None else np.zeros(n), tw, tv)
    qp = oc.build_qp(oc.ControlProblem(**okw), oc.Grid(level), ctx)
    qp.precond_setup(oc.ThetaBlocks(ty, tw, tv),
                     oc.IpmParams(solver={"pd": "minres-pd", "pt": "gmres-pt",
                                          "ppi": "gmres-ppi"}[kind], smoother="lex"))
    r = rng.uniform(-1, 1, 4 * n)
    assert rel(qp.precond_apply(kind, r), R.precond_apply(kind, r)) <= 1e-11


def _gmres_restarted(A, P, b, m, tol, maxit):
    """Right-preconditioned GMRES(m) (krylov.cpp:133-212 per cycle, restarted
    from the current iterate with r0 = b - A x); the stopping test is the true
    relative residual ||b - A x|| / ||b|| after every iteration."""
    bnorm = np.linalg.norm(b)
    x = np.zeros_like(b)
    total = 0
    while total < maxit:
        r0 = b - A(x) if total else b.copy()
        beta = np.linalg.norm(r0)
        V, Z, H, cs, sn, g = [r0 / beta], [], [], [], [], [beta]
        xb = x.copy()
        for j in range(min(m, maxit - total)):
            Z.append(P(V[j]))
            w = A(Z[-1])
            h = np.zeros(j + 2)
            for i in range(j + 1):
                h[i] = w @ V[i]
                w = w - h[i] * V[i]
            hn = np.linalg.norm(w)
            for i in range(j):
                t = cs[i] * h[i] + sn[i] * h[i + 1]
                h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1]
                h[i] = t
            rr = np.hypot(h[j], hn)
            cs.append(h[j] / rr)
            sn.append(hn / rr)
            h[j] = rr
            g.append(-sn[-1] * g[-1])
            g[j] *= cs[-1]
            H.append(h)
            V.append(w / hn)
            k = j + 1
            y = np.zeros(k)
            for i in range(k - 1, -1, -1):
                y[i] = (g[i] - sum(H[q][i] * y[q] for q in range(i + 1, k))) / H[i][i]
            x = xb + sum(y[i] * Z[i] for i in range(k))
            total += 1
            if np.linalg.norm(b - A(x)) / bnorm <= tol:
                return x, total
    return x, total


@pytest.mark.parametrize("m", [2, 3])
def test_gmres_restart_matches_restated_fgmres(oc, ctx, m):
    from paper_1806_05896_b200 import configs

    c = configs.C4.with_level(5)
    n = c.n
    qp = oc.build_qp(oc.ControlProblem(pde="convdiff", **_kw(c)), oc.Grid(c.level), ctx)
    rng = np.random.default_rng(2)
    th = oc.ThetaBlocks(None, *rng.uniform(0.1, 10.0, (2, n)))
    prm = oc.IpmParams(solver="gmres-pt", gmres_restart=m, smoother="color4")
    r1, r2, r3 = rng.uniform(-1, 1, n), rng.uniform(-1, 1, 2 * n), rng.uniform(-1, 1, n)
    dy, dz, dp, rep = qp.newton_solve(th, r1, r2, r3, prm)
    assert rep.converged and rep.iterations > m  # at least one restart ran
    # the restatement over the device's own KKT operator and (same) preconditioner
    qp.precond_setup(th, prm)
    A = lambda v: qp.kkt_apply(th, v)  # noqa: E731
    P = lambda v: qp.precond_apply("pt", v)  # noqa: E731
    b = np.r_[r1, r2, r3]
    x, its = _gmres_restarted(A, P, b, m, 1e-10, 200)
    assert its == rep.iterations
    assert rel(np.r_[dy, dz, dp], x) <= 1e-8
    # restart >= iterations is the full GMRES, bit for bit
    full = qp.newton_solve(th, r1, r2, r3, oc.IpmParams(solver="gmres-pt", smoother="color4"))
    big = qp.newton_solve(th, r1, r2, r3, oc.IpmParams(solver="gmres-pt", smoother="color4",
                                                       gmres_restart=200))
    for a, b_ in zip(full[:3], big[:3]):
        assert np.array_equal(a, b_)
