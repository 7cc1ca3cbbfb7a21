"""Device component tests mirroring the reference's unit suites
(test_multigrid.cpp, test_krylov.cpp, test_precond.cpp): multigrid properties,
the 4-colour V-cycle against its numpy restatement, Chebyshev and the block
preconditioners against the reference, and the reference's error behaviour."""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def port():
    from oracle import port

    return port


def apply9(coef, x, level):
    nx = (1 << level) - 1
    X = x.reshape(nx, nx)
    out = np.zeros_like(X)
    P = np.pad(X, 1)
    for d in range(9):
        dx, dy = d % 3 - 1, d // 3 - 1
        out += coef[d].reshape(nx, nx) * P[1 + dy:1 + dy + nx, 1 + dx:1 + dx + nx]
    return out.reshape(-1)


# ------------------------------------------------------------------ multigrid
def test_mg_depth(oc, ctx):
    for ell in (3, 4, 5, 8):
        mg = oc.MgHierarchy(oc.assemble9("poisson", ell), ell, ctx=ctx)
        assert mg.depth() == ell - 2


def test_mg_galerkin_identity_is_rtp(oc, ctx, port):
    ell = 4
    n = 15 * 15
    ident = np.zeros((9, n))
    ident[4] = 1.0
    mg = oc.MgHierarchy(ident, ell, ctx=ctx)
    P = port.prolongation(ell)
    rp = (P.T @ P).toarray()
    got = port.to_csr(mg.level_matrix(1)).toarray()
    assert np.linalg.norm(got - rp) <= 1e-13


@pytest.mark.parametrize("what", ["poisson", "mass"])
def test_mg_galerkin_equals_assembled_coarse(oc, ctx, what):
    for ell in (4, 9):
        mg = oc.MgHierarchy(oc.assemble9(what, ell), ell, ctx=ctx)
        Lc = oc.assemble9(what, ell - 1)
        assert np.linalg.norm(mg.level_matrix(1) - Lc) <= 1e-12 * np.linalg.norm(Lc)


def test_mg_zero_rhs_gives_zero(oc, ctx):
    mg = oc.MgHierarchy(oc.assemble9("poisson", 8), 8, ctx=ctx)
    assert np.all(mg.solve(np.zeros(255 * 255)) == 0.0)


@pytest.mark.parametrize("ell", [5, 8, 10])
def test_mg_three_cycles_reduce_by_1e3(oc, ctx, ell):
    L = oc.assemble9("poisson", ell)
    mg = oc.MgHierarchy(L, ell, ctx=ctx)
    b = np.random.default_rng(3).uniform(-1, 1, L.shape[1])
    x = mg.solve(b, 3, 5, 5)
    assert np.linalg.norm(b - apply9(L, x, ell)) <= 1e-3 * np.linalg.norm(b)


def test_mg_diagonal_shift_converges_no_slower(oc, ctx):
    ell = 5
    L = oc.assemble9("poisson", ell)
    Ls = L.copy()
    Ls[4] += 50.0
    b = np.random.default_rng(5).uniform(-1, 1, L.shape[1])
    r0 = np.linalg.norm(b - apply9(L, oc.MgHierarchy(L, ell, ctx=ctx).solve(b), ell))
    r1 = np.linalg.norm(b - apply9(Ls, oc.MgHierarchy(Ls, ell, ctx=ctx).solve(b), ell))
    assert r1 <= r0 * (1 + 1e-12)


def test_mg_is_linear_and_spd(oc, ctx):
    ell = 6
    L = oc.assemble9("poisson", ell)
    rng = np.random.default_rng(11)
    L[4] += 10 ** rng.uniform(-2, 1, L.shape[1])
    mg = oc.MgHierarchy(L, ell, ctx=ctx)
    u, v = rng.uniform(-1, 1, (2, L.shape[1]))
    lhs = mg.solve(-0.8 * u + 2.4 * v)
    rhs = -0.8 * mg.solve(u) + 2.4 * mg.solve(v)
    assert np.max(np.abs(lhs - rhs) / (1 + np.abs(lhs))) <= 1e-12
    for _ in range(3):
        x, y = rng.uniform(-1, 1, (2, L.shape[1]))
        vx, vy = mg.solve(x), mg.solve(y)
        assert x @ vx > 0
        assert abs(y @ vx - x @ vy) <= 1e-10 * abs(x @ vy)


@pytest.mark.parametrize("ell", [4, 6, 7])
def test_mg_matches_color4_restatement(oc, ctx, port, ell):
    # the device V-cycle is exactly the 4-colour algorithm restated in numpy
    L = oc.assemble9("poisson", ell)
    rng = np.random.default_rng(ell)
    L[4] += 10 ** rng.uniform(-3, 0, L.shape[1])
    b = rng.uniform(-1, 1, L.shape[1])
    x_gpu = oc.MgHierarchy(L, ell, ctx=ctx).solve(b)
    x_np = port.MgHierarchy(port.to_csr(L), ell, smoother="color4").solve(b)
    assert rel(x_gpu, x_np) <= 1e-11


def test_mg_smoother_sweep_matches_restatement(oc, ctx, port):
    ell = 7
    L = oc.assemble9("convdiff", ell, eps=0.02)
    rng = np.random.default_rng(1)
    b, x0 = rng.uniform(-1, 1, (2, L.shape[1]))
    mg = oc.MgHierarchy(L, ell, ctx=ctx)
    A = port.to_csr(L)
    for fwd in (True, False):
        assert rel(mg.smooth(b, x0, fwd), port.gs_color4(A, b, x0, fwd)) <= 1e-13


@pytest.mark.parametrize("eps", [1e-1, 1e-2])
def test_mg_rediscretized_convdiff(oc, ctx, eps):
    ell = 5
    L = oc.assemble9("convdiff", ell, eps=eps)
    mg = oc.MgHierarchy(L, ell, rediscretize=1, eps=eps, ctx=ctx)
    b = np.random.default_rng(13).uniform(-1, 1, L.shape[1])
    x = mg.solve(b, 3, 5, 5)
    assert np.linalg.norm(b - apply9(L, x, ell)) <= 1e-4 * np.linalg.norm(b)


def test_mg_rediscretized_keeps_perturbation(oc, ctx, port):
    # test_multigrid.cpp:153-175: coarse = rediscretised base + R diag P
    ell, eps = 4, 1e-2
    L = oc.assemble9("convdiff", ell, eps=eps)
    d = 10 ** np.random.default_rng(17).uniform(-2, 0, L.shape[1])
    A = L.copy()
    A[4] += d
    mg = oc.MgHierarchy(A, ell, rediscretize=1, eps=eps, ctx=ctx)
    P = port.prolongation(ell)
    import scipy.sparse as sp

    expect = port.to_csr(oc.assemble9("convdiff", ell - 1, eps=eps)).toarray() + \
        (P.T @ sp.diags(d) @ P).toarray()
    got = port.to_csr(mg.level_matrix(1)).toarray()
    assert np.linalg.norm(got - expect) <= 1e-12 * np.linalg.norm(expect)


def test_mg_rejects_small_levels(oc, ctx):
    with pytest.raises(oc.OptconInvalidArgument):
        oc.MgHierarchy(oc.assemble9("poisson", 2), 2, ctx=ctx)


# ------------------------------------------------------------------ Chebyshev
def test_chebyshev_matches_reference(oc, ctx, refmod):
    rng = np.random.default_rng(5)
    for level, scale, extra in [(4, 1.0, None), (6, 0.3, True), (8, 1.0 / 128, None)]:
        n = ((1 << level) - 1) ** 2
        e = 10 ** rng.uniform(-6, -3, n) if extra else None
        b = rng.uniform(-1, 1, n)
        a = oc.cheb_apply(level, scale, e, 20, b, ctx)
        r = refmod.cheb_apply(level, scale, e, 20, b)
        assert rel(a, r) <= 1e-13


def test_chebyshev_error_bound(oc, ctx, port):
    # test_krylov.cpp:131-163: <= 2e-6 after 20 steps
    level = 5
    M = port.to_csr(port.assemble("mass", level))
    n = M.shape[0]
    rng = np.random.default_rng(7)
    e = 10 ** rng.uniform(-3, 0, n) * M.diagonal().max()
    b = rng.uniform(-1, 1, n)
    x = oc.cheb_apply(level, 1.0, e, 20, b, ctx)
    import scipy.sparse.linalg as spla

    xs = spla.spsolve((M + __import__("scipy.sparse", fromlist=["diags"]).diags(e)).tocsc(), b)
    assert np.linalg.norm(x - xs) <= 2e-6 * np.linalg.norm(xs)


# ----------------------------------------------------------- preconditioners
def random_theta(n, rng, with_state):
    tw = 10 ** rng.uniform(-2, 2, n)
    tv = 10 ** rng.uniform(-2, 2, n)
    ty = 10 ** rng.uniform(-3, 0, n) if with_state else None
    return ty, tw, tv


@pytest.mark.parametrize("pde", ["poisson", "convdiff"])
def test_block_preconditioners_against_reference(oc, ctx, refmod, pde):
    from paper_1806_05896_b200 import configs

    level = 6
    n = 63 * 63
    yd = configs.sine_modes(level)
    kw = dict(alpha=1e-2, beta=1e-3, y_d=yd, u_a=-2.0, u_b=2.0)
    if pde == "convdiff":
        kw["eps"] = 0.02
    R = refmod.RefProblem(pde, level, **kw)
    qp = oc.build_qp(oc.ControlProblem(pde=pde, **kw), oc.Grid(level), ctx)
    rng = np.random.default_rng(3)
    ty, tw, tv = random_theta(n, rng, False)
    R.precond_setup(np.zeros(n), tw, tv)
    r = rng.uniform(-1, 1, 4 * n)
    for kind, solver in (("pd", "minres-pd"), ("pt", "gmres-pt")):
        qp.precond_setup(oc.ThetaBlocks(None, tw, tv), oc.IpmParams(solver=solver))
        a = qp.precond_apply(kind, r)
        b = R.precond_apply(kind, r)
        # Chebyshev and 2x2 blocks: same algorithm -> rounding
        assert rel(a[:n], b[:n]) <= 1e-13
        assert rel(a[n:3 * n], b[n:3 * n]) <= 1e-14
        # Schur block: multigrid with the 4-colour smoother vs lexicographic GS
        assert rel(a[3 * n:], b[3 * n:]) <= 5e-3


def test_schur_approximation_is_spd_for_symmetric_l(oc, ctx):
    from paper_1806_05896_b200 import configs

    level = 7
    n = 127 * 127
    qp = oc.build_qp(oc.ControlProblem(alpha=1e-2, beta=1e-3, y_d=configs.sine_modes(level),
                                       u_a=-2.0, u_b=2.0), oc.Grid(level), ctx)
    rng = np.random.default_rng(9)
    ty, tw, tv = random_theta(n, rng, False)
    qp.precond_setup(oc.ThetaBlocks(None, tw, tv), oc.IpmParams(solver="minres-pd"))
    x, y = rng.uniform(-1, 1, (2, n))
    sx, sy = qp.schur_apply(x), qp.schur_apply(y)
    assert x @ sx > 0
    assert abs(y @ sx - x @ sy) <= 1e-9 * abs(x @ sy)


def test_permuted_preconditioner_against_restatement(oc, ctx, port):
    # P_Pi with the same (4-colour) smoother in the numpy restatement
    from paper_1806_05896_b200 import configs

    level = 5
    n = 31 * 31
    yd = configs.sine_modes(level)
    obs = (0.0, 0.5, 0.0, 1.0)
    qp = oc.build_qp(oc.ControlProblem(alpha=1e-4, beta=1e-3, y_d=yd, u_a=-2.0, u_b=2.0,
                                       y_a=-0.2, y_b=0.3, observation=obs), oc.Grid(level), ctx)
    Q = port.Qp(level=level, pde="poisson", alpha=1e-4, beta=1e-3, y_d=yd, u_a=-2.0, u_b=2.0,
                y_a=-0.2, y_b=0.3, obs=obs, smoother="color4")
    rng = np.random.default_rng(21)
    ty, tw, tv = random_theta(n, rng, True)
    qp.precond_setup(oc.ThetaBlocks(ty, tw, tv), oc.IpmParams(solver="gmres-ppi"))
    Q.setup(ty, tw, tv, "ppi")
    r = rng.uniform(-1, 1, 4 * n)
    assert rel(qp.precond_apply("ppi", r), Q.precond("ppi", r)) <= 1e-11


# ------------------------------------------------------------------- errors
def test_reference_error_behaviour(oc, ctx):
    from paper_1806_05896_b200 import configs

    level = 4
    yd = configs.sine_modes(level)
    part = oc.build_qp(oc.ControlProblem(alpha=1e-4, beta=1e-3, y_d=yd, u_a=-2.0, u_b=1.5,
                                         observation=(0.2, 0.4, 0.4, 0.9)), oc.Grid(level), ctx)
    n = part.ny
    th = oc.ThetaBlocks(None, np.ones(n), np.ones(n))
    with pytest.raises(oc.OptconInvalidArgument, match="minres-pd requires a nonsingular"):
        part.newton_solve(th, np.ones(n), np.ones(2 * n), np.ones(n), oc.IpmParams(solver="minres-pd"))
    with pytest.raises(oc.OptconInvalidArgument, match="gmres-pt requires a nonsingular"):
        part.newton_solve(th, np.ones(n), np.ones(2 * n), np.ones(n), oc.IpmParams(solver="gmres-pt"))
    r = oc.ipm_solve(part, oc.IpmParams(solver="gmres-ppi", sigma=0.25))
    assert r.stats.converged and all(i.lin_converged for i in r.stats.iterations[1:])
    with pytest.raises(oc.OptconInvalidArgument, match="sigma must lie in"):
        oc.ipm_solve(part, oc.IpmParams(sigma=1.5, solver="gmres-ppi"))
    with pytest.raises(oc.OptconInvalidArgument, match="alpha0 must lie in"):
        oc.ipm_solve(part, oc.IpmParams(alpha0=1.0, solver="gmres-ppi"))
    with pytest.raises(oc.OptconInvalidArgument, match="control bounds"):
        oc.build_qp(oc.ControlProblem(alpha=1e-4, beta=1e-3, y_d=yd, u_a=0.5, u_b=1.5),
                    oc.Grid(level), ctx)
    with pytest.raises(oc.OptconInvalidArgument, match="alpha must be positive"):
        oc.build_qp(oc.ControlProblem(alpha=0.0, beta=1e-3, y_d=yd, u_a=-1.0, u_b=1.5),
                    oc.Grid(level), ctx)
    with pytest.raises(oc.OptconInvalidArgument, match="tau must divide"):
        oc.assemble_spacetime(oc.ControlProblem(pde="heat", tau=0.3, alpha=1e-3, beta=0.0,
                                                y_d=yd, u_a=-1.0, u_b=1.0), oc.Grid(level), ctx)
    heat = oc.assemble_spacetime(oc.ControlProblem(pde="heat", tau=0.25, alpha=1e-3, beta=0.0,
                                                   y_d=yd, u_a=-1.0, u_b=1.0), oc.Grid(level), ctx)
    with pytest.raises(oc.OptconInvalidArgument, match="unsupported solver kind"):
        oc.ipm_solve(heat, oc.IpmParams(solver="gmres-ppi"))


def test_sparsity_monotone_in_beta(oc, ctx):
    # test_ipm.cpp:364-380
    from paper_1806_05896_b200 import configs

    level = 4
    last = 101.0
    for beta in (1e-1, 1e-2, 1e-3):
        qp = oc.build_qp(oc.ControlProblem(alpha=1e-2, beta=beta, y_d=configs.sin_sin(level),
                                           u_a=-2.0, u_b=1.5), oc.Grid(level), ctx)
        r = oc.ipm_solve(qp, oc.IpmParams(eps_p=1e-10, eps_d=1e-10, eps_c=1e-10,
                                          max_iterations=40))
        assert r.stats.converged
        assert r.sparsity.percent_below_threshold <= last + 1e-9
        last = r.sparsity.percent_below_threshold


def test_convdiff_aggressive_sigma_nli(oc, ctx):
    # test_ipm.cpp:450-472: eps 1e-2, sigma 0.4 -> NLI 16
    level = 6
    nx = 63
    h = 1 / 64
    idx = np.arange(nx * nx)
    x, y = (idx % nx + 1) * h, (idx // nx + 1) * h
    yd = np.exp(-64.0 * ((x - 0.5) ** 2 + (y - 0.5) ** 2))
    qp = oc.build_qp(oc.ControlProblem(pde="convdiff", eps=1e-2, alpha=1e-4, beta=1e-3, y_d=yd,
                                       u_a=-2.0, u_b=1.5), oc.Grid(level), ctx)
    r = oc.ipm_solve(qp, oc.IpmParams(sigma=0.4))
    assert r.stats.converged and r.stats.nli == 16


# ------------------------------------------------------------ device assembly
@pytest.mark.parametrize("what,kw", [("mass", {}), ("poisson", {}), ("convdiff", {"eps": 0.1}),
                                     ("convdiff", {"eps": 0.02}),
                                     ("partial_mass", {"obs": [0.0, 0.5, 0.0, 1.0]})])
@pytest.mark.parametrize("ell", [3, 6, 9])
def test_device_assembly_matches_host_assembly(oc, ctx, what, kw, ell):
    # same element formulas, same accumulation order, no FMA contraction: equal
    # to the host assembly up to the last ulp of hypot in the SUPG parameter
    h = oc.assemble9(what, ell, **kw)
    d = oc.assemble9_device(what, ell, ctx=ctx, **kw)
    if what == "convdiff":
        assert np.max(np.abs(d - h)) <= 4e-16 * np.max(np.abs(h))
    else:
        assert np.array_equal(d, h)
