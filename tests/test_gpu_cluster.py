"""Cluster-resident multigrid bottom (k_mg_cluster.cu): the dense operator of
the V-cycle below level 5 and the whole-solve level-8 variant used by the heat
time blocks, each against the launch-per-level path on the same data."""
import dataclasses

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


@pytest.fixture()
def lib():
    from paper_1806_05896_b200 import _lib

    L = _lib.load()
    yield L
    _lib.check(L.oc_set_tuning(b"cluster_bottom", 1))
    _lib.check(L.oc_set_tuning(b"cluster_top8", 1))


def _tune(lib, name, value):
    from paper_1806_05896_b200 import _lib

    _lib.check(lib.oc_set_tuning(name, value))


@pytest.mark.parametrize("ell", [6, 7, 8])
def test_cluster_bottom_matches_single_cta_levels(oc, ctx, lib, ell):
    """Levels <= 7 in the 16-CTA cluster (levels <= 4 as one dense operator)
    give the V-cycle of the single-CTA bottom up to rounding."""
    L = oc.assemble9("poisson", ell)
    L[4] += 1.0
    b = np.random.default_rng(ell).uniform(-1, 1, L.shape[1])
    out = {}
    for cb in (0, 1):
        _tune(lib, b"cluster_bottom", cb)
        mg = oc.MgHierarchy(L, ell, ctx=ctx)
        out[cb] = [mg.solve(b, cyc, 5, 5) for cyc in (1, 3)]
    for a, c in zip(out[1], out[0]):
        assert rel(a, c) <= 1e-13


@pytest.mark.parametrize("pre,post", [(5, 5), (2, 3)])
def test_coarse_operator_is_symmetric_for_symmetric_levels(oc, ctx, lib, pre, post):
    """The levels <= 4 cycle (forward colours pre, backward post, exact level-2
    solve) of a symmetric hierarchy is a symmetric operator when pre == post;
    its columns are finite and it changes with the sweep counts."""
    from paper_1806_05896_b200 import _lib

    ell = 7
    L = oc.assemble9("poisson", ell)
    L[4] += 0.5
    mg = oc.MgHierarchy(L, ell, ctx=ctx)
    B = np.zeros((225, 225))
    _lib.check(lib.oc_debug_coarse_op(mg.h, pre, post, B.ctypes.data))
    assert np.isfinite(B).all() and np.abs(B).max() > 0
    asym = np.abs(B - B.T).max() / np.abs(B).max()
    if pre == post:
        assert asym <= 1e-13
    else:
        assert asym > 1e-8


@pytest.mark.parametrize("solver", ["gmres-pt", "minres-pd"])
def test_heat_level8_blocks_in_cluster_match_tiled(oc, ctx, lib, solver):
    """Heat time blocks (level 8, M + tau L + diag(mhat_k)) solved whole in the
    cluster kernel reproduce the tiled level-8 path bit for bit (MINRES needs
    the block solves to stay symmetric, which equality implies)."""
    from paper_1806_05896_b200 import configs

    c = dataclasses.replace(configs.C5, horizon=2 * configs.C5.tau)
    res = {}
    for top8 in (0, 1):
        _tune(lib, b"cluster_top8", top8)
        qp = oc.QpProblem(oc.ControlProblem(pde="heat", alpha=c.alpha, beta=c.beta, y_d=c.y_d(),
                                            u_a=c.u_a, u_b=c.u_b, tau=c.tau, horizon=c.horizon),
                          oc.Grid(c.level), ctx)
        res[top8] = oc.ipm_solve(qp, oc.IpmParams(sigma=c.sigma, solver=solver))
    a, b = res[1], res[0]
    assert a.stats.converged and b.stats.converged
    assert [i.lin_iters for i in a.stats.iterations] == [i.lin_iters for i in b.stats.iterations]
    assert rel(a.u, b.u) <= 1e-13 and rel(a.state.y, b.state.y) <= 1e-13


def test_colour_split_coefficients_give_identical_sweeps(oc, ctx, lib):
    """Tiled sweeps reading the colour-split copy of the off-diagonals (levels
    >= 511^2) reproduce the canonical-layout sweeps bit for bit."""
    ell = 10
    L = oc.assemble9("convdiff", ell, eps=0.02)
    L[4] += 1.0
    b = np.random.default_rng(7).uniform(-1, 1, L.shape[1])
    out = {}
    try:
        for v in (0, 1):
            _tune(lib, b"colour_split", v)
            mg = oc.MgHierarchy(L, ell, rediscretize=1, eps=0.02, ctx=ctx)
            out[v] = mg.solve(b, 2, 5, 5)
    finally:
        _tune(lib, b"colour_split", 1)
    assert np.array_equal(out[0], out[1])


@pytest.mark.parametrize("pde", ["poisson", "heat"])
def test_blocked_chebyshev_equals_stepwise(oc, ctx, lib, pde):
    """Five Chebyshev steps per launch (temporal blocking over 32x32 tiles)
    reproduce the one-step-per-launch semi-iteration bit for bit."""
    from paper_1806_05896_b200 import configs

    c = configs.C5 if pde == "heat" else configs.C1
    kw = dict(pde=pde, alpha=c.alpha, beta=c.beta, u_a=c.u_a, u_b=c.u_b)
    level = 6
    if pde == "heat":
        kw.update(tau=c.tau, horizon=3 * c.tau)
        kw["y_d"] = configs.sine_modes_spacetime(level, 3, c.tau, 42)
    else:
        kw["y_d"] = configs.sine_modes(level, seed=42)
    out = {}
    try:
        for v in (0, 1):
            _tune(lib, b"cheb_block", v)
            qp = oc.QpProblem(oc.ControlProblem(**kw), oc.Grid(level), ctx)
            out[v] = oc.ipm_solve(qp, oc.IpmParams(sigma=0.2, solver="gmres-pt")).u
    finally:
        _tune(lib, b"cheb_block", 1)
    assert np.array_equal(out[0], out[1])


@pytest.mark.parametrize("fuse", [0, 1])
def test_divergence_check_raises_with_and_without_fusion(oc, ctx, lib, fuse):
    """MgHierarchy::solve's residual-growth check (multigrid.cpp:141-157) on a
    tiled fine level, run by the cycle's last sweep launch (fuse_norm=1) or by
    its own launch (0): an indefinite operator without diagonal dominance
    (the Poisson stencil with centre -1: Gauss-Seidel diverges) raises the
    reference's runtime_error; a definite one does not."""
    from paper_1806_05896_b200 import _lib

    ell = 9
    b = np.random.default_rng(3).uniform(-1, 1, ((1 << ell) - 1) ** 2)
    try:
        _tune(lib, b"fuse_norm", fuse)
        good = oc.assemble9("poisson", ell)
        good[4] += 1.0
        oc.MgHierarchy(good, ell, ctx=ctx).solve(b, 3, 5, 5)
        bad = oc.assemble9("poisson", ell)
        bad[4] = -1.0
        with pytest.raises(_lib.OptconError, match="residual growth"):
            oc.MgHierarchy(bad, ell, ctx=ctx).solve(b, 3, 5, 5)
    finally:
        _tune(lib, b"fuse_norm", 1)


@pytest.mark.parametrize("knob", [b"fuse_norm", b"fuse_restrict", b"colour_split", b"cheb_block"])
def test_fusion_knobs_leave_solutions_bitwise_unchanged(oc, ctx, lib, knob):
    """Each kernel fusion (divergence check or residual restriction folded into
    the last sweep launch, colour-split coefficients, blocked Chebyshev) only
    regroups the same arithmetic: a C2-style solve at 513^2 with the knob off
    and on gives identical bits."""
    from paper_1806_05896_b200 import configs

    c = configs.C2_CELLS[4]
    out = {}
    try:
        for v in (0, 1):
            _tune(lib, knob, v)
            qp = oc.QpProblem(oc.ControlProblem(pde="poisson", alpha=c.alpha, beta=c.beta, y_d=c.y_d(),
                                                u_a=c.u_a, u_b=c.u_b), oc.Grid(c.level), ctx)
            r = oc.ipm_solve(qp, oc.IpmParams(sigma=c.sigma, solver=c.solver))
            out[v] = (r.u, [i.lin_iters for i in r.stats.iterations])
    finally:
        _tune(lib, knob, 1)
    assert np.array_equal(out[0][0], out[1][0]) and out[0][1] == out[1][1]


@pytest.mark.parametrize("cfg", ["C3@7", "C2"])
def test_persistent_mgs_bitwise_equal(oc, ctx, lib, cfg):
    """GMRES orthogonalisation in one persistent launch (w in shared memory,
    grid barrier between steps) against the launch-per-step sequence: same
    element-to-partial map and summation order, so identical bits — on C3's
    long P_Pi solves (j up to 200) and C2's short P_T solves (every column)."""
    from paper_1806_05896_b200 import configs

    name, _, lvl = cfg.partition("@")
    c = configs.C2_CELLS[4] if name == "C2" else configs.ALL[name].with_level(int(lvl))
    kw = dict(pde=c.pde, alpha=c.alpha, beta=c.beta, y_d=c.y_d(), u_a=c.u_a, u_b=c.u_b)
    if c.y_a is not None:
        kw.update(y_a=c.y_a, y_b=c.y_b)
    if c.obs is not None:
        kw["observation"] = c.obs
    out = {}
    try:
        for v in (0, 1):
            _tune(lib, b"mgs_persistent", v)
            qp = oc.QpProblem(oc.ControlProblem(**kw), oc.Grid(c.level), ctx)
            r = oc.ipm_solve(qp, oc.IpmParams(sigma=c.sigma, solver=c.solver))
            out[v] = (r.u, [i.lin_iters for i in r.stats.iterations])
    finally:
        _tune(lib, b"mgs_persistent", 8)
    if name == "C3":
        assert max(out[1][1]) > 8
    assert np.array_equal(out[0][0], out[1][0]) and out[0][1] == out[1][1]


@pytest.mark.parametrize("solver", ["minres-pd", "gmres-pt"])
def test_chained_heat_substitution_equals_per_block_launches(oc, ctx, lib, solver):
    """One chained cluster launch per substitution direction (right-hand side
    r_k + M x_{k-1} formed from the previous solution in shared memory,
    timedep.cpp:268-311) reproduces the per-block launches (k_rhs_plus_mass +
    one cluster launch per time block) bit for bit, Krylov counts included."""
    from paper_1806_05896_b200 import configs

    nt = 5
    c = dataclasses.replace(configs.C5, horizon=nt * configs.C5.tau)
    out = {}
    try:
        for v in (0, 1):
            _tune(lib, b"heat_chain", v)
            qp = oc.QpProblem(oc.ControlProblem(pde="heat", alpha=c.alpha, beta=c.beta, y_d=c.y_d(),
                                                u_a=c.u_a, u_b=c.u_b, tau=c.tau, horizon=c.horizon),
                              oc.Grid(c.level), ctx)
            l0 = oc.Context.launch_count()
            r = oc.ipm_solve(qp, oc.IpmParams(sigma=c.sigma, solver=solver))
            out[v] = (r.u, r.state.y, [i.lin_iters for i in r.stats.iterations],
                      oc.Context.launch_count() - l0)
    finally:
        _tune(lib, b"heat_chain", 1)
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
    assert out[0][2] == out[1][2]
    assert out[1][3] < out[0][3]  # the chained path really ran (fewer launches)


def test_tiled_heat_kkt_apply_equals_per_node_kernel(oc, ctx, lib):
    """The shared-memory heat KKT apply (k_kkt_heat_tiled) gives the bits of the
    per-node kernel on random x and Theta, first, interior and last time blocks
    included (their neighbour-block terms are skipped, not zeroed)."""
    from paper_1806_05896_b200 import configs

    level, nt = 6, 4
    c = configs.C5
    yd = configs.sine_modes_spacetime(level, nt, c.tau, 42)
    qp = oc.QpProblem(oc.ControlProblem(pde="heat", alpha=c.alpha, beta=c.beta, y_d=yd, u_a=c.u_a,
                                        u_b=c.u_b, tau=c.tau, horizon=nt * c.tau), oc.Grid(level), ctx)
    rng = np.random.default_rng(3)
    ny = qp.ny
    x = rng.standard_normal(4 * ny)
    th = oc.ThetaBlocks(theta_y=None, theta_w=rng.random(ny) + 0.1, theta_v=rng.random(ny) + 0.1)
    out = {}
    try:
        for v in (0, 1):
            _tune(lib, b"kkt_tiled", v)
            out[v] = np.array(qp.kkt_apply(th, x))
    finally:
        _tune(lib, b"kkt_tiled", 1)
    assert np.array_equal(out[0], out[1])


@pytest.mark.parametrize("lean,ell", [(0, 9), (2, 9), (3, 9), (3, 10)])
def test_lean_variable_sweeps_bitwise_equal(oc, ctx, lib, lean, ell):
    """Variable-coefficient tiled sweeps that stage 1/a_ii (0), read b in the
    colour passes too (2), or take their node records from a shared-memory ring
    filled by a producer warp's bulk copies (3) reproduce the default bits."""
    L = oc.assemble9("convdiff", ell, eps=0.02)
    L[4] += 1.0
    b = np.random.default_rng(11).uniform(-1, 1, L.shape[1])
    out = {}
    try:
        for v in (1, lean):
            _tune(lib, b"sweep_lean", v)
            mg = oc.MgHierarchy(L, ell, rediscretize=1, eps=0.02, ctx=ctx)
            out[v] = mg.solve(b, 2, 5, 5)
    finally:
        _tune(lib, b"sweep_lean", 1)
    assert np.array_equal(out[1], out[lean])
