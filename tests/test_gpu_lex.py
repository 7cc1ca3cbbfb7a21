"""Faithful mode: the reference's lexicographic Gauss-Seidel smoother
(gauss_seidel_sweep, multigrid.cpp:44-66) on the device as a skewed wavefront
(k_mg_lex.cu, lex_gs.cuh). Sweeps and V-cycles are checked against the
reference order (numpy triangular-solve restatement / the reference library),
and whole IPM solves against the reference's golden outputs, including C3 in
the capped-Krylov regime where only the reference smoother reproduces the
reference's answer."""
import numpy as np
import pytest

from conftest import load_golden, rel
from test_gpu_parity import active_sets, qp_from_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def port():
    from oracle import port

    return port


def operator(oc, kind, ell, seed):
    rng = np.random.default_rng(seed)
    if kind == "poisson+diag":
        A = oc.assemble9("poisson", ell)
        A[4] += 10 ** rng.uniform(-3, 0, A.shape[1])
    else:  # nonsymmetric variable coefficients (SUPG convection-diffusion)
        A = oc.assemble9("convdiff", ell, eps=0.02)
    return A


@pytest.mark.parametrize("ell", [3, 5, 6, 7, 9])
@pytest.mark.parametrize("kind", ["poisson+diag", "convdiff"])
def test_lex_sweep_is_reference_order(oc, ctx, port, ell, kind):
    # one forward and one backward sweep from a random iterate: the device
    # result equals the sequential sweep up to rounding (reassociated sum)
    A = operator(oc, kind, ell, ell)
    rng = np.random.default_rng(100 + ell)
    b, x0 = rng.uniform(-1, 1, (2, A.shape[1]))
    mg = oc.MgHierarchy(A, ell, ctx=ctx, smoother="lex")
    Acsr = port.to_csr(A)
    for fwd in (True, False):
        got = mg.smooth(b, x0, fwd)
        want = port.gs_lex(Acsr, b, x0, fwd)
        assert rel(got, want) <= 1e-12, (fwd, rel(got, want))


@pytest.mark.parametrize("ell", [3, 6, 7, 8, 10])
@pytest.mark.parametrize("kind", ["poisson+diag", "convdiff"])
def test_lex_sweep_bitwise_equals_reference(oc, ctx, refmod, ell, kind):
    # the node update follows multigrid.cpp:49-60 operation by operation
    # (ascending columns, separate multiply and subtract, s / a_ii correctly
    # rounded): a sweep equals the reference library's gauss_seidel_sweep
    # bit for bit, forward and backward, on every level size (one band,
    # several bands, 32 bands at 1023^2)
    A = operator(oc, kind, ell, ell)
    rng = np.random.default_rng(200 + ell)
    b, x0 = rng.uniform(-1, 1, (2, A.shape[1]))
    mg = oc.MgHierarchy(A, ell, ctx=ctx, smoother="lex")
    for fwd in (True, False):
        got = mg.smooth(b, x0, fwd)
        want = refmod.gs_sweep(ell, A, b, x0, fwd)
        assert np.array_equal(got, want), (fwd, rel(got, want), int((got != want).sum()))


def test_lex_division_is_correctly_rounded(oc, ctx):
    # the update's quotient (RN(1/d) product + one Markstein correction) equals
    # the IEEE division on random operands over many binades and on the
    # solver's own kind of data (diagonals of L + diag, coarse Galerkin rows)
    import ctypes as C

    from paper_1806_05896_b200 import _lib

    rng = np.random.default_rng(11)
    n = 1 << 22
    cases = [
        (rng.standard_normal(n) * 10.0 ** rng.uniform(-30, 30, n),
         rng.standard_normal(n) * 10.0 ** rng.uniform(-30, 30, n)),
        (rng.uniform(-1, 1, n), 8.0 / 3.0 + 10.0 ** rng.uniform(-6, 2, n)),
        (rng.uniform(-1, 1, n) * 1e-9, rng.uniform(0.1, 100.0, n)),
        (rng.uniform(1, 2, n), rng.uniform(1, 2, n)),  # one binade: rounding-boundary stress
    ]
    L = _lib.load()
    for num, den in cases:
        num = np.ascontiguousarray(num)
        den = np.ascontiguousarray(den)
        bad = C.c_ulonglong(0)
        _lib.check(L.oc_debug_lex_div(ctx.h, num.ctypes.data, den.ctypes.data, n, C.byref(bad)))
        assert bad.value == 0


def test_lex_sweeps_repeat_bitwise(oc, ctx):
    # the mailbox is restored after every sweep: repeated sweeps are identical
    ell = 8
    A = oc.assemble9("poisson", ell)
    b = np.random.default_rng(3).uniform(-1, 1, A.shape[1])
    mg = oc.MgHierarchy(A, ell, ctx=ctx, smoother="lex")
    x0 = np.zeros(A.shape[1])
    first = [mg.smooth(b, x0, True), mg.smooth(b, x0, False)]
    for _ in range(3):
        assert np.array_equal(mg.smooth(b, x0, True), first[0])
        assert np.array_equal(mg.smooth(b, x0, False), first[1])


@pytest.mark.parametrize("ell,kind,sweeps", [(7, "poisson", 5), (8, "convdiff", 5), (9, "convdiff", 7),
                                             (9, "poisson", 2), (10, "convdiff", 5)])
def test_pipelined_lex_batches_equal_sequential_sweeps(oc, ctx, ell, kind, sweeps):
    """The sweeps of a smoothing phase launched as a pipelined batch (one launch
    per sweep on its own stream, paced by per-band progress counters, one
    mailbox set each; more than five sweeps split into batches) give the bits of
    the one-after-the-other launches, forward and backward, repeatedly."""
    from paper_1806_05896_b200 import _lib

    lib = _lib.load()
    A = oc.assemble9(kind, ell, eps=0.02) if kind == "convdiff" else oc.assemble9(kind, ell)
    A[4] += 1.0
    b = np.random.default_rng(13).uniform(-1, 1, A.shape[1])
    out = {}
    try:
        for v in (0, 1, 1):
            _lib.check(lib.oc_set_tuning(b"lex_pipeline", v))
            mg = oc.MgHierarchy(A, ell, ctx=ctx, smoother="lex")
            x = mg.solve(b, 2, sweeps, sweeps)
            if v in out:
                assert np.array_equal(out[v], x)  # rerun: mailboxes and counters were left clean
            out[v] = x
            mg.close()
    finally:
        _lib.check(lib.oc_set_tuning(b"lex_pipeline", 1))
    assert np.array_equal(out[0], out[1])


@pytest.mark.parametrize("ell", [4, 6, 7, 9])
def test_lex_vcycle_matches_reference_library(oc, ctx, refmod, ell):
    A = operator(oc, "poisson+diag", ell, 7 + ell)
    b = np.random.default_rng(ell).uniform(-1, 1, A.shape[1])
    x_gpu = oc.MgHierarchy(A, ell, ctx=ctx, smoother="lex").solve(b, 3, 5, 5)
    x_ref = refmod.RefMg(ell, A).solve(b, 3, 5, 5)
    assert rel(x_gpu, x_ref) <= 1e-11


def test_lex_rediscretized_convdiff_matches_reference_library(oc, ctx, refmod):
    ell, eps = 7, 0.02
    A = oc.assemble9("convdiff", ell, eps=eps)
    b = np.random.default_rng(21).uniform(-1, 1, A.shape[1])
    x_gpu = oc.MgHierarchy(A, ell, rediscretize=1, eps=eps, ctx=ctx, smoother="lex").solve(b)
    x_ref = refmod.RefMg(ell, A, rediscretize_convdiff=True, eps=eps).solve(b)
    assert rel(x_gpu, x_ref) <= 1e-11


def test_lex_differs_from_color4(oc, ctx):
    # sanity: the two smoothers are different algorithms
    ell = 6
    A = oc.assemble9("poisson", ell)
    b = np.random.default_rng(5).uniform(-1, 1, A.shape[1])
    x_lex = oc.MgHierarchy(A, ell, ctx=ctx, smoother="lex").solve(b, 1, 1, 1)
    x_c4 = oc.MgHierarchy(A, ell, ctx=ctx).solve(b, 1, 1, 1)
    assert rel(x_lex, x_c4) > 1e-6


def test_unknown_smoother_rejected(oc, ctx):
    with pytest.raises(oc.OptconInvalidArgument):
        oc.MgHierarchy(oc.assemble9("poisson", 4), 4, ctx=ctx, smoother="jacobi")
    g = load_golden("smoke_l5")
    qp = qp_from_golden(oc, ctx, g)
    with pytest.raises(oc.OptconInvalidArgument):
        oc.ipm_solve(qp, oc.IpmParams(smoother=7))


LEX_GOLDEN = ["known_answer_l6", "c1_l6_gmres", "c1_l6_minres", "c3_l5", "c3_l6_capped",
              "c3_l6_maxit200", "c4_l6", "c5_l5_nt16"]


@pytest.mark.parametrize("name", LEX_GOLDEN)
def test_lex_ipm_matches_reference_golden(oc, ctx, name):
    g = load_golden(name)
    qp = qp_from_golden(oc, ctx, g)
    s = g["meta"]["solve"]
    r = oc.ipm_solve(qp, oc.IpmParams(sigma=s["sigma"], solver=s["solver"], smoother="lex",
                                      linear_maxit=s.get("linear_maxit", 200)))
    assert r.stats.converged
    assert abs(r.stats.nli - int(g["nli"])) <= 1
    assert rel(r.u, g["u"]) <= 1e-8, rel(r.u, g["u"])
    assert rel(r.state.y, g["y"]) <= 1e-8
    J = float(g["objective"])
    assert abs(r.objective - J) <= 1e-8 * abs(J)
    assert int((np.abs(r.u) < 1e-2).sum()) == int((np.abs(g["u"]) < 1e-2).sum())
    pk = g["meta"]["problem"]
    for a, b in zip(active_sets(r.u, pk["u_a"], pk["u_b"]), active_sets(g["u"], pk["u_a"], pk["u_b"])):
        assert np.array_equal(a, b)
    # with the reference smoother the Krylov iteration counts are the reference's
    lin_ref = [int(x) for x in g["records"][1:, 5]]
    lin_gpu = [it.lin_iters for it in r.stats.iterations[1:]]
    assert lin_gpu == lin_ref, (lin_gpu, lin_ref)


def test_capped_c3_needs_the_reference_smoother(oc, ctx):
    # documents why the faithful mode exists: with capped Krylov solves the
    # 4-colour smoother lands on a different (equally valid) iterate
    g = load_golden("c3_l6_capped")
    qp = qp_from_golden(oc, ctx, g)
    s = g["meta"]["solve"]
    r = oc.ipm_solve(qp, oc.IpmParams(sigma=s["sigma"], solver=s["solver"], smoother="color4",
                                      linear_maxit=s["linear_maxit"]))
    assert rel(r.u, g["u"]) > 1e-8


@pytest.mark.parametrize("name", ["c3_l6_capped", "c3_l6_maxit200"])
def test_capped_c3_default_auto_smoother_matches_reference(oc, ctx, name):
    # the default smoother ("auto") redoes the first capped Newton solve with the
    # lexicographic smoother and keeps it: the capped fixtures then match
    g = load_golden(name)
    qp = qp_from_golden(oc, ctx, g)
    s = g["meta"]["solve"]
    r = oc.ipm_solve(qp, oc.IpmParams(sigma=s["sigma"], solver=s["solver"],
                                      linear_maxit=s["linear_maxit"]))
    assert r.lex_from >= 1 and r.discarded_lin >= s["linear_maxit"]
    assert rel(r.u, g["u"]) <= 1e-8, rel(r.u, g["u"])
    assert rel(r.state.y, g["y"]) <= 1e-8
    assert int((np.abs(r.u) < 1e-2).sum()) == int((np.abs(g["u"]) < 1e-2).sum())
    lin_ref = [int(x) for x in g["records"][1:, 5]]
    lin_gpu = [it.lin_iters for it in r.stats.iterations[1:]]
    assert lin_gpu == lin_ref, (lin_gpu, lin_ref)


def test_auto_smoother_is_colour_when_nothing_is_capped(oc, ctx):
    # converging Newton solves never trigger the fallback: bitwise the colour path
    g = load_golden("c1_l6_gmres")
    qp = qp_from_golden(oc, ctx, g)
    s = g["meta"]["solve"]
    ra = oc.ipm_solve(qp, oc.IpmParams(sigma=s["sigma"], solver=s["solver"]))
    rc = oc.ipm_solve(qp, oc.IpmParams(sigma=s["sigma"], solver=s["solver"], smoother="color4"))
    assert ra.lex_from == 0 and ra.discarded_lin == 0
    assert np.array_equal(ra.u, rc.u) and np.array_equal(ra.state.y, rc.state.y)
