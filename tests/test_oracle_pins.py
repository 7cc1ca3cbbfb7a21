"""Pin the CPU oracle (the reference compiled from its own sources, oracle/_ref)
against the reference's own known answers and tests, and check
the committed golden fixtures are reproducible. CPU only."""
import math

import numpy as np
import pytest

from conftest import golden_names, load_golden, rel


def test_golden_known_answer_pins():
    # test_ipm.cpp:317-343: l=6 Poisson, alpha 1e-4, beta 1e-2, sigma 0.2, gmres-pt
    g = load_golden("known_answer_l6")
    assert int(g["nli"]) == 9
    assert int(g["converged"]) == 1
    assert abs(float(g["mu"]) - 0.2 ** 9) <= 1e-12 * 0.2 ** 9
    rec = g["records"]
    for k in range(1, rec.shape[0]):
        assert abs(rec[k, 1] - 0.2 * rec[k - 1, 1]) <= 1e-12 * rec[k - 1, 1]
        assert rec[k, 4] <= 2.0 * rec[k, 1]       # ||xi_c|| <= 2 mu
        assert rec[k, 7] == 1                     # every Newton solve converged
    # test_output.txt:37 / SURVEY §8c: av-li 4.67 for this cell
    assert abs(float(g["av_li"]) - 14.0 / 3.0) < 1e-12


def test_golden_documented_bands():
    # heat NLI in 9..14 (test_timedep.cpp:342-365); P_Pi converges (test_ipm.cpp:474-496)
    assert 9 <= int(load_golden("c5_l5_nt16")["nli"]) <= 14
    c3 = load_golden("c3_l5")
    assert int(c3["converged"]) == 1 and all(c3["records"][1:, 7] == 1)
    for name in golden_names("c"):
        g = load_golden(name)
        assert int(g["converged"]) == 1, name


@pytest.mark.parametrize("name", ["known_answer_l6", "c1_l6_minres", "c4_l6", "c5_l5_nt16"])
def test_live_oracle_reproduces_golden(refmod, name):
    from golden.make_golden import IPM_CASES, ref_problem

    pkw, skw = next((p, s) for n, p, s in IPM_CASES if n == name)
    r = ref_problem(pkw).solve(**skw)
    g = load_golden(name)
    assert r.nli == int(g["nli"])
    assert rel(r.u, g["u"]) <= 1e-12 and rel(r.y, g["y"]) <= 1e-12
    assert abs(r.objective - float(g["objective"])) <= 1e-12 * abs(float(g["objective"]))


def test_oracle_theta_midpoint(refmod):
    # test_ipm.cpp:62-78: at the initial point theta = 4/span
    level = 3
    n = 49
    yd = np.sin(np.pi * np.arange(n) / n)
    P = refmod.RefProblem("poisson", level, alpha=1e-2, beta=1e-2, y_d=yd, u_a=-2.0, u_b=1.5)
    za = np.r_[np.zeros(n), np.zeros(n)]
    zb = np.r_[np.full(n, 1.5), np.full(n, 2.0)]
    z = 0.5 * (za + zb)
    out = P.ipm_pieces(yd, z, np.zeros(n), np.ones(2 * n), np.ones(2 * n), mu_state=1.0)
    assert np.allclose(out["theta_w"], 4.0 / 1.5, rtol=1e-12)
    assert np.allclose(out["theta_v"], 4.0 / 2.0, rtol=1e-12)
    assert np.all(out["theta_y"] == 0.0)


def test_oracle_multigrid_pins(refmod):
    # test_multigrid.cpp:61-73 (>= 1e3 in 3 V-cycles) and :33-41 (Galerkin = assembled)
    level = 5
    L = refmod.assemble9("poisson", level)
    mg = refmod.RefMg(level, L)
    assert mg.depth() == level - 2
    rng = np.random.default_rng(3)
    b = rng.uniform(-1, 1, L.shape[1])
    x = mg.solve(b, 3, 5, 5)
    r = b - apply9(L, x, level)
    assert np.linalg.norm(r) <= 1e-3 * np.linalg.norm(b)
    Lc = refmod.assemble9("poisson", level - 1)
    assert np.linalg.norm(mg.level_matrix(1) - Lc) <= 1e-12 * np.linalg.norm(Lc)


def test_oracle_chebyshev_pin(refmod):
    # test_krylov.cpp:131-163: 20 steps reach <= 2e-6 relative error
    level = 4
    M = refmod.assemble9("mass", level)
    n = M.shape[1]
    rng = np.random.default_rng(5)
    extra = 10 ** rng.uniform(-3, 0, n) * M[4].max()
    b = rng.uniform(-1, 1, n)
    x = refmod.cheb_apply(level, 1.0, extra, 20, b)
    A = dense9(M, level) + np.diag(extra)
    xs = np.linalg.solve(A, b)
    assert np.linalg.norm(x - xs) <= 2e-6 * np.linalg.norm(xs)


def apply9(coef, x, level):
    nx = (1 << level) - 1
    X = x.reshape(nx, nx)
    out = np.zeros_like(X)
    P = np.pad(X, 1)
    for d in range(9):
        dx, dy = d % 3 - 1, d // 3 - 1
        out += coef[d].reshape(nx, nx) * P[1 + dy:1 + dy + nx, 1 + dx:1 + dx + nx]
    return out.reshape(-1)


def dense9(coef, level):
    nx = (1 << level) - 1
    n = nx * nx
    A = np.zeros((n, n))
    for i in range(n):
        gx, gy = i % nx, i // nx
        for d in range(9):
            jx, jy = gx + d % 3 - 1, gy + d // 3 - 1
            if 0 <= jx < nx and 0 <= jy < nx:
                A[i, jy * nx + jx] = coef[d, i]
    return A


def test_golden_sizes_are_small():
    import os

    from conftest import GOLDEN

    total = sum(os.path.getsize(os.path.join(GOLDEN, f)) for f in os.listdir(GOLDEN)
                if f.endswith(".npz"))
    assert total < 8 * 1024 * 1024
    assert math.isfinite(total)
