"""Pin the numpy restatement (oracle/port.py) against the reference: the
committed golden fixtures (made by the reference itself) and, when available,
the live reference library. CPU only."""
import numpy as np
import pytest

from conftest import load_golden, rel


def make_qp(g, port, smoother="lex"):
    pk = g["meta"]["problem"]
    kw = dict(level=pk["level"], pde=pk["pde"], alpha=pk["alpha"], beta=pk["beta"],
              y_d=g["y_d"], u_a=pk["u_a"], u_b=pk["u_b"], eps=pk.get("eps", 0.1),
              smoother=smoother)
    if "y_a" in pk:
        kw.update(y_a=pk["y_a"], y_b=pk["y_b"])
    if "obs" in pk:
        kw.update(obs=tuple(pk["obs"]))
    return port.Qp(**kw)


@pytest.fixture(scope="module")
def port():
    from oracle import port

    return port


@pytest.mark.parametrize("what", ["mass", "poisson", "convdiff", "partial_mass", "lumped"])
def test_port_assembly(port, what):
    g = load_golden("assembly")
    for lvl in (3, 4):
        ref = g[f"{what}_l{lvl}"]
        kw = dict(eps=0.02) if what == "convdiff" else {}
        obs = (0.0, 0.5, 0.0, 1.0) if what == "partial_mass" else None
        mine = port.assemble(what, lvl, obs=obs, **kw)
        assert np.abs(mine - ref).max() <= 4e-16 * np.abs(ref).max()


@pytest.mark.parametrize("name", ["kkt_poisson_l5", "kkt_convdiff_l5", "kkt_partial_l5"])
def test_port_kkt_matches_golden(port, name):
    g = load_golden(name)
    qp = make_qp(g, port)
    ax = qp.kkt(g["theta_y"], g["theta_w"], g["theta_v"], g["x"])
    assert rel(ax, g["ax"]) <= 1e-14


@pytest.mark.parametrize("name", ["smoke_l5", "c3_l4"])
def test_port_ipm_matches_golden(port, name):
    g = load_golden(name)
    qp = make_qp(g, port)
    s = g["meta"]["solve"]
    r = port.ipm_solve(qp, sigma=s["sigma"], solver=s["solver"],
                       linear_maxit=s.get("linear_maxit", 200))
    assert abs(r["nli"] - int(g["nli"])) <= 1
    assert rel(r["u"], g["u"]) <= 1e-8
    assert rel(r["y"], g["y"]) <= 1e-8
    assert abs(r["objective"] - float(g["objective"])) <= 1e-8 * abs(float(g["objective"]))
    assert int((np.abs(r["u"]) < 1e-2).sum()) == int((np.abs(g["u"]) < 1e-2).sum())


def test_port_multigrid_matches_live_reference(port, refmod):
    # lexicographic smoother restated: same V-cycle as multigrid.cpp to rounding
    level = 5
    L = refmod.assemble9("poisson", level)
    rng = np.random.default_rng(11)
    d = 10 ** rng.uniform(-2, 1, L.shape[1])
    A = L.copy()
    A[4] += d
    b = rng.uniform(-1, 1, L.shape[1])
    x_ref = refmod.RefMg(level, A).solve(b)
    x_port = port.MgHierarchy(port.to_csr(A), level).solve(b)
    assert rel(x_port, x_ref) <= 1e-12


def test_port_chebyshev_matches_live_reference(port, refmod):
    level = 4
    rng = np.random.default_rng(13)
    n = 225
    e = 10 ** rng.uniform(-6, -3, n)
    b = rng.uniform(-1, 1, n)
    M = port.to_csr(port.assemble("mass", level))
    assert rel(port.chebyshev(M, 0.3, e, 20, b), refmod.cheb_apply(level, 0.3, e, 20, b)) <= 1e-13


def test_port_color4_vcycle_is_spd(port):
    # the GPU smoother variant keeps the V-cycle map symmetric positive definite
    level = 4
    L = port.assemble("poisson", level)
    rng = np.random.default_rng(17)
    L[4] += 10 ** rng.uniform(-2, 1, L.shape[1])
    mg = port.MgHierarchy(port.to_csr(L), level, smoother="color4")
    x, y = rng.uniform(-1, 1, (2, L.shape[1]))
    assert x @ mg.solve(x) > 0
    assert abs(y @ mg.solve(x) - x @ mg.solve(y)) <= 1e-10 * abs(x @ mg.solve(y))
