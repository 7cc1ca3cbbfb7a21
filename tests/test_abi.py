"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/optcon_b200.h declares, refuses to compute without a device
(no CPU fallback), and its host-side assembly matches the reference's."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_golden


def header_functions():
    txt = open(os.path.join(ROOT, "include", "optcon_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(oc_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_expected_entry_points():
    fns = header_functions()
    for must in ["oc_create", "oc_problem_create", "oc_ipm_solve", "oc_kkt_apply",
                 "oc_precond_apply", "oc_newton_solve", "oc_mg_solve", "oc_cheb_apply"]:
        assert must in fns


def test_library_exports_every_declared_symbol():
    from paper_1806_05896_b200 import _lib

    L = _lib.load()
    for fn in header_functions():
        assert hasattr(L, fn), fn
    assert set(header_functions()) == set(_lib.EXPORTS)
    assert L.oc_abi_version() == 2


def test_no_cpu_fallback_without_device():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    from paper_1806_05896_b200 import _lib, optcon as oc

    with pytest.raises(_lib.OptconCudaError):
        oc.Context(0)
    h = C.c_void_p()
    assert _lib.load().oc_create(C.byref(h), 0) == _lib.OC_CUDA_ERROR


def test_default_params_match_reference():
    from paper_1806_05896_b200 import _lib

    p = _lib.IpmParamsC()
    assert _lib.load().oc_default_params(C.byref(p)) == 0
    # IpmParams defaults (ipm.hpp:17-32)
    assert (p.alpha0, p.sigma, p.eps_p, p.mu0, p.max_iterations) == (0.995, 0.2, 1e-6, 1.0, 100)
    assert (p.linear_tol, p.linear_maxit, p.cheb_steps) == (1e-10, 200, 20)
    assert (p.mg_cycles, p.mg_pre, p.mg_post, p.solver) == (3, 5, 5, 0)


@pytest.mark.parametrize("what", ["mass", "poisson", "convdiff", "partial_mass", "lumped"])
@pytest.mark.parametrize("level", [3, 4])
def test_host_assembly_matches_reference(what, level):
    from paper_1806_05896_b200 import optcon as oc

    g = load_golden("assembly")
    ref = g[f"{what}_l{level}"]
    kw = dict(eps=0.02) if what == "convdiff" else {}
    obs = (0.0, 0.5, 0.0, 1.0) if what == "partial_mass" else None
    mine = oc.assemble9(what, level, obs=obs, **kw)
    # same element formulas; only the duplicate-summation order differs (<= 2 ulp)
    scale = np.abs(ref).max()
    assert np.abs(mine - ref).max() <= 4e-16 * scale
    assert np.array_equal(mine != 0, ref != 0) or what == "convdiff"


def test_assemble_rejects_bad_arguments():
    from paper_1806_05896_b200 import optcon as oc

    with pytest.raises(oc.OptconInvalidArgument):
        oc.assemble9("convdiff", 3, eps=0.0)
    with pytest.raises(oc.OptconInvalidArgument):
        oc.assemble9("mass", 15)


def test_configs_match_baseline():
    from paper_1806_05896_b200 import configs

    assert configs.C1.level == 6 and configs.C1.n == 63 * 63
    assert len(configs.C2_CELLS) == 9 and {c.level for c in configs.C2_CELLS} == {9}
    assert configs.C3.obs == (0.0, 0.5, 0.0, 1.0) and configs.C3.y_a == -0.2
    assert configs.C4.eps == 0.02 and configs.C4.gmres_restart == 30
    assert configs.C5.nt == 128 and configs.C5.level == 8
    y = configs.sine_modes(5, 42)
    assert np.array_equal(y, configs.sine_modes(5, 42))
    assert not np.array_equal(y, configs.sine_modes(5, 43))
