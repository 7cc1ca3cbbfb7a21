"""Benchmark harness on the device backend (reference bench.cpp):
configuration parsing and validation, sweep expansion and CSV formats on CPU;
on the GPU the artefacts of run_benchmark against the reference library and
bit-identical reruns."""
import filecmp
import os

import numpy as np
import pytest

from paper_1806_05896_b200 import harness as hz
from paper_1806_05896_b200 import optcon as oc


def test_config_from_map_and_defaults():
    c = hz.config_from_map({"pde": "convdiff", "ell": "7", "alpha": "1e-4", "eps": "0.02",
                            "solver": "gmres-pt", "T": "2", "out": "o", "obs_box": "0,0.5,0,1"})
    assert (c.pde, c.ell, c.alpha, c.eps, c.horizon, c.out_dir) == ("convdiff", 7, 1e-4, 0.02, 2.0, "o")
    assert c.obs_box == (0.0, 0.5, 0.0, 1.0)
    d = hz.RunConfig()
    assert (d.ell, d.alpha, d.beta, d.ua, d.ub, d.tau, d.lintol) == (5, 1e-2, 1e-2, -2.0, 1.5, 0.04, 1e-10)
    with pytest.raises(oc.OptconInvalidArgument, match="unknown pde"):
        hz.config_from_map({"pde": "wave"})


@pytest.mark.parametrize("cfg,msg", [
    (hz.RunConfig(obs_box=(0, 0.5, 0, 1)), "partial observation"),
    (hz.RunConfig(pde="heat", solver="minres-pd"), "gmres-pt only"),
    (hz.RunConfig(ya=-0.1), "pair"),
    (hz.RunConfig(ell=13), "ell out of supported range"),
])
def test_validate_config_messages(cfg, msg):
    with pytest.raises(oc.OptconInvalidArgument, match=msg):
        hz.validate_config(cfg)


def test_sweep_presets_expand_like_the_reference():
    assert len(hz.sweep_cells(hz.sweep_preset("table1"))) == 9
    assert len(hz.sweep_cells(hz.sweep_preset("table2"))) == 12
    t6 = hz.sweep_cells(hz.sweep_preset("table6"))
    assert len(t6) == 27 and t6[1].tau == 0.02 and t6[3].alpha == 1e-4
    t1 = hz.sweep_cells(hz.sweep_preset("table1"))
    assert [(c.alpha, c.beta) for c in t1[:4]] == [(1e-2, 1e-1), (1e-2, 1e-2), (1e-2, 1e-3), (1e-4, 1e-1)]


def test_formats():
    assert hz.fmt(0.1) == "0.10000000000000001"
    assert hz.summary_header() == "pde,ell,alpha,beta,sigma,eps,tau,solver,nli,av_li,sparsity,l1,converged"
    sp = hz.nodal_sparsity(np.array([0.0, 0.5, -0.005, 1.0] + [0.0] * 5), 2)  # nx = 3, 25 nodes
    assert sp.percent_below_threshold == pytest.approx(100.0 * (7 + 16) / 25)
    assert sp.l1_norm == pytest.approx(1.505)


@pytest.mark.gpu
def test_run_benchmark_matches_reference_and_reruns_bitwise(tmp_path, refmod):
    cfg = hz.RunConfig(pde="poisson", ell=6, alpha=1e-4, beta=1e-2, out_dir=str(tmp_path / "a"),
                       dump_solution=True)
    art = hz.run_benchmark(cfg)
    R = refmod.RefProblem("poisson", 6, alpha=1e-4, beta=1e-2, y_d=hz.default_desired_state("poisson", 6),
                          u_a=-2.0, u_b=1.5).solve("gmres-pt", sigma=0.2)
    sp_ref = hz.nodal_sparsity(R.u, 6)
    assert art.converged and abs(art.stats.nli - R.nli) <= 1
    assert art.sparsity.percent_below_threshold == sp_ref.percent_below_threshold
    assert abs(art.sparsity.l1_norm - sp_ref.l1_norm) <= 1e-8 * sp_ref.l1_norm
    for f in ("stats.csv", "summary.csv", "solution.csv"):
        assert os.path.getsize(tmp_path / "a" / f) > 0
    hz.run_benchmark(hz.RunConfig(**{**cfg.__dict__, "out_dir": str(tmp_path / "b")}))
    for f in ("stats.csv", "summary.csv", "solution.csv"):
        assert filecmp.cmp(tmp_path / "a" / f, tmp_path / "b" / f, shallow=False), f


@pytest.mark.gpu
def test_run_sweep_rows_in_cell_order(tmp_path):
    spec = hz.SweepSpec(hz.RunConfig(pde="poisson", sigma=0.2), [4], [1e-2, 1e-4], betas=[1e-2, 1e-3])
    path = tmp_path / "sweep.csv"
    assert hz.run_sweep(spec, str(path), workers=3) == 4
    lines = path.read_text().splitlines()
    assert lines[0] == hz.summary_header() and len(lines) == 5
    assert [ln.split(",")[2:4] for ln in lines[1:]] == [
        [hz.fmt(1e-2), hz.fmt(1e-2)], [hz.fmt(1e-2), hz.fmt(1e-3)],
        [hz.fmt(1e-4), hz.fmt(1e-2)], [hz.fmt(1e-4), hz.fmt(1e-3)]]
    path2 = tmp_path / "sweep2.csv"
    hz.run_sweep(spec, str(path2), workers=2)
    assert filecmp.cmp(path, path2, shallow=False)
