"""The algorithmic byte model reproduces SURVEY.md §8d's table (CPU)."""
import pytest

from paper_1806_05896_b200 import bytes_model as bm


def test_mg_solve_words():
    assert bm.mg_solve_words(10) == pytest.approx(287.0, abs=0.1)
    assert bm.mg_solve_words(10, variable=True) == pytest.approx(575.0, abs=0.1)
    assert bm.mg_solve_words(10, with_diag=False) == pytest.approx(152.0, abs=0.2)


def test_survey_totals():
    # SURVEY §8d "Totals per KKT + P"
    assert bm.precond_words("pt", 10) == pytest.approx(665.0, abs=0.2)
    assert bm.precond_words("pd", 10) == pytest.approx(660.0, abs=0.2)
    assert bm.kkt_words() == 10.0
    assert bm.precond_words("ppi", 10, state_bounds=True) == pytest.approx(742.0, abs=0.3)
    assert bm.kkt_words(state_bounds=True) == 11.0
    assert bm.precond_words("pt", 10, pde="convdiff") == pytest.approx(1250.0, abs=0.3)
    assert bm.kkt_words(variable_l=True) == 19.0
    assert bm.precond_words("pt", 8, pde="heat") == pytest.approx(671.0, abs=0.3)


def test_apply_bytes_1025():
    n = 1023 * 1023
    k, p = bm.apply_bytes("pt", 10, n)
    assert (k + p) / 1e9 == pytest.approx(5.65, abs=0.01)   # 675 V at 1025^2
    assert bm.cheb_words() == 78.0
    assert bm.sweep_bytes(n) == 32.0 * n
