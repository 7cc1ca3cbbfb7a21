"""Algorithmic byte model of the hot path, in units of
V = 8 * ny bytes (one FP64 field vector).

Rules: each distinct operand vector is read once and each output written
once per pass; grid-constant stencils (Poisson L, M, M + tau L, masked M_obs)
cost no coefficient bytes; variable stencils (SUPG L, Galerkin coarse levels)
cost 9 words per node; diagonals cost 1 word. These are the bytes
``roofline.achieved`` divides by the measured kernel time.
"""
from __future__ import annotations


def coarse_fraction(level: int) -> float:
    """sum over coarse levels (level-1 .. 2) of n_l / n_fine."""
    nf = ((1 << level) - 1) ** 2
    return sum(((1 << l) - 1) ** 2 for l in range(2, level)) / nf


def sweep_words(variable: bool, with_diag: bool = True) -> float:
    """One fine smoothing sweep: read x, b (+ diag), write x; variable stencils
    read 9 coefficient arrays instead of the diagonal (SURVEY: 4V const+diag,
    12V SUPG, 3V constant L alone)."""
    if variable:
        return 12.0
    return 4.0 if with_diag else 3.0


def mg_solve_words(level: int, cycles=3, pre=5, post=5, variable=False, with_diag=True,
                   exact_coarse=False) -> float:
    """MgHierarchy::solve: per cycle the fine-level sweeps + residual (4V) +
    restriction (1.25V) + prolongation (2.25V) + divergence-check residual (3V),
    plus coarse levels at 135.5 words/node (12-word sweeps, residual, transfers).
    SURVEY §8d approximates the coarse sum by 1/3 of the fine size."""
    fine = (pre + post) * sweep_words(variable, with_diag) + 4.0 + 1.25 + 2.25 + 3.0
    if variable:
        # residual reads 9 coefficient words (12V), divergence check 11V (SURVEY: 575V/solve)
        fine = (pre + post) * 12.0 + 12.0 + 1.25 + 2.25 + 11.0
    if not with_diag and not variable:
        # MG on L alone (P_Pi's L-solve): all-constant stencils (SURVEY: 38.5V fine)
        fine = (pre + post) * 3.0 + 3.0 + 1.25 + 2.25 + 2.0
        coarse = 12.2
    else:
        coarse = 135.5 * (coarse_fraction(level) if exact_coarse else 1.0 / 3.0)
    return cycles * (fine + coarse)


def kkt_words(state_bounds=False, variable_l=False) -> float:
    return 10.0 + (1.0 if state_bounds else 0.0) + (9.0 if variable_l else 0.0)


def cheb_words(steps=20, state_bounds=False) -> float:
    return 2.0 + (steps - 1) * 4.0 + (steps if state_bounds else 0.0)


def precond_words(kind: str, level: int, pde="poisson", state_bounds=False, steps=20,
                  cycles=3, pre=5, post=5) -> float:
    var = pde == "convdiff"
    mg = mg_solve_words(level, cycles, pre, post, variable=var)
    if pde == "heat":
        mg += 3.0  # per-block rhs r_k + M t_{k-1} of the time substitution
    cheb = cheb_words(steps, state_bounds and kind != "ppi")
    if kind == "ppi":
        mg_l = mg_solve_words(level, cycles, pre, post, variable=var, with_diag=False) if not var \
            else mg_solve_words(level, cycles, pre, post, variable=True)
        return 6.0 + 4.0 + mg_l + 4.0 + mg + 2.0 + mg
    coupling = 5.0 + (9.0 if var else 0.0)
    middle = 2.0
    if kind == "pt":
        return cheb + 6.0 + coupling + mg + middle + mg
    return cheb + 6.0 + mg + middle + mg


def apply_bytes(kind: str, level: int, ny: int, pde="poisson", state_bounds=False, **kw):
    """(kkt_bytes, precond_bytes) for one KKT apply and one preconditioner apply."""
    V = 8.0 * ny
    return (kkt_words(state_bounds, pde == "convdiff") * V,
            precond_words(kind, level, pde, state_bounds, **kw) * V)


def sweep_bytes(ny_level: int, variable=False, with_diag=True) -> float:
    return sweep_words(variable, with_diag) * 8.0 * ny_level
