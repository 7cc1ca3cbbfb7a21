"""The BASELINE.json configurations and the seeded synthetic desired state.

No dataset is involved: BASELINE.json asks for y_d = a seeded sum of 4 sine
modes sin(k pi x1) sin(l pi x2), k, l in [1, 4], amplitudes U(-1, 1). The
recipe here is ours (numpy PCG64 via ``default_rng(seed)``; per mode draw k,
l, a in that order); both the GPU path and the CPU reference receive the same
host array, so the recipe only has to be deterministic, not libstdc++-exact.
Heat (config 5) multiplies by exp(-t_k) with t_k = (k+1) tau, the
backward-Euler time of block k.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Tuple

import numpy as np


def sine_modes(level: int, seed: int = 42, modes: int = 4) -> np.ndarray:
    nx = (1 << level) - 1
    h = 1.0 / (1 << level)
    idx = np.arange(nx * nx)
    x = (idx % nx + 1) * h
    y = (idx // nx + 1) * h
    rng = np.random.default_rng(seed)
    out = np.zeros(nx * nx)
    for _ in range(modes):
        k = int(rng.integers(1, 5))
        l = int(rng.integers(1, 5))
        a = float(rng.uniform(-1.0, 1.0))
        out += a * np.sin(k * np.pi * x) * np.sin(l * np.pi * y)
    return out


def sine_modes_spacetime(level: int, nt: int, tau: float, seed: int = 42) -> np.ndarray:
    base = sine_modes(level, seed)
    t = (np.arange(nt) + 1) * tau
    return (np.exp(-t)[:, None] * base[None, :]).reshape(-1)


def sin_sin(level: int) -> np.ndarray:
    """The reference CLI's hard-coded y_d (bench.cpp:63-70)."""
    nx = (1 << level) - 1
    h = 1.0 / (1 << level)
    idx = np.arange(nx * nx)
    x = (idx % nx + 1) * h
    y = (idx // nx + 1) * h
    return np.sin(np.pi * x) * np.sin(np.pi * y)


@dataclass
class Config:
    name: str
    pde: str
    level: int
    alpha: float
    beta: float
    solver: str
    u_a: float = -2.0
    u_b: float = 2.0
    y_a: Optional[float] = None
    y_b: Optional[float] = None
    obs: Optional[Tuple[float, float, float, float]] = None
    eps: float = 0.1
    tau: float = 0.04
    horizon: float = 1.0
    sigma: float = 0.2
    gmres_restart: int = 0
    seed: int = 42
    extra: dict = field(default_factory=dict)

    @property
    def nx(self) -> int:
        return (1 << self.level) - 1

    @property
    def n(self) -> int:
        return self.nx * self.nx

    @property
    def nt(self) -> int:
        return int(round(self.horizon / self.tau)) if self.pde == "heat" else 1

    def y_d(self) -> np.ndarray:
        if self.pde == "heat":
            return sine_modes_spacetime(self.level, self.nt, self.tau, self.seed)
        return sine_modes(self.level, self.seed)

    def with_level(self, level: int, **kw) -> "Config":
        d = dict(self.__dict__)
        d.update(kw)
        d["level"] = level
        return Config(**d)


# BASELINE.json "configs" (SURVEY.md §8d decisions: sigma 0.2; C5 tau = 1/128).
C1 = Config("C1", "poisson", 6, 1e-2, 1e-3, "minres-pd")
C2_CELLS = [Config(f"C2[a={a:g},b={b:g}]", "poisson", 9, a, b, "gmres-pt")
            for a in (1e-2, 1e-4, 1e-6) for b in (1e-2, 1e-3, 1e-4)]
C3 = Config("C3", "poisson", 10, 1e-4, 1e-3, "gmres-ppi", y_a=-0.2, y_b=0.3,
            obs=(0.0, 0.5, 0.0, 1.0))
C4 = Config("C4", "convdiff", 10, 1e-4, 1e-3, "gmres-pt", eps=0.02, gmres_restart=30)
C5 = Config("C5", "heat", 8, 1e-3, 1e-4, "gmres-pt", u_a=-1.0, u_b=1.0, tau=1.0 / 128)
ALL = {"C1": C1, "C2": C2_CELLS[0], "C3": C3, "C4": C4, "C5": C5}
