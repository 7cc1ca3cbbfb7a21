"""optcon-b200: B200-native (sm_100a, FP64) interior-point Newton solves for
L1-sparse, box-constrained PDE control (arXiv 1806.05896).

The hot path — KKT saddle-operator apply, block preconditioners (Chebyshev,
2x2 control inverse, matching-Schur factors by geometric multigrid), MINRES /
GMRES and the IPM step logic — runs as hand-written CUDA kernels in
``_lib/liboptcon_b200.so`` behind the C ABI declared in
``include/optcon_b200.h``. ``optcon`` mirrors the reference solver API.
"""
from . import configs  # noqa: F401

__all__ = ["optcon", "configs"]
