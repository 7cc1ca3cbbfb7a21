"""ctypes binding of the in-tree C-ABI library ``_lib/liboptcon_b200.so``.

The library is the product: every compute entry point runs sm_100a kernels.
There is no CPU fallback — if the shared object is missing this module raises
at import-use time, and if no CUDA device is present the library itself
returns OC_CUDA_ERROR.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# OPTCON_B200_LIB: another build of the same library (A/B runs of tools/ab_lib.py)
LIB_PATH = os.environ.get("OPTCON_B200_LIB") or os.path.join(_HERE, "_lib", "liboptcon_b200.so")

OC_OK, OC_INVALID_ARGUMENT, OC_RUNTIME_ERROR, OC_CUDA_ERROR = 0, 1, 2, 3

_dp = C.POINTER(C.c_double)


class ProblemDesc(C.Structure):
    _fields_ = [
        ("pde", C.c_int), ("level", C.c_int), ("eps", C.c_double), ("tau", C.c_double),
        ("horizon", C.c_double), ("quadrature", C.c_int), ("alpha", C.c_double),
        ("beta", C.c_double), ("y_d", C.c_void_p), ("y_d_len", C.c_longlong),
        ("f", C.c_void_p), ("u_a", C.c_void_p), ("u_b", C.c_void_p), ("y_a", C.c_void_p),
        ("y_b", C.c_void_p), ("has_obs", C.c_int), ("obs", C.c_double * 4),
    ]


class IpmParamsC(C.Structure):
    _fields_ = [
        ("alpha0", C.c_double), ("sigma", C.c_double), ("eps_p", C.c_double),
        ("eps_d", C.c_double), ("eps_c", C.c_double), ("mu0", C.c_double),
        ("max_iterations", C.c_int), ("linear_tol", C.c_double), ("linear_maxit", C.c_int),
        ("cheb_steps", C.c_int), ("mg_cycles", C.c_int), ("mg_pre", C.c_int),
        ("mg_post", C.c_int), ("solver", C.c_int), ("smoother", C.c_int),
        ("gmres_restart", C.c_int),
    ]


class IterRecordC(C.Structure):
    _fields_ = [
        ("k", C.c_int), ("mu", C.c_double), ("norm_xp", C.c_double), ("norm_xd", C.c_double),
        ("norm_xc", C.c_double), ("lin_iters", C.c_int), ("lin_relres", C.c_double),
        ("lin_converged", C.c_int), ("newton_ms", C.c_double),
    ]


class IpmResultC(C.Structure):
    _fields_ = [
        ("y", C.c_void_p), ("z", C.c_void_p), ("p", C.c_void_p), ("lam_ya", C.c_void_p),
        ("lam_yb", C.c_void_p), ("lam_za", C.c_void_p), ("lam_zb", C.c_void_p),
        ("u", C.c_void_p), ("records", C.POINTER(IterRecordC)), ("records_cap", C.c_int),
        ("n_records", C.c_int), ("nli", C.c_int), ("converged", C.c_int),
        ("av_li", C.c_double), ("mu", C.c_double), ("objective", C.c_double),
        ("sparsity_pct", C.c_double), ("l1", C.c_double), ("nodal_sparsity_pct", C.c_double),
        ("total_lin", C.c_longlong), ("solve_ms", C.c_double), ("newton_ms", C.c_double),
        ("discarded_lin", C.c_longlong), ("lex_from", C.c_int),
    ]


class SolveReportC(C.Structure):
    _fields_ = [
        ("iterations", C.c_int), ("relative_residual", C.c_double), ("converged", C.c_int),
        ("breakdown", C.c_int), ("message", C.c_char * 96),
    ]


class ProblemInfoC(C.Structure):
    _fields_ = [
        ("n", C.c_int), ("nt", C.c_int), ("ny", C.c_longlong), ("kkt_dim", C.c_longlong),
        ("has_state_bounds", C.c_int), ("partial_observation", C.c_int),
        ("symmetric_k", C.c_int), ("level", C.c_int), ("h2d_bytes", C.c_longlong),
    ]


class OptconError(RuntimeError):
    """std::runtime_error raised by the device solver."""


class OptconInvalidArgument(ValueError):
    """std::invalid_argument raised by the device solver."""


class OptconCudaError(RuntimeError):
    """CUDA failure (no device, launch error) — never silently falls back."""


# Every symbol the C header declares (tests check they are all exported).
EXPORTS = [
    "oc_last_error", "oc_abi_version", "oc_create", "oc_destroy", "oc_synchronize",
    "oc_problem_create", "oc_problem_destroy", "oc_problem_info_get", "oc_default_params",
    "oc_ipm_solve", "oc_kkt_apply", "oc_precond_setup", "oc_precond_apply", "oc_schur_apply",
    "oc_newton_solve", "oc_ipm_pieces", "oc_objective", "oc_time_applies", "oc_mg_create",
    "oc_mg_solve", "oc_mg_depth", "oc_mg_level_matrix", "oc_mg_destroy", "oc_mg_smooth",
    "oc_cheb_apply", "oc_assemble9", "oc_launch_count", "oc_profile", "oc_profile_read",
    "oc_event_record", "oc_event_elapsed", "oc_debug_cluster_probes", "oc_debug_coarse_op", "oc_event_elapsed_between",
    "oc_set_tuning", "oc_get_tuning", "oc_assemble9_device", "oc_debug_lex_div",
]

_lib = None


def load():
    """Load the product library or fail loudly (no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"optcon-b200 CUDA library not built: {LIB_PATH}. Run __graft_entry__.build() "
            "or `make -C paper_1806_05896_b200/csrc`.")
    L = C.CDLL(LIB_PATH)
    L.oc_last_error.restype = C.c_char_p
    L.oc_abi_version.restype = C.c_int
    L.oc_destroy.argtypes = [C.c_void_p]
    L.oc_destroy.restype = None
    L.oc_problem_destroy.argtypes = [C.c_void_p]
    L.oc_problem_destroy.restype = None
    L.oc_mg_destroy.argtypes = [C.c_void_p]
    L.oc_mg_destroy.restype = None
    L.oc_mg_depth.argtypes = [C.c_void_p]
    L.oc_create.argtypes = [C.POINTER(C.c_void_p), C.c_int]
    L.oc_synchronize.argtypes = [C.c_void_p]
    L.oc_problem_create.argtypes = [C.c_void_p, C.POINTER(ProblemDesc), C.POINTER(C.c_void_p)]
    L.oc_problem_info_get.argtypes = [C.c_void_p, C.POINTER(ProblemInfoC)]
    L.oc_default_params.argtypes = [C.POINTER(IpmParamsC)]
    L.oc_ipm_solve.argtypes = [C.c_void_p, C.POINTER(IpmParamsC), C.POINTER(IpmResultC)]
    vp = C.c_void_p
    L.oc_kkt_apply.argtypes = [vp, vp, vp, vp, vp, vp]
    L.oc_precond_setup.argtypes = [vp, vp, vp, vp, C.POINTER(IpmParamsC)]
    L.oc_precond_apply.argtypes = [vp, C.c_int, vp, vp]
    L.oc_schur_apply.argtypes = [vp, vp, vp]
    L.oc_newton_solve.argtypes = [vp, vp, vp, vp, vp, vp, vp, C.POINTER(IpmParamsC), vp, vp, vp,
                                  C.POINTER(SolveReportC)]
    L.oc_ipm_pieces.argtypes = [vp] * 8 + [C.c_double, C.c_double] + [vp] * 7
    L.oc_objective.argtypes = [vp, vp, vp, _dp]
    L.oc_time_applies.argtypes = [vp, C.c_int, C.c_int, _dp, _dp]
    L.oc_mg_create.argtypes = [vp, C.c_int, vp, C.c_int, C.c_double, C.c_int, C.POINTER(C.c_void_p)]
    L.oc_mg_solve.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int, vp]
    L.oc_mg_level_matrix.argtypes = [vp, C.c_int, vp]
    L.oc_mg_smooth.argtypes = [vp, vp, vp, C.c_int]
    L.oc_cheb_apply.argtypes = [vp, C.c_int, C.c_double, vp, C.c_int, vp, vp]
    L.oc_assemble9.argtypes = [C.c_int, C.c_int, C.c_double, vp, vp]
    L.oc_assemble9_device.argtypes = [vp, C.c_int, C.c_int, C.c_double, vp, vp]
    L.oc_launch_count.restype = C.c_longlong
    L.oc_launch_count.argtypes = []
    L.oc_profile.argtypes = [vp, C.c_int]
    L.oc_profile_read.argtypes = [vp, _dp, C.POINTER(C.c_longlong)]
    L.oc_event_record.argtypes = [vp, C.c_int]
    L.oc_event_elapsed.argtypes = [vp, C.c_int, C.c_int, _dp]
    L.oc_event_elapsed_between.argtypes = [vp, C.c_int, vp, C.c_int, _dp]
    L.oc_debug_cluster_probes.argtypes = [C.c_int, vp]
    L.oc_debug_coarse_op.argtypes = [vp, C.c_int, C.c_int, vp]
    L.oc_debug_lex_div.argtypes = [vp, vp, vp, C.c_longlong, C.POINTER(C.c_ulonglong)]
    L.oc_set_tuning.argtypes = [C.c_char_p, C.c_int]
    L.oc_get_tuning.argtypes = [C.c_char_p, C.POINTER(C.c_int)]
    _lib = L
    return L


def check(rc: int):
    if rc == OC_OK:
        return
    msg = load().oc_last_error().decode()
    if rc == OC_INVALID_ARGUMENT:
        raise OptconInvalidArgument(msg)
    if rc == OC_CUDA_ERROR:
        raise OptconCudaError(msg)
    raise OptconError(msg)
