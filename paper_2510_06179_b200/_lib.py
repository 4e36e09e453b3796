"""ctypes binding of libdocp_cuda.so (include/docp_cuda.h).

The library is built in-tree (paper_2510_06179_b200/lib/libdocp_cuda.so) by
build.py. There is no CPU fallback: importing the product path without the
CUDA library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DOCP_LIB_PATH") or os.path.join(HERE, "lib", "libdocp_cuda.so")  # override: A/B builds

AFFINE_QUADRATIC, CARTPOLE, ATTITUDE, DRIFT = 1, 2, 3, 4
OK, DIMENSION, EVALUATION, NUMERICAL, BREAKDOWN, DIVERGENCE, UNSUPPORTED, CUDA_ERROR, INVALID = range(9)
PCG_FAST, PCG_PARITY, PCG_FP32 = 0, 1, 2
RHS_FORWARD, RHS_ADJOINT = 0, 1
MAX_STEP_CANDIDATES = 8

(F_THETA, F_Z, F_LAMBDA, F_LAMBDA_TILDE, F_LOSS_GRAD_Z, F_GRAD_THETA, F_GAMMA, F_Z_QP, F_STATUS, F_SQP_ITERS,
 F_CONVERGED, F_KKT, F_PCG_ITERS, F_PCG_CONVERGED, F_FINAL_ETA, F_PCG_HISTORY, F_STEP_SIZES, F_PD_PROJECTED, F_MU,
 F_ALPHA, F_ACCEPTED, F_LOSS, F_ROLLOUT_STATUS, F_REWARD) = range(24)
AT_ROLLOUT_ENV = 14


class Problem(C.Structure):
    _fields_ = [("family", C.c_int32), ("n_x", C.c_int32), ("n_u", C.c_int32), ("horizon", C.c_int32),
                ("cost_scale", C.c_double), ("cart_mass", C.c_double), ("pole_mass", C.c_double),
                ("length", C.c_double), ("gravity", C.c_double), ("dt", C.c_double)]


class Status(C.Structure):
    _fields_ = [("code", C.c_int32), ("where", C.c_int32), ("index", C.c_int32), ("step", C.c_int32)]


class PcgConfigC(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("max_iters", C.c_int32), ("mode", C.c_int32)]


class SqpConfigC(C.Structure):
    _fields_ = [("max_sqp_iters", C.c_int32), ("n_step_candidates", C.c_int32),
                ("step_candidates", C.c_double * MAX_STEP_CANDIDATES), ("eta_armijo", C.c_double),
                ("rho_penalty", C.c_double), ("pcg", PcgConfigC), ("convergence_tol", C.c_double),
                ("mu_floor_denominator", C.c_double), ("eps_pd", C.c_double)]


PROF_KINDS = 7
PROF_NAMES = ("assemble", "gamma", "pcg", "recover", "step", "kkt", "vjp")


class Profile(C.Structure):
    _fields_ = [("launches", C.c_int32 * PROF_KINDS), ("ms", C.c_double * PROF_KINDS),
                ("pcg_iterations", C.c_uint64), ("pcg_solves", C.c_uint64),
                ("pcg_bytes_per_iteration", C.c_double), ("pcg_algorithmic_bytes", C.c_double),
                ("span_ms", C.c_double), ("gap_ms", C.c_double), ("max_gap_ms", C.c_double),
                ("max_gap_after", C.c_int32), ("max_gap_before", C.c_int32)]


# every symbol include/docp_cuda.h declares, with its ctypes signature
_vp, _i32, _u64, _dbl, _sz = C.c_void_p, C.c_int32, C.c_uint64, C.c_double, C.c_size_t
_dp = C.POINTER(C.c_double)
SIGNATURES = {
    "docp_abi_version": (C.c_int, []),
    "docp_theta_size": (C.c_int, [C.POINTER(Problem)]),
    "docp_batch_create": (C.c_int, [C.POINTER(Problem), _i32, _i32, C.POINTER(_vp)]),
    "docp_batch_destroy": (None, [_vp]),
    "docp_batch_set_stream": (C.c_int, [_vp, _vp]),
    "docp_batch_sync": (C.c_int, [_vp]),
    "docp_batch_size": (_i32, [_vp]),
    "docp_batch_field_ptr": (C.c_int, [_vp, _i32, C.POINTER(_vp), C.POINTER(_sz)]),
    "docp_batch_upload": (C.c_int, [_vp, _i32, _vp, _i32]),
    "docp_batch_download": (C.c_int, [_vp, _i32, _vp, _i32]),
    "docp_batch_upload_schur": (C.c_int, [_vp, _dp, _dp, _dp, _dp]),
    "docp_batch_download_schur": (C.c_int, [_vp, _dp, _dp, _dp, _dp]),
    "docp_batch_download_qp": (C.c_int, [_vp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]),
    "docp_linearize": (C.c_int, [_vp, _dbl]),
    "docp_assemble_schur": (C.c_int, [_vp]),
    "docp_assemble_gamma": (C.c_int, [_vp, _i32]),
    "docp_pcg_solve": (C.c_int, [_vp, C.POINTER(PcgConfigC), _i32]),
    "docp_recover_primal": (C.c_int, [_vp, _i32, _i32]),
    "docp_line_search": (C.c_int, [_vp, C.POINTER(SqpConfigC)]),
    "docp_kkt_residual": (C.c_int, [_vp]),
    "docp_sqp_solve": (C.c_int, [_vp, C.POINTER(SqpConfigC)]),
    "docp_backward_vjp": (C.c_int, [_vp, C.POINTER(PcgConfigC)]),
    "docp_il_epoch": (C.c_int, [_vp, C.POINTER(SqpConfigC), _vp, _i32, _i32, _vp, _dbl, _vp, _vp]),
    "docp_il_failures": (C.c_int, [_vp, C.POINTER(_i32), C.POINTER(_i32)]),
    "docp_rollout": (C.c_int, [_vp, C.POINTER(SqpConfigC), _vp, _i32, _i32]),
    "docp_rollout_backward": (C.c_int, [_vp, C.POINTER(PcgConfigC)]),
    "docp_generate_affine_quadratic": (C.c_int, [_i32, _i32, _u64, _i32, _i32, _dp]),
    "docp_generate_uniform": (C.c_int, [_u64, _i32, _dbl, _dbl, _dp]),
    "docp_generate_drift_sequence": (C.c_int, [_i32, _i32, _u64, _i32, _dbl, _dp]),
    "docp_generate_cartpole_x0": (C.c_int, [_u64, _i32, _dp]),
    "docp_profile_begin": (C.c_int, [_vp]),
    "docp_profile_end": (C.c_int, [_vp, C.POINTER(Profile)]),
    "docp_pcg_invocations": (_u64, []),
    "docp_kernel_launches": (_u64, []),
    "docp_last_error": (C.c_char_p, []),
    "docp_format_status": (C.c_int, [C.POINTER(Status), C.c_char_p, _i32]),
    "docp_describe": (C.c_int, [C.POINTER(Problem), C.c_char_p, _i32]),
}

_lib = None


def lib():
    """The loaded library (raises if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libdocp_cuda.so not built at {LIB_PATH}: run `python build.py` (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        if L.docp_abi_version() != 1:
            raise ImportError("libdocp_cuda.so ABI version mismatch")
        _lib = L
    return _lib
