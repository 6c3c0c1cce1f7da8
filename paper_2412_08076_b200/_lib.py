"""ctypes binding of librichgpu.so (include/richgpu.h).

This is the only module that talks to the native library.  It fails loudly
when the library is missing: there is no CPU fallback anywhere in the
package.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("RICHGPU_LIB", _PKG / "librichgpu.so"))

RG_F32, RG_F64, RG_C128 = 1, 2, 3
RG_CONST9, RG_DIAG5, RG_VAR9 = 1, 2, 3
RG_PLAIN, RG_MOM, RG_NAG, RG_NAGEX = 0, 1, 2, 3
RG_PRECOND_NONE, RG_PRECOND_JACOBI_SCALAR, RG_PRECOND_JACOBI_FIELD = 0, 1, 2
RG_CHECK_OUTER, RG_CHECK_INNER = 0, 1
RG_TRI_SOR, RG_TRI_SSOR, RG_TRI_SOR_T, RG_TRI_SSOR_T = 1, 2, 3, 4
RG_ACTIVE, RG_CONVERGED, RG_DIVERGED, RG_MAXED = 0, 1, 2, 3
RG_KERNEL_STEP, RG_KERNEL_TILE, RG_KERNEL_WAVE, RG_KERNEL_CLUSTER = 0, 1, 2, 3
KERNEL_NAMES = {0: "step", 1: "tile", 2: "wave", 3: "cluster"}
RG_OK, RG_EINVAL, RG_ESIZE, RG_ENULL, RG_EUNSUPPORTED, RG_ECUDA, RG_ESTATE = 0, -1, -2, -3, -4, -5, -6

VARIANT_CODE = {"plain": RG_PLAIN, "mom": RG_MOM, "nag": RG_NAG, "nagex": RG_NAGEX}


class rg_op_desc(C.Structure):
    _fields_ = [("dtype", C.c_int), ("kind", C.c_int), ("batch", C.c_int), ("side", C.c_int),
                ("stencil", C.c_void_p), ("diag", C.c_void_p), ("shared", C.c_int)]


class rg_sched(C.Structure):
    _fields_ = [("variant", C.c_int), ("m", C.c_int), ("omega", C.c_void_p),
                ("alpha", C.c_void_p), ("alpha_tilde", C.c_void_p), ("precond", C.c_int),
                ("scale", C.c_void_p)]


class rg_report(C.Structure):
    _fields_ = [("status", C.c_int), ("iterations", C.c_int), ("inner_iterations", C.c_int),
                ("ans_buf", C.c_int), ("final_relative_residual", C.c_double),
                ("trace0", C.c_double), ("fnorm", C.c_double), ("bad_rel", C.c_double)]


# (name, restype, argtypes) for every symbol declared in include/richgpu.h
_P = C.c_void_p
_I = C.c_int
_SIGS = [
    ("rg_version", _I, []),
    ("rg_last_error", C.c_char_p, []),
    ("rg_op_create", _I, [C.POINTER(_P), C.POINTER(rg_op_desc)]),
    ("rg_op_destroy", _I, [_P]),
    ("rg_matvec", _I, [_P, _P, _P, _P]),
    ("rg_residual", _I, [_P, _P, _P, _P, _P, _P]),
    ("rg_power_steps", _I, [_P, _I, _P, _P, _P, _P, C.c_double, _I, _P, _P, _P, _P]),
    ("rg_inner_update", _I, [_P, C.POINTER(rg_sched), _I, _P, _P, _P, _P, _P, _P, _I, _P]),
    ("rg_tri_apply", _I, [_P, _I, C.c_double, _P, _P, _P, _P]),
    ("rg_unroll_adjoint_init", _I, [_P, _P, _P, _P, _P, _P, _P, _P, _P]),
    ("rg_unroll_adjoint_step", _I, [_P, _P, C.POINTER(rg_sched), _I, _P, _P, _P, _P, _P, _P, _P,
                                    _P]),
    ("rg_unroll_adjoint_step_ext", _I, [_P, _P, C.POINTER(rg_sched), _I, _P, _P, _P, _P, _P, _P,
                                        _P, _I, _P]),
    ("rg_precond_update", _I, [_P, C.POINTER(rg_sched), _I, _P, _P, _P, _P, _P]),
    ("rg_sweep", _I, [_P, C.POINTER(rg_sched), _I, _I, _I, _P, _P, _P, _P, _P, C.POINTER(_I), _P]),
    ("rg_sweep_from_zero", _I, [_P, C.POINTER(rg_sched), _I, _I, _I, _P, _P, _P, _P, _P, _I, C.POINTER(_I), _P]),
    ("rg_sweep_norm", _I, [_P, C.POINTER(rg_sched), _I, _I, _I, _P, _P, _P, _P, _P, _P, C.POINTER(_I), _P]),
    ("rg_dst_create", _I, [C.POINTER(_P), _I, _I]),
    ("rg_dst_destroy", _I, [_P]),
    ("rg_dst2", _I, [_P, _P, _P, _P]),
    ("rg_fns_correct", _I, [_P, _P, _P, _P, _P, _P]),
    ("rg_restrict", _I, [_I, _I, _I, _P, _P, _P]),
    ("rg_prolong_add", _I, [_I, _I, _I, _P, _P, _P]),
    ("rg_dense_apply", _I, [_I, _I, _I, _P, _I, _P, _P, _P]),
    ("rg_mgs_step", _I, [_I, _I, _I, _P, C.c_longlong, _P, C.c_longlong, _P, _P, C.c_longlong, _P,
                         _P, _P]),
    ("rg_mgs_arnoldi", _I, [_I, _I, _I, _P, C.c_longlong, _P, C.c_longlong, _I, _P, _P, _P]),
    ("rg_arnoldi_tail", _I, [_I, _I, _I, _P, C.c_longlong, _P, C.c_longlong, _P, _I, _P, _P, _P]),
    ("rg_krylov_update", _I, [_I, _I, _P, _P, C.c_longlong, _P, _I, _P]),
    ("rg_solver_create", _I, [C.POINTER(_P), _P, C.POINTER(rg_sched), C.c_double, _I, _I, _I]),
    ("rg_solver_destroy", _I, [_P]),
    ("rg_solver_begin", _I, [_P, _P, _P, _P, _P, _P, _P]),
    ("rg_solver_step", _I, [_P, _P, C.POINTER(_I)]),
    ("rg_solver_run", _I, [_P, _I, _P]),
    ("rg_solver_flush", _I, [_P, _P]),
    ("rg_solver_poll", _I, [_P, _P, C.POINTER(_I), C.POINTER(_I)]),
    ("rg_solver_report", _I, [_P, _I, C.POINTER(rg_report)]),
    ("rg_solver_trace", _I, [_P, _I, C.POINTER(C.c_double), _I, C.POINTER(_I)]),
    ("rg_solver_plan", _I, [_P, C.POINTER(_I), C.POINTER(_I), C.POINTER(_I)]),
    ("rg_solver_info", _I, [_P, C.POINTER(C.c_longlong), C.POINTER(_I), C.POINTER(_I)]),
]
SYMBOLS = [s[0] for s in _SIGS]


class RichGpuError(RuntimeError):
    """A librichgpu call failed (usage error or CUDA error)."""

    def __init__(self, code, message):
        super().__init__(f"librichgpu error {code}: {message}")
        self.code = code


_lib = None


def load():
    """Load librichgpu.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2412_08076_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH))
    for name, res, args in _SIGS:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.rg_version() != 1:
        raise RuntimeError(f"librichgpu ABI version {lib.rg_version()} != 1")
    _lib = lib
    return lib


def check(rc):
    """Raise on a non-zero librichgpu return code."""
    if rc != RG_OK:
        msg = load().rg_last_error().decode(errors="replace")
        if rc in (RG_ESIZE,):
            from .errors import DimensionMismatch
            raise DimensionMismatch(msg)
        if rc in (RG_EINVAL,):
            raise ValueError(msg)
        if rc == RG_EUNSUPPORTED:
            from .errors import UnsupportedOperator
            raise UnsupportedOperator(msg)
        raise RichGpuError(rc, msg)
    return rc


def ptr(t):
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else C.c_void_p(t.data_ptr())


def stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)
