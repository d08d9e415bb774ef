"""ctypes binding of libmfwq.so (include/mfwq.h).

The product path has no fallback: if the shared library is missing or no
CUDA device is present, every operator raises instead of computing on the
CPU.
"""

import ctypes as C
import os

import numpy as np

from .errors import (DegenerateGeometryError, EigenSolveError,
                     IndefiniteOperatorError, WQConstructionError)

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MFWQ_LIB") or os.path.join(_PKG, "libmfwq.so")  # override: experiments only

_lib = None

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)


class StiffnessDesc(C.Structure):
    _fields_ = [("p", C.c_int * 3), ("nknots", C.c_int * 3), ("knots", dp * 3),
                ("npts", C.c_int * 3), ("pts", dp * 3),
                ("indptr", ip * 18), ("indices", ip * 18), ("data", dp * 18)]


class KrylovReportC(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("matvecs", C.c_int),
                ("precond_applies", C.c_int), ("n_residuals", C.c_int)]


_SIGS = {
    "mfwq_last_error": (C.c_char_p, []),
    "mfwq_version": (C.c_int, []),
    "mfwq_launch_count": (C.c_longlong, []),
    "mfwq_set_lapack": (C.c_int, [C.c_char_p, C.c_char_p]),
    "mfwq_lapack_active": (C.c_int, []),
    "mfwq_rule1d_build": (C.c_int, [C.c_int, C.c_int, dp, C.POINTER(C.c_void_p)]),
    "mfwq_rule1d_sizes": (C.c_int, [C.c_void_p, ip, ip, ip, ip]),
    "mfwq_rule1d_export": (C.c_int, [C.c_void_p, dp, C.POINTER(ip), C.POINTER(ip), C.POINTER(dp)]),
    "mfwq_rule1d_destroy": (None, [C.c_void_p]),
    "mfwq_univariate_km": (C.c_int, [C.c_int, C.c_int, dp, dp, dp]),
    "mfwq_stiffness_create": (C.c_int, [C.POINTER(StiffnessDesc), C.POINTER(C.c_void_p)]),
    "mfwq_stiffness_set_geometry": (C.c_int, [C.c_void_p, C.c_int, dp, dp, C.c_void_p, C.c_void_p, C.c_void_p]),
    "mfwq_stiffness_set_on_the_fly": (C.c_int, [C.c_void_p, C.c_int, dp, dp, C.c_void_p]),
    "mfwq_stiffness_set_coeffs": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.c_void_p]),
    "mfwq_mass_set": (C.c_int, [C.c_void_p, C.c_int, dp, C.c_void_p, C.c_double, C.c_void_p, C.c_int, C.c_void_p]),
    "mfwq_mass_apply": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "mfwq_mass_flops": (C.c_int, [C.c_void_p, C.POINTER(C.c_longlong)]),
    "mfwq_stiffness_get_coeff": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]),
    "mfwq_stiffness_sizes": (C.c_int, [C.c_void_p, ip, ip, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]),
    "mfwq_stiffness_apply": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "mfwq_stiffness_apply_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "mfwq_stiffness_host_join": (C.c_int, [C.c_void_p, C.c_void_p]),
    "mfwq_stiffness_apply_pageable": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "mfwq_stiffness_set_path": (C.c_int, [C.c_void_p, C.c_int]),
    "mfwq_stiffness_set_deterministic": (C.c_int, [C.c_void_p, C.c_int]),
    "mfwq_stiffness_set_slab": (C.c_int, [C.c_void_p, C.c_int, C.c_int]),
    "mfwq_stiffness_slab_info": (C.c_int, [C.c_void_p, ip]),
    "mfwq_stiffness_info": (C.c_int, [C.c_void_p, ip, ip, ip]),
    "mfwq_stiffness_flops": (C.c_int, [C.c_void_p, C.POINTER(C.c_longlong)]),
    "mfwq_stiffness_flops_active": (C.c_int, [C.c_void_p, C.POINTER(C.c_longlong)]),
    "mfwq_stiffness_destroy": (None, [C.c_void_p]),
    "mfwq_fd_create": (C.c_int, [ip, C.POINTER(dp), C.POINTER(dp), C.c_double, C.POINTER(C.c_void_p)]),
    "mfwq_fd_apply": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "mfwq_fd_eigen": (C.c_int, [C.c_void_p, C.c_int, dp, dp]),
    "mfwq_fd_apply_dir": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                    C.c_int, C.c_int, C.c_void_p]),
    "mfwq_fd_destroy": (None, [C.c_void_p]),
    "mfwq_pcg_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int,
                                 dp, C.POINTER(KrylovReportC), C.c_void_p]),
    "mfwq_nccl_unique_id": (C.c_int, [C.c_char_p, C.c_char_p]),
    "mfwq_comm_create_nccl": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "mfwq_comm_create_local": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "mfwq_comm_info": (C.c_int, [C.c_void_p, ip, ip, ip]),
    "mfwq_comm_destroy": (None, [C.c_void_p]),
    "mfwq_pcg_solve_comm": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.c_void_p, C.POINTER(C.c_void_p),
                                      C.POINTER(C.c_void_p), C.c_double, C.c_int, dp, C.POINTER(KrylovReportC),
                                      C.c_void_p]),
    "mfwq_dot": (C.c_int, [C.c_void_p, C.c_void_p, C.c_longlong, dp, C.c_void_p]),
    "mfwq_dot2": (C.c_int, [C.c_void_p, C.c_void_p, C.c_longlong, dp, C.c_void_p]),
    "mfwq_axpy": (C.c_int, [C.c_void_p, C.c_void_p, C.c_longlong, C.c_double, C.c_void_p]),
    "mfwq_bicg_p": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong, C.c_double, C.c_double, C.c_void_p]),
    "mfwq_bicg_s": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong, C.c_double, dp, C.c_void_p]),
    "mfwq_bicg_xr": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong,
                               C.c_double, C.c_double, dp, C.c_void_p]),
    "mfwq_kron_apply": (C.c_int, [C.c_int, ip, ip, C.POINTER(dp), C.c_void_p, C.c_void_p, C.c_int,
                                  C.c_void_p]),
    "mfwq_quad_create": (C.c_int, [ip, ip, C.POINTER(dp), C.c_int, C.POINTER(C.c_void_p)]),
    "mfwq_quad_sizes": (C.c_int, [C.c_void_p, ip, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]),
    "mfwq_quad_points": (C.c_int, [C.c_void_p, C.c_int, dp, dp]),
    "mfwq_quad_rhs": (C.c_int, [C.c_void_p, C.c_int, dp, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "mfwq_quad_errors": (C.c_int, [C.c_void_p, C.c_int, dp, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_int, dp, C.c_void_p]),
    "mfwq_quad_destroy": (None, [C.c_void_p]),
}

EXPORTED = sorted(_SIGS)


def lib():
    """Load (once) and return the ctypes handle; raises if the .so is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} not built: run `python -m paper_1712_08565_b200.build` "
                "(no CPU fallback exists for the MF-WQ hot path)")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(h, name)
            f.restype = res
            f.argtypes = args
        _lib = h
        _register_lapack(h)
    return _lib


def numpy_lapack():
    """(library path, dgelsd symbol) of the LAPACK numpy's own ``np.linalg.lstsq`` calls, i.e. the
    driver the reference's WQ rows are solved with (wq.py:97), or None if it cannot be found."""
    import glob
    libs = os.path.join(os.path.dirname(os.path.dirname(np.__file__)), "numpy.libs")
    for pat in ("libscipy_openblas64_*.so*",):
        for path in sorted(glob.glob(os.path.join(libs, pat))):
            return path, "scipy_dgelsd_64_"
    return None


def _register_lapack(h):
    """Point the native WQ rule builder at numpy's dgelsd (bit-identical weights to the
    reference); MFWQ_NO_NUMPY_LAPACK=1 keeps the built-in Jacobi SVD (tests of that path)."""
    if os.environ.get("MFWQ_NO_NUMPY_LAPACK") == "1":
        return
    found = numpy_lapack()
    if found is not None:
        h.mfwq_set_lapack(found[0].encode(), found[1].encode())  # best effort: falls back to Jacobi


_CODES = {1: ValueError, 2: WQConstructionError, 3: DegenerateGeometryError, 4: EigenSolveError,
          5: IndefiniteOperatorError, 6: RuntimeError, 7: NotImplementedError, 8: RuntimeError}


def check(rc):
    if rc != 0:
        msg = lib().mfwq_last_error().decode(errors="replace")
        exc = _CODES.get(rc, RuntimeError)
        if exc is WQConstructionError:
            raise exc(-1, float("nan"), msg)
        if exc is DegenerateGeometryError:
            raise exc(None, float("nan"), msg)
        raise exc(msg)


def dptr(a: np.ndarray):
    return a.ctypes.data_as(dp)


def iptr(a: np.ndarray):
    return a.ctypes.data_as(ip)
