"""ctypes binding of the oracle C kernels (TEST INFRASTRUCTURE ONLY)."""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_BUILD = os.path.join(_HERE, "_build")


def build():
    """Compile the oracle libraries (make in oracle/)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def _load(name):
    path = os.path.join(_BUILD, name)
    if not os.path.exists(path):
        build()
    return C.CDLL(path)


_lib = None
_rcm = None

P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int
D = C.c_double


def lib():
    global _lib
    if _lib is None:
        _lib = _load("libhodg_oracle.so")
        for sfx in ("_f64", "_f32"):
            getattr(_lib, "ora_flux_pass" + sfx).argtypes = [I32, I64, I32, I32, P, P, P, P, P, P, P, D, I32, P, P]
            getattr(_lib, "ora_rhs_pass" + sfx).argtypes = [I32, I64, I32, I32, I32, I32, P, P, P, P, P, P, P, P,
                                                            P, P, P, P, D, P, P, P]
            getattr(_lib, "ora_dt_pass" + sfx).argtypes = [I32, I64, I32, P, P, P, D, D, D, I32, P, P]
            getattr(_lib, "ora_axpy" + sfx).argtypes = [I64, I32, P, P, P, P]
            getattr(_lib, "ora_combine" + sfx).argtypes = [I64, I32, P, P, P, P, P]
            getattr(_lib, "ora_rk_combo" + sfx).argtypes = [I64, I32, D, D, P, P, P, P, P]
            getattr(_lib, "ora_point_flux" + sfx).argtypes = [I32, I64, P, P, P, D, I32, P, P]
            getattr(_lib, "ora_point_bstate" + sfx).argtypes = [I32, I64, I32, P, P, P, D, P]
            getattr(_lib, "ora_qhat_pass" + sfx).argtypes = [I64, I32, I32, P, P, P, P, P, P, P, P, D, P, P]
            getattr(_lib, "ora_aux_pass" + sfx).argtypes = [I64, I32, I32, I32, I32] + [P] * 17
            getattr(_lib, "ora_flux_pass_ns" + sfx).argtypes = [I64, I32, I32] + [P] * 9 + [D] * 4 + [P] * 4
            getattr(_lib, "ora_rhs_pass_ns" + sfx).argtypes = [I64, I32, I32, I32, I32] + [P] * 15 + [D] * 4 + \
                [P] * 3
        _lib.ora_set_threads.argtypes = [I32]
        _lib.ora_set_threads.restype = I32
    return _lib


def rcm_lib():
    global _rcm
    if _rcm is None:
        _rcm = _load("librcm_oracle.so")
        _rcm.ora_cuthill_mckee.argtypes = [I64, P, P, P]
        _rcm.ora_cuthill_mckee.restype = I32
    return _rcm


def ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(C.c_void_p)


def sfx(dtype) -> str:
    dt = np.dtype(dtype)
    if dt == np.float64:
        return "_f64"
    if dt == np.float32:
        return "_f32"
    raise ValueError(f"unsupported precision {dt}")


def set_threads(n: int) -> int:
    return lib().ora_set_threads(int(n))
