"""ctypes binding of libhodg_b200.so (include/hodg_b200.h).

The library is built in-tree (paper_2209_01877_b200/_build/) by
`__graft_entry__.build()` / `make -C paper_2209_01877_b200/csrc`.  There is
no CPU fallback: every compute entry point raises if the library or a
B200-class (sm_100) device is missing.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HODG_B200_LIB") or os.path.join(_HERE, "_build", "libhodg_b200.so")

HODG_OK, HODG_EINVAL, HODG_ECUDA, HODG_ENODEV = 0, 2, 3, 4
HODG_ETOPOLOGY = 5
PREC_F64, PREC_MIXED = 64, 32
FLUX_ROE, FLUX_LLF = 0, 1
BC_CODES = {"far_field": 1, "slip_wall": 2, "no_slip_wall": 3}

P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int
D = C.c_double


class MeshDesc(C.Structure):
    _fields_ = [
        ("n_elems", C.c_int64),
        ("n_faces", C.c_int64),
        ("order", C.c_int),
        ("flux_kind", C.c_int),
        ("gamma", C.c_double),
        ("qinf", C.c_double * 5),
        ("egeo", P),
        ("econv", P),
        ("efaces", P),
        ("fcells", P),
        ("finfo", P),
        ("fnrm", P),
    ]


class StageArgs(C.Structure):
    _fields_ = [
        ("us", P),
        ("u0", P),
        ("out", P),
        ("res", P),
        ("a", C.c_double),
        ("b", C.c_double),
        ("combine", C.c_int),
        ("dt_is_vector", C.c_int),
        ("dt", P),
        ("norm_partial", P),
        ("dt_next", P),
        ("dt_vec_out", P),
        ("dt_reset", P),
        ("cfl", C.c_double),
        ("out32", P),
    ]


# every symbol declared in include/hodg_b200.h: name -> (restype, argtypes)
SIGNATURES = {
    "hodg_version": (I32, []),
    "hodg_device_ok": (I32, []),
    "hodg_mesh_create": (I32, [C.POINTER(MeshDesc), C.POINTER(P)]),
    "hodg_mesh_destroy": (I32, [P]),
    "hodg_state_row_stride": (I32, [I32]),
    "hodg_n_basis": (I32, [I32]),
    "hodg_n_face_points": (I32, [I32]),
    "hodg_n_vol_points": (I32, [I32]),
    "hodg_elem_tile": (I32, [I32]),
    "hodg_face_record_stride": (I32, [I32, I32]),
    "hodg_stage_blocks": (I64, [P, I32]),
    "hodg_face_flux": (I32, [P, I32, P, P, P, P]),
    "hodg_face_flux_range": (I32, [P, I32, P, P, I64, I64, I32, P, P]),
    "hodg_state32_row_stride": (I32, [I32]),
    "hodg_state_to_f32": (I32, [P, P, I64, P, P]),
    "hodg_face_flux_range32": (I32, [P, P, P, I64, I64, I32, P, P]),
    "hodg_face_flux_range32_es": (I32, [P, P, P, I64, I64, I32, P, P]),
    "hodg_elem_stage": (I32, [P, I32, P, C.POINTER(StageArgs), P, P]),
    "hodg_face_flux_range_es": (I32, [P, I32, P, P, I64, I64, I32, P, P]),
    "hodg_elem_stage_es": (I32, [P, I32, P, C.POINTER(StageArgs), P, P]),
    "hodg_elem_record_stride": (I32, [I32]),
    "hodg_elem_record_len": (I64, [P, I32]),
    "hodg_partition_rcb": (I32, [I64, P, I32, P]),
    "hodg_mesh_setup_work_bytes": (I64, [I64]),
    "hodg_mesh_setup": (I32, [I64, I64] + [P] * 16),
    "hodg_element_records": (I32, [I64, I32] + [P] * 11),
    "hodg_halo_unique_id": (I32, [P]),
    "hodg_halo_create": (I32, [I32, I32, P, I32, P, P, P, P, P, I32, C.POINTER(C.c_void_p)]),
    "hodg_halo_exchange": (I32, [P, P, P]),
    "hodg_halo_allreduce": (I32, [P, P, I64, I32, P]),
    "hodg_halo_destroy": (I32, [P]),
    "hodg_local_dt": (I32, [P, P, D, P, P, P, P]),
    "hodg_norm_finalize": (I32, [P, I64, P, P]),
    "hodg_last_error": (I32, [P]),
    "hodg_residual_l2": (I32, [P, P, P, P, P]),
    "hodg_min_reduce_f64": (I32, [P, I64, P, P, P]),
    "hodg_dt_fill": (I32, [P, D, P]),
    "hodg_modal_transform": (I32, [P, I32, P, P, P]),
    "hodg_err_reset": (I32, [P, P]),
    "hodg_err_decode": (I32, [P, C.POINTER(C.c_int64)]),
    "hodg_rcm_work_bytes": (I64, [I64, I64]),
    "hodg_rcm": (I32, [I64, P, P, P, P, P, P]),
    "hodg_launch_count": (I64, []),
    "hodg_point_flux": (I32, [I32, I64, P, P, P, D, I32, P, P, P]),
    "hodg_point_bstate": (I32, [I32, I64, I32, P, P, P, D, P, P]),
    "hodg_face_sort_work_bytes": (I64, [I64]),
    "hodg_face_sort": (I32, [I64, I64, P, P, P, P]),
    "hodg2d_flux_pass": (I32, [I32, I64, I32, I32, P, P, P, P, P, P, P, P, D, I32, P, P, P]),
    "hodg2d_rhs_pass": (I32, [I32, I64, I32, I32, I32, I32, P, P, P, P, P, P, P, P, P, P, P, P, P, D, P, P, P]),
    "hodg2d_qhat_pass": (I32, [I32, I64, I32, I32, P, P, P, P, P, P, P, P, D, P, P, P]),
    "hodg2d_aux_pass": (I32, [I32, I64, I32, I32, I32, I32] + [P] * 17),
    "hodg2d_flux_pass_ns": (I32, [I32, I64, I32, I32] + [P] * 9 + [D] * 4 + [P] * 5),
    "hodg2d_rhs_pass_ns": (I32, [I32, I64, I32, I32, I32, I32] + [P] * 15 + [D] * 4 + [P] * 3),
    "hodg2d_dt_pass": (I32, [I32, I64, I32, P, P, P, D, D, D, I32, P, P, P]),
    "hodg2d_axpy": (I32, [I32, I64, I32, P, P, P, P, P]),
    "hodg2d_combine": (I32, [I32, I64, I32, P, P, P, P, P, P]),
}

_lib = None


class HodgError(RuntimeError):
    pass


def load():
    """Load the shared library (no device required)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise HodgError(f"libhodg_b200.so not built ({LIB_PATH}); run __graft_entry__.build()")
        lib = C.CDLL(LIB_PATH)
        # an A/B variant library (HODG_B200_LIB) may predate later entry
        # points; the in-tree library must export every declared symbol
        variant = bool(os.environ.get("HODG_B200_LIB"))
        for name, (res, args) in SIGNATURES.items():
            try:
                fn = getattr(lib, name)
            except AttributeError:
                if variant:
                    continue
                raise
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def lib():
    """The library, after checking there is an sm_100 device to run on."""
    L = load()
    import torch

    if not torch.cuda.is_available():
        raise HodgError("no CUDA device: the B200 kernels have no CPU fallback")
    torch.cuda.init()
    if not L.hodg_device_ok():
        raise HodgError("current device is not sm_100 (B200)")
    return L


def check(rc, what):
    if rc != HODG_OK:
        detail = ""
        if rc == HODG_ECUDA:
            try:
                site = C.c_int(0)
                code = lib().hodg_last_error(C.byref(site))
                detail = f" (CUDA error {code} at launcher site {site.value})"
            except Exception:  # noqa: BLE001 -- diagnostics only
                pass
        raise HodgError(f"{what} failed with status {rc}{detail}")


def ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def stream_ptr(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def launch_count() -> int:
    return int(load().hodg_launch_count())
