"""The C-ABI library loads without a GPU and exports every symbol declared
in include/hodg_b200.h; host-side argument checks need no device."""

import ctypes as C
import os
import re

from conftest import ROOT


def declared_symbols():
    with open(os.path.join(ROOT, "include", "hodg_b200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^\s*(?:int64_t|int)\s+(hodg\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_seam():
    syms = declared_symbols()
    for need in ("hodg_face_flux", "hodg_elem_stage", "hodg_local_dt", "hodg_min_reduce_f64",
                 "hodg_residual_l2", "hodg_rcm", "hodg_mesh_create", "hodg_err_decode"):
        assert need in syms


def test_library_exports_every_declared_symbol():
    from paper_2209_01877_b200 import _lib

    lib = _lib.load()
    for s in declared_symbols():
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, s


def test_host_side_argument_checks():
    from paper_2209_01877_b200 import _lib

    L = _lib.load()
    assert L.hodg_version() >= 1
    assert [L.hodg_n_basis(p) for p in range(4)] == [1, 4, 10, 20]
    assert [L.hodg_state_row_stride(p) for p in range(4)] == [6, 20, 50, 100]
    assert L.hodg_n_basis(4) == -1
    from paper_2209_01877_b200.geometry import TILE

    assert [L.hodg_elem_tile(p) for p in range(4)] == [TILE[p] for p in range(4)]
    assert [L.hodg_face_record_stride(p, 64) for p in range(4)] == [6, 30, 36, 76]
    assert [L.hodg_face_record_stride(p, 32) for p in range(4)] == [8, 32, 36, 76]
    h = C.c_void_p()
    d = _lib.MeshDesc()
    d.order = 7
    assert L.hodg_mesh_create(C.byref(d), C.byref(h)) == _lib.HODG_EINVAL
    err = (C.c_uint32 * 4)(0xFFFFFFFF, 12, 0xFFFFFFFF, 0xFFFFFFFF)
    idv = C.c_int64()
    assert L.hodg_err_decode(err, C.byref(idv)) == 2 and idv.value == 12
    ok = (C.c_uint32 * 4)(0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF)
    assert L.hodg_err_decode(ok, C.byref(idv)) == 0
