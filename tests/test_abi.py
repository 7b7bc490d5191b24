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


def test_host_side_edge_cases():
    """Invalid or empty inputs are rejected before any device work (the
    reference's argument-validation tests, restated for the ABI)."""
    import numpy as np

    from paper_2209_01877_b200 import _lib

    L = _lib.load()
    EINVAL = _lib.HODG_EINVAL
    # element-slot record strides: 20 NQF + 1 (odd) for the CTA element
    # kernel, 20 NQF + 2 for the warp-group kernel; a tile of blocks is a
    # 16-byte multiple at FP32 and FP64
    strides = [L.hodg_elem_record_stride(p) for p in range(4)]
    for p, (s, nqf) in enumerate(zip(strides, (1, 6, 7, 15))):
        assert s in (20 * nqf + 1, 20 * nqf + 2)
        assert (s * L.hodg_elem_tile(p) * 4) % 16 == 0
    assert L.hodg_elem_record_stride(4) == -1 and L.hodg_elem_record_stride(-1) == -1
    assert L.hodg_face_record_stride(2, 16) == -1
    # device mesh setup sizing
    assert L.hodg_mesh_setup_work_bytes(0) == -1 and L.hodg_mesh_setup_work_bytes(1 << 29) == -1
    assert L.hodg_mesh_setup_work_bytes(1000) > 0
    # RCB: bounds and determinism on host
    pts = np.random.default_rng(0).random((10, 3))
    part = np.zeros(10, dtype=np.int32)
    assert L.hodg_partition_rcb(10, pts.ctypes.data, 11, part.ctypes.data) == EINVAL
    assert L.hodg_partition_rcb(0, pts.ctypes.data, 1, part.ctypes.data) == EINVAL
    assert L.hodg_partition_rcb(10, pts.ctypes.data, 0, part.ctypes.data) == EINVAL
    assert L.hodg_partition_rcb(10, pts.ctypes.data, 10, part.ctypes.data) == _lib.HODG_OK
    assert sorted(part.tolist()) == list(range(10))
    # null handles / buffers
    assert L.hodg_face_flux(None, 64, None, None, None, None) == EINVAL
    assert L.hodg_elem_stage(None, 64, None, None, None, None) == EINVAL
    assert L.hodg_halo_exchange(None, None, None) == EINVAL
    assert L.hodg_halo_destroy(None) == _lib.HODG_OK
    assert L.hodg2d_qhat_pass(64, 0, 2, 3, *([None] * 8), 1.4, None, None, None) == EINVAL
    assert L.hodg2d_aux_pass(64, 5, 7, 4, 2, 4, *([None] * 17)) == EINVAL  # nb > 6
