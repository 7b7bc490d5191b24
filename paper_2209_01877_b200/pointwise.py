"""Point evaluations of the device interface physics: the reference's
Python API over its scalar kernels (`roe_flux`, `boundary_state`,
`hodg/physics.py:436-479`), batched on the GPU through `hodg_point_flux` /
`hodg_point_bstate` -- the same device functions the face kernel inlines."""

from __future__ import annotations

import numpy as np

from . import _lib
from .physics import AdmissibilityError, Conserved, GasModel

__all__ = ["point_flux", "point_bstate", "roe_flux", "boundary_state"]

_BC = {"far_field": 1, "slip_wall": 2, "no_slip_wall": 3}


def _dev(a, dtype):
    import torch

    return torch.as_tensor(np.ascontiguousarray(a, dtype=dtype)).cuda()


def point_flux(qL, qR, normals, gamma=1.4, flux="roe", dtype=np.float64):
    """(n, 5) interface fluxes and (n,) ok flags for states (n, 5), unit normals (n, 3)."""
    import torch

    L = _lib.lib()
    a, b, nr = _dev(qL, dtype), _dev(qR, dtype), _dev(normals, dtype)
    n = a.shape[0]
    out = torch.empty_like(a)
    ok = torch.empty(n, dtype=torch.uint8, device=a.device)
    prec = _lib.PREC_F64 if dtype == np.float64 else _lib.PREC_MIXED
    _lib.check(L.hodg_point_flux(prec, n, _lib.ptr(a), _lib.ptr(b), _lib.ptr(nr), float(gamma),
                                 _lib.FLUX_LLF if flux == "llf" else _lib.FLUX_ROE, _lib.ptr(out), _lib.ptr(ok),
                                 _lib.stream_ptr()), "hodg_point_flux")
    return out.cpu().numpy(), ok.cpu().numpy().astype(bool)


def point_bstate(kind, q, normals, freestream, gamma=1.4, dtype=np.float64):
    import torch

    L = _lib.lib()
    a, nr, qf = _dev(q, dtype), _dev(normals, dtype), _dev(freestream, dtype)
    out = torch.empty_like(a)
    code = _BC[kind] if isinstance(kind, str) else int(kind)
    prec = _lib.PREC_F64 if dtype == np.float64 else _lib.PREC_MIXED
    _lib.check(L.hodg_point_bstate(prec, a.shape[0], code, _lib.ptr(a), _lib.ptr(nr), _lib.ptr(qf), float(gamma),
                                   _lib.ptr(out), _lib.stream_ptr()), "hodg_point_bstate")
    return out.cpu().numpy()


def roe_flux(qL: Conserved, qR: Conserved, n, gas: GasModel, flux="roe") -> np.ndarray:
    """hodg/physics.py:436-445 (single state pair, raises on ok = 0)."""
    f, ok = point_flux(qL.as_array()[None], qR.as_array()[None], np.asarray(n, dtype=np.float64)[None], gas.gamma,
                       flux)
    if not ok[0]:
        raise AdmissibilityError("inadmissible state or failed Roe average")
    return f[0]


def boundary_state(q_in: Conserved, kind: str, n, freestream: Conserved, gas: GasModel) -> Conserved:
    """hodg/physics.py:466-479."""
    if kind not in _BC:
        raise ValueError(f"unknown boundary kind {kind!r}")
    q = q_in.as_array()
    p = (gas.gamma - 1.0) * (q[4] - 0.5 * (q[1] ** 2 + q[2] ** 2 + q[3] ** 2) / q[0]) if q[0] > 0 else -1.0
    if not (q[0] > 0.0) or not (p > 0.0):
        raise AdmissibilityError("inadmissible interior state")
    out = point_bstate(kind, q[None], np.asarray(n, dtype=np.float64)[None], freestream.as_array(), gas.gamma)[0]
    return Conserved(*map(float, out))
