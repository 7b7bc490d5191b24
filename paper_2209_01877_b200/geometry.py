"""Compact per-element / per-face geometry for the device kernels.

Replaces the reference's per-cell x per-quadrature-point tables
(`hodg/geometry.py:33-220`; about 8 GB at one million P2 tetrahedra) by
16 doubles per element and 4 per face:

  egeo  16 fields: J^-1 (row-major, 9), fc[s] = sgn_s * area_s / vol (4), h, vol, 0
  econv (N, 18): A = J / h and A^-1 (modal transforms to/from the Taylor basis)
  efaces 4 fields: face id of local face s
  fcells (F, 2), finfo (F,) = slotL | slotR << 2 | bc << 4, fnrm (F, 4)

egeo and efaces are stored tile-major, [tile][field][T] with T elements per
element-kernel CTA (TILE below == hodg_elem_tile), so one tile is one TMA
bulk copy and every per-field shared-memory read is unit-stride.

with J = [V1 - V0, V2 - V0, V3 - V0] (vertices ascending) the affine map of
the reference tetrahedron.  Everything else is a compile-time constant of
the order (refelem.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .mesh import TetMesh
from .refelem import ref_tables

__all__ = ["GeometryError", "DeviceGeometry", "compute_geometry", "volume_points", "TILE", "tile_major"]

class _Tiles:
    """Elements per element-kernel CTA (hodg_kernels.cuh: E), as compiled into
    libhodg_b200 (hodg_elem_tile); the built-in table if the library is not
    built yet (host-only use)."""

    _default = {0: 64, 1: 32, 2: 32, 3: 32}

    def __init__(self):
        self._cache = {}

    def __getitem__(self, order: int) -> int:
        t = self._cache.get(order)
        if t is None:
            try:
                from . import _lib

                t = int(_lib.load().hodg_elem_tile(int(order)))
            except Exception:
                t = self._default[order]
            if t <= 0:
                raise KeyError(order)
            self._cache[order] = t
        return t


TILE = _Tiles()


def tile_major(a: np.ndarray, tile: int) -> np.ndarray:
    """(N, F) -> flat [ceil(N/tile)][F][tile], zero padded."""
    n, nf = a.shape
    nt = (n + tile - 1) // tile
    pad = np.zeros((nt * tile, nf), dtype=a.dtype)
    pad[:n] = a
    return np.ascontiguousarray(pad.reshape(nt, tile, nf).transpose(0, 2, 1)).ravel()


def _devkey(device) -> str:
    import torch

    d = torch.device(device)
    if d.type == "cuda" and d.index is None:
        d = torch.device("cuda", torch.cuda.current_device())
    return str(d)


class GeometryError(Exception):
    pass


@dataclass
class DeviceGeometry:
    order: int
    n_basis: int
    egeo: np.ndarray
    econv: np.ndarray
    efaces: np.ndarray
    fcells: np.ndarray
    finfo: np.ndarray
    fnrm: np.ndarray
    face_perm: np.ndarray = None  # device face k is mesh face face_perm[k]
    face_inv: np.ndarray = None  # mesh face j is device face face_inv[j]
    n_int0: int = 0  # device faces [0, n_int0): interior
    n_bnd: int = 0  # [n_int0, n_int0 + n_bnd): boundary; the rest: interior (partition faces)
    _dev: dict = field(default_factory=dict, repr=False)
    _disc_cache: dict = field(default_factory=dict, repr=False)

    @property
    def n_vol_points(self) -> int:
        return ref_tables(self.order).nqv

    @property
    def n_face_points(self) -> int:
        return ref_tables(self.order).nqf

    def device(self, device="cuda"):
        """Device copies (torch tensors), uploaded once per device."""
        import torch

        d = self._dev.setdefault(_devkey(device), {})
        for k in ("egeo", "econv", "efaces", "fcells", "finfo", "fnrm"):
            if k not in d:
                d[k] = torch.from_numpy(np.ascontiguousarray(getattr(self, k))).to(device)
        return d

    def constant_count(self) -> int:
        n = 0
        for k in ("egeo", "econv", "fnrm"):
            a = getattr(self, k)
            n += a.size if a is not None else next(d[k].numel() for d in self._dev.values() if k in d)
        return n


def element_jacobians(mesh: TetMesh):
    V = mesh.node_xy[mesh.cell_nodes.astype(np.int64)]
    J = np.stack([V[:, 1] - V[:, 0], V[:, 2] - V[:, 0], V[:, 3] - V[:, 0]], axis=2)  # J[:, d, k]
    return V, J


def compute_geometry(mesh: TetMesh, order: int, split: int | None = None, device=None) -> DeviceGeometry:
    """Device geometry.  Faces are laid out [interior | boundary | interior
    tail]: mesh faces [0, split) split into interior then boundary faces
    (order kept within each class), mesh faces [split, F) -- a partition's
    ghost faces, all interior -- after them; the interior ranges run the
    face-kernel variant without boundary-state code.

    device="cuda": the element records (egeo, econv) are built on the GPU by
    hodg_element_records and kept there only (geo.egeo / geo.econv are None);
    J^-1 agrees with the host's LAPACK inverse to a few ulp."""
    if order not in (0, 1, 2, 3):
        raise GeometryError(f"unsupported order {order}; expected 0..3")
    codes = mesh.boundary_kind_codes()
    if np.any(codes < 0):
        raise GeometryError(f"boundary face {int(np.flatnonzero(codes < 0)[0])} has no boundary patch")
    n = mesh.n_cells
    if device is not None:
        return _with_face_layout(mesh, order, split, codes, None, None, _device_records(mesh, order, device))
    V, J = element_jacobians(mesh)
    det = np.linalg.det(J)
    if np.any(np.abs(det) <= 0.0):
        raise GeometryError("degenerate element")
    Jinv = np.linalg.inv(J)
    vol = mesh.cell_area
    h = mesh.cell_h
    fc = mesh.cell_fsign * mesh.face_length[mesh.cell_faces] / vol[:, None]
    egeo = np.zeros((n, 16))
    egeo[:, 0:9] = Jinv.reshape(n, 9)
    egeo[:, 9:13] = fc
    egeo[:, 13] = h
    egeo[:, 14] = vol
    econv = np.empty((n, 18))
    econv[:, 0:9] = (J / h[:, None, None]).reshape(n, 9)
    econv[:, 9:18] = (Jinv * h[:, None, None]).reshape(n, 9)
    return _with_face_layout(mesh, order, split, codes, egeo, econv, None)


def _device_records(mesh: TetMesh, order: int, device):
    """(egeo, econv) device tensors from hodg_element_records."""
    import torch

    from . import _lib

    L = _lib.lib()
    dev = torch.device(device)
    n, T = mesh.n_cells, TILE[order]
    up = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev)  # noqa: E731
    X = up(mesh.node_xy, np.float64)
    tets = up(mesh.cell_nodes, np.int32)
    vol, h = up(mesh.cell_area, np.float64), up(mesh.cell_h, np.float64)
    area = up(mesh.face_length, np.float64)
    cf, fs = up(mesh.cell_faces, np.int32), up(mesh.cell_fsign, np.int8)
    egeo = torch.empty(((n + T - 1) // T) * 16 * T, dtype=torch.float64, device=dev)
    econv = torch.empty((n, 18), dtype=torch.float64, device=dev)
    flag = torch.empty(1, dtype=torch.int32, device=dev)
    rc = L.hodg_element_records(n, order, *[_lib.ptr(t) for t in (X, tets, vol, h, area, cf, fs, egeo, econv, flag)],
                                _lib.stream_ptr())
    if rc == _lib.HODG_ETOPOLOGY:
        raise GeometryError("degenerate element")
    _lib.check(rc, "hodg_element_records")
    return {"egeo": egeo, "econv": econv}


def _with_face_layout(mesh, order, split, codes, egeo, econv, dev_records):
    F = mesh.n_faces
    split = F if split is None else int(split)
    ids = np.arange(F)
    bnd = mesh.face_cells[:, 1] < 0
    if np.any(bnd[split:]):
        raise GeometryError("faces past the split must be interior")
    head = ids[:split]
    perm = np.concatenate([head[~bnd[:split]], head[bnd[:split]], ids[split:]])
    inv = np.empty(F, dtype=np.int64)
    inv[perm] = np.arange(F)
    slots = mesh.face_slots.astype(np.int32)[perm]
    finfo = (slots[:, 0] | (np.maximum(slots[:, 1], 0) << 2) | (codes[perm].astype(np.int32) << 4)).astype(np.int32)
    fnrm = np.zeros((F, 4))
    fnrm[:, :3] = mesh.face_normal[perm]
    T = TILE[order]
    efaces = inv[mesh.cell_faces.astype(np.int64)].astype(np.int32)
    efaces[mesh.cell_faces < 0] = 0
    geo = DeviceGeometry(order, ref_tables(order).nb, None if egeo is None else tile_major(egeo, T), econv,
                         tile_major(efaces, T), mesh.face_cells.astype(np.int32)[perm], finfo, fnrm, perm, inv,
                         int(np.count_nonzero(~bnd[:split])), int(np.count_nonzero(bnd[:split])))
    if dev_records is not None:
        geo._dev[_devkey(dev_records["egeo"].device)] = dict(dev_records)
    return geo


def volume_points(mesh: TetMesh, order: int) -> np.ndarray:
    """(N, nqv, 3) physical volume quadrature points, x = V0 + J xi."""
    V, J = element_jacobians(mesh)
    xi = ref_tables(order).vol_points[:, 1:4]
    return V[:, None, 0, :] + np.einsum("ndk,qk->nqd", J, xi)
