"""DG spatial operator on the B200: state containers and the residual API.

Keeps the reference's Python surface (`hodg/dg.py:48-99`, `:549-663`):
`DofState`, `FaceFluxBuffer`, `Residual`, `BoundaryConditions`,
`project_initial`, `face_flux_pass`, `accumulate_rhs`, `rhs`, `cell_means`.
State tensors are torch CUDA tensors in the reference's layout
(n_cells, n_vars, nb) and the reference's physical Taylor basis; the
kernels work in the reference-element basis (refelem.py) and the wrappers
convert with `hodg_modal_transform` on the device.

Precision is dispatched on the state dtype as in the reference
(`hodg/dg.py:496`): float64 runs FP64 kernels, float32 runs the mixed
kernels (FP32 traces / flux / quadrature, FP64 accumulation and mass
solve).  Residuals are always float64.

Errors: the kernels never raise; they record the first inadmissible face /
cell in a device error word that the wrapper reads once per call and turns
into `AdmissibilityError(..., face|cell, iteration)` (`hodg/dg.py:537-546`).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .geometry import DeviceGeometry, volume_points
from .mesh import TetMesh
from .physics import AdmissibilityError, Conserved, GasModel
from .refelem import ref_tables

__all__ = [
    "N_VARS",
    "BoundaryConditions",
    "DofState",
    "FaceFluxBuffer",
    "Residual",
    "Discretization",
    "project_initial",
    "face_flux_pass",
    "accumulate_rhs",
    "rhs",
    "cell_means",
    "density_l2_error",
]

N_VARS = 5
FLUX_KINDS = {"roe": _lib.FLUX_ROE, "llf": _lib.FLUX_LLF}


def _torch():
    import torch

    return torch


@dataclass(frozen=True)
class BoundaryConditions:
    """Far-field freestream state (hodg/dg.py:48-53) and the interface flux."""

    freestream: Conserved
    flux: str = "roe"

    def __post_init__(self):
        if self.flux not in FLUX_KINDS:
            raise ValueError(f"unknown flux {self.flux!r}; expected 'roe' or 'llf'")


@dataclass
class DofState:
    """Per-element modal coefficients (n_cells, 5, nb) in the Taylor basis."""

    coeffs: object
    iteration: int = 0

    @property
    def dtype(self):
        return self.coeffs.dtype

    @property
    def precision_bits(self) -> int:
        return self.coeffs.element_size() * 8

    @property
    def n_basis(self) -> int:
        return self.coeffs.shape[2]

    def copy(self) -> "DofState":
        return DofState(self.coeffs.clone(), self.iteration)


@dataclass
class FaceFluxBuffer:
    """Interface flux at each face quadrature point, (n_faces, nqf, 5)."""

    inviscid: object


@dataclass
class Residual:
    """dQ/dt modal coefficients (n_cells, 5, nb), always float64."""

    res: object


class Discretization:
    """Device handle for one (mesh, geometry, gas, boundary) setup
    (hodg/dg.py:476-534): the C-ABI mesh descriptor over device geometry,
    plus the error word and scratch reused across calls."""

    def __init__(self, mesh: TetMesh, geo: DeviceGeometry, gas: GasModel, bcs: BoundaryConditions, device="cuda",
                 n_elems: int | None = None):
        if gas.ivis:
            raise NotImplementedError("viscous (BR1) terms are not in the B200 path yet; use ivis=0")
        torch = _torch()
        self.L = _lib.lib()
        self.mesh, self.geo, self.gas, self.bcs = mesh, geo, gas, bcs
        self.device = torch.device(device)
        self.order = geo.order
        self.nb = geo.n_basis
        self.nqf = geo.n_face_points
        self.rs = int(self.L.hodg_state_row_stride(self.order))
        # state rows (owned + ghost elements in a partitioned run) vs the
        # elements the element kernel updates (the owned ones, stored first)
        self.n_rows = mesh.n_cells
        self.n = mesh.n_cells if n_elems is None else int(n_elems)
        self.nf = mesh.n_faces
        d = geo.device(self.device)
        self._d = d
        desc = _lib.MeshDesc()
        desc.n_elems = self.n
        desc.n_faces = self.nf
        desc.order = self.order
        desc.flux_kind = FLUX_KINDS[bcs.flux]
        desc.gamma = gas.gamma
        for i, x in enumerate(bcs.freestream.as_array()):
            desc.qinf[i] = float(x)
        desc.egeo = _lib.ptr(d["egeo"])
        desc.econv = _lib.ptr(d["econv"])
        desc.efaces = _lib.ptr(d["efaces"])
        desc.fcells = _lib.ptr(d["fcells"])
        desc.finfo = _lib.ptr(d["finfo"])
        desc.fnrm = _lib.ptr(d["fnrm"])
        self.desc = desc
        h = C.c_void_p()
        _lib.check(self.L.hodg_mesh_create(C.byref(desc), C.byref(h)), "hodg_mesh_create")
        self.handle = h
        self.err = torch.empty(4, dtype=torch.int32, device=self.device)
        self.nblk = int(self.L.hodg_stage_blocks(h, 64))
        self._hbuf = {}
        self._ebuf = {}
        self._scratch = torch.empty(max(self.nblk, (self.n + 255) // 256) * 5 + 1024, dtype=torch.float64,
                                    device=self.device)

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.L.hodg_mesh_destroy(self.handle)
        except Exception:
            pass

    # -- buffers ---------------------------------------------------------
    def face_buffer(self, prec):
        torch = _torch()
        b = self._hbuf.get(prec)
        if b is None:
            dt = torch.float32 if prec == _lib.PREC_MIXED else torch.float64
            hs = int(self.L.hodg_face_record_stride(self.order, prec))
            b = torch.zeros((self.nf, hs), dtype=dt, device=self.device)
            self._hbuf[prec] = b
        return b

    def elem_buffer(self, prec):
        """Element-slot record buffer (include/hodg_b200.h: hodg_face_flux_range_es):
        1-D, so face_flux / stage select the element-slot kernels by shape."""
        torch = _torch()
        b = self._ebuf.get(prec)
        if b is None:
            dt = torch.float32 if prec == _lib.PREC_MIXED else torch.float64
            b = torch.zeros(int(self.L.hodg_elem_record_len(self.handle, prec)), dtype=dt, device=self.device)
            self._ebuf[prec] = b
        return b

    def new_state(self, rows=None):
        return _torch().zeros((self.n_rows if rows is None else rows, self.rs), dtype=_torch().float64,
                              device=self.device)

    # -- basis conversions -------------------------------------------------
    def to_reference(self, coeffs, out=None):
        """(n, 5, nb) Taylor coefficients -> (n, rs) reference-basis rows."""
        torch = _torch()
        c = torch.as_tensor(coeffs, device=self.device).to(torch.float64)
        if tuple(c.shape) != (self.n, N_VARS, self.nb):
            raise ValueError(f"state shape {tuple(c.shape)} != {(self.n, N_VARS, self.nb)}")
        if self.rs == N_VARS * self.nb and self.n_rows == self.n and c.is_contiguous():
            src = c  # the (5, nb) blocks already are the kernel's rows: no staging copy
        else:
            src = self.new_state()
            src[: self.n, : N_VARS * self.nb] = c.reshape(self.n, -1)
        out = self.new_state() if out is None else out
        _lib.check(self.L.hodg_modal_transform(self.handle, 1, _lib.ptr(src), _lib.ptr(out), _lib.stream_ptr()),
                   "hodg_modal_transform")
        return out

    def from_reference(self, rows):
        """(n, rs) reference-basis rows -> (n, 5, nb) Taylor coefficients."""
        out = self.new_state()
        _lib.check(self.L.hodg_modal_transform(self.handle, 0, _lib.ptr(rows), _lib.ptr(out), _lib.stream_ptr()),
                   "hodg_modal_transform")
        # a fresh buffer: a view of it never aliases the caller's rows
        return out[: self.n, : N_VARS * self.nb].reshape(self.n, N_VARS, self.nb).contiguous()

    # -- kernels -----------------------------------------------------------
    def reset_errors(self):
        _lib.check(self.L.hodg_err_reset(_lib.ptr(self.err), _lib.stream_ptr()), "hodg_err_reset")

    def raise_errors(self, iteration=None):
        """Read the error word (one device sync) and raise the reference's
        exception for the first flagged face / cell."""
        host = self.err.cpu().numpy().astype(np.uint32)
        idv = C.c_int64(-1)
        kind = self.L.hodg_err_decode(host.ctypes.data_as(C.c_void_p), C.byref(idv))
        if kind == 1:
            raise AdmissibilityError("inadmissible face trace", face=int(idv.value), iteration=iteration)
        if kind == 2:
            raise AdmissibilityError("inadmissible volume state", cell=int(idv.value), iteration=iteration)
        if kind == 3:
            raise AdmissibilityError("inadmissible cell mean", cell=int(idv.value), iteration=iteration)

    def face_segments(self, f_begin=0, f_end=None):
        """The face-kernel launches over [f_begin, f_end): (lo, hi, interior_only)."""
        f_end = self.nf if f_end is None else f_end
        g = self.geo
        b0, b1 = g.n_int0, g.n_int0 + g.n_bnd
        segs = [(max(lo, f_begin), min(hi, f_end), interior)
                for lo, hi, interior in ((0, b0, 1), (b0, b1, 0), (b1, self.nf, 1))]
        segs = [sg for sg in segs if sg[1] > sg[0]]
        if len(segs) >= 2 and segs[-2][2] == 0:
            # boundary range + partition tail: one launch of the general
            # variant (it treats interior faces exactly as the interior one)
            segs[-2:] = [(segs[-2][0], segs[-1][1], 0)]
        return segs

    def face_flux(self, rows, prec, hbuf=None, stream=None, f_begin=0, f_end=None):
        """Face kernel over device faces [f_begin, f_end): interior ranges use
        the kernel variant without boundary states, the boundary range the
        general one (extended over a partition tail that follows it: one
        launch fewer)."""
        hbuf = self.face_buffer(prec) if hbuf is None else hbuf
        for lo, hi, interior in self.face_segments(f_begin, f_end):
            fn = self.L.hodg_face_flux_range_es if hbuf.dim() == 1 else self.L.hodg_face_flux_range
            _lib.check(fn(self.handle, prec, _lib.ptr(rows), _lib.ptr(hbuf), int(lo), int(hi), interior,
                          _lib.ptr(self.err), _lib.stream_ptr(stream)), "hodg_face_flux_range")
        return hbuf

    # -- mixed precision: the FP32 shadow of the state ----------------------
    @property
    def rs32(self) -> int:
        return int(self.L.hodg_state32_row_stride(self.order))

    def new_state32(self, rows=None):
        return _torch().zeros((self.n_rows if rows is None else rows, self.rs32), dtype=_torch().float32,
                              device=self.device)

    def shadow_of(self, rows, out32):
        """FP32 shadow of FP64 state rows (all rows, ghosts included)."""
        _lib.check(self.L.hodg_state_to_f32(self.handle, _lib.ptr(rows), rows.shape[0], _lib.ptr(out32),
                                            _lib.stream_ptr()), "hodg_state_to_f32")
        return out32

    def face_flux32(self, rows32, hbuf, stream=None, f_begin=0, f_end=None):
        """Mixed-precision face kernel reading the FP32 shadow rows."""
        for lo, hi, interior in self.face_segments(f_begin, f_end):
            fn = self.L.hodg_face_flux_range32_es if hbuf.dim() == 1 else self.L.hodg_face_flux_range32
            _lib.check(fn(self.handle, _lib.ptr(rows32), _lib.ptr(hbuf), int(lo), int(hi), interior,
                          _lib.ptr(self.err), _lib.stream_ptr(stream)), "hodg_face_flux_range32")
        return hbuf

    def face_flux_split(self, rows, prec, hbuf, side, rows32=None):
        """face_flux over all faces with the boundary (+ partition) range on
        the `side` stream, issued after the interior range: its CTAs take the
        SM slots the persistent interior kernel frees in its tail instead of
        running as a separate, mostly-ramp launch afterwards.  Joined back
        into the current stream."""
        torch = _torch()
        segs = self.face_segments()

        def run(stream=None, f_begin=0, f_end=None):
            if rows32 is not None:
                self.face_flux32(rows32, hbuf, stream=stream, f_begin=f_begin, f_end=f_end)
            else:
                self.face_flux(rows, prec, hbuf, stream=stream, f_begin=f_begin, f_end=f_end)

        if side is None or len(segs) < 2:
            run()
            return hbuf
        cur = torch.cuda.current_stream()
        side.wait_stream(cur)
        run(f_begin=segs[0][0], f_end=segs[0][1])
        run(stream=side, f_begin=segs[1][0], f_end=self.nf)
        cur.wait_stream(side)
        return hbuf

    def stage(self, prec, hbuf, args: _lib.StageArgs, stream=None):
        fn = self.L.hodg_elem_stage_es if hbuf.dim() == 1 else self.L.hodg_elem_stage
        _lib.check(fn(self.handle, prec, _lib.ptr(hbuf), C.byref(args), _lib.ptr(self.err),
                                          _lib.stream_ptr(stream)), "hodg_elem_stage")

    def residual_rows(self, rows, hbuf, prec, res=None):
        res = self.new_state() if res is None else res
        a = _lib.StageArgs()
        a.us = _lib.ptr(rows)
        a.res = _lib.ptr(res)
        a.combine = -1
        self.stage(prec, hbuf, a)
        return res


def _get_disc(mesh, geo, gas, bcs) -> Discretization:
    key = (id(mesh), gas, bcs)
    disc = geo._disc_cache.get(key)
    if disc is None:
        disc = Discretization(mesh, geo, gas, bcs)
        geo._disc_cache[key] = disc
    return disc


def _prec_of(state) -> int:
    torch = _torch()
    if state.coeffs.dtype == torch.float64:
        return _lib.PREC_F64
    if state.coeffs.dtype == torch.float32:
        return _lib.PREC_MIXED
    raise ValueError(f"unsupported precision {state.coeffs.dtype}")


def project_initial(mesh: TetMesh, geo: DeviceGeometry, field, gas: GasModel, device="cuda") -> DofState:
    """L2 projection of a primitive field onto the basis (hodg/dg.py:549-569).
    `field(x, y, z)` gets flat arrays over all volume quadrature points and
    returns a Primitive of arrays.  In the reference-element basis the
    projector is one constant (nb x nqv) matrix for every element."""
    torch = _torch()
    t = ref_tables(geo.order)
    xyz = volume_points(mesh, geo.order)
    w = field(xyz[..., 0].ravel(), xyz[..., 1].ravel(), xyz[..., 2].ravel())
    shape = xyz.shape[:2]
    rho, u, v, ww, p = (np.broadcast_to(np.asarray(a, dtype=np.float64), (shape[0] * shape[1],)).reshape(shape)
                        for a in (w.rho, w.u, w.v, w.w, w.p))
    if np.any(rho <= 0.0) or np.any(p <= 0.0):
        raise AdmissibilityError("initial field is inadmissible")
    disc = _get_disc(mesh, geo, gas, BoundaryConditions(Conserved(1.0, 0.0, 0.0, 0.0, 1.0)))
    # conserved variables and the projection on the device (the callback is
    # the reference's host API; the rest is one batched contraction)
    dev = disc.device
    rho_d, u_d, v_d, w_d, p_d = (torch.from_numpy(np.array(a, dtype=np.float64)).to(dev) for a in (rho, u, v, ww, p))
    e = p_d / (gas.gamma - 1.0) + 0.5 * rho_d * (u_d * u_d + v_d * v_d + w_d * w_d)
    q = torch.stack([rho_d, rho_d * u_d, rho_d * v_d, rho_d * w_d, e], dim=-1)  # (n, nqv, 5)
    proj = torch.from_numpy(t.projector).to(dev)
    ref = torch.einsum("iq,nqv->nvi", proj, q)  # (n, 5, nb) reference basis
    rows = disc.new_state()
    rows[: mesh.n_cells, : N_VARS * t.nb] = ref.reshape(mesh.n_cells, -1)
    return DofState(disc.from_reference(rows))


def face_flux_pass(state: DofState, aux, mesh: TetMesh, geo: DeviceGeometry, bcs: BoundaryConditions,
                   gas: GasModel) -> FaceFluxBuffer:
    """Interface fluxes at every face quadrature point (hodg/dg.py:594-621)."""
    if aux is not None:
        raise NotImplementedError("viscous auxiliary gradients are not in the B200 path")
    disc = _get_disc(mesh, geo, gas, bcs)
    prec = _prec_of(state)
    rows = disc.to_reference(state.coeffs)
    disc.reset_errors()
    hbuf = disc.face_flux(rows, prec, hbuf=_torch().empty_like(disc.face_buffer(prec)))
    disc.raise_errors(state.iteration)
    h = hbuf[:, : N_VARS * disc.nqf].reshape(disc.nf, N_VARS, disc.nqf)
    inv = _torch().as_tensor(geo.face_inv, device=disc.device)
    return FaceFluxBuffer(inviscid=h.index_select(0, inv).transpose(1, 2))  # mesh face order


def accumulate_rhs(state: DofState, aux, fluxes: FaceFluxBuffer, mesh: TetMesh, geo: DeviceGeometry,
                   bcs: BoundaryConditions, gas: GasModel) -> Residual:
    """Volume terms plus the gather of stored face fluxes (hodg/dg.py:624-649)."""
    torch = _torch()
    disc = _get_disc(mesh, geo, gas, bcs)
    prec = _prec_of(state)
    rows = disc.to_reference(state.coeffs)
    dt = torch.float32 if prec == _lib.PREC_MIXED else torch.float64
    hbuf = torch.zeros_like(disc.face_buffer(prec))
    perm = torch.as_tensor(geo.face_perm, device=disc.device)
    h = torch.as_tensor(fluxes.inviscid, device=disc.device).to(dt).index_select(0, perm)  # device face order
    hbuf[:, : N_VARS * disc.nqf] = h.transpose(1, 2).reshape(disc.nf, -1)
    disc.reset_errors()
    res = disc.residual_rows(rows, hbuf, prec)
    disc.raise_errors(state.iteration)
    return Residual(res=disc.from_reference(res))


def rhs(state: DofState, mesh: TetMesh, geo: DeviceGeometry, bcs: BoundaryConditions, gas: GasModel) -> Residual:
    """Full spatial residual: face-flux pass then element accumulation
    (hodg/dg.py:652-663)."""
    disc = _get_disc(mesh, geo, gas, bcs)
    prec = _prec_of(state)
    rows = disc.to_reference(state.coeffs)
    disc.reset_errors()
    hbuf = disc.face_flux(rows, prec)
    res = disc.residual_rows(rows, hbuf, prec)
    disc.raise_errors(state.iteration)
    return Residual(res=disc.from_reference(res))


def cell_means(state: DofState, geo: DeviceGeometry):
    """Cell-average conserved state (n_cells, 5) float64 (hodg/dg.py:666-668):
    the mean of the reference-basis expansion."""
    disc = next(iter(geo._disc_cache.values()), None)
    if disc is None:
        raise RuntimeError("no discretization bound to this geometry yet")
    rows = disc.to_reference(state.coeffs)
    t = ref_tables(geo.order)
    mean = _torch().from_numpy(t.MEAN).to(disc.device)
    return rows[:, : N_VARS * t.nb].reshape(disc.n, N_VARS, t.nb) @ mean


def density_l2_error(state: DofState, mesh: TetMesh, geo: DeviceGeometry, rho_exact) -> float:
    """Quadrature L2 norm of the density error against rho_exact(x, y, z)
    (hodg/dg.py:671-677), evaluating the Taylor expansion at the volume
    quadrature points."""
    from .basis import exponents
    from .refelem import monomials

    t = ref_tables(geo.order)
    pts = volume_points(mesh, geo.order)
    X = (pts - mesh.cell_centroid[:, None, :]) / mesh.cell_h[:, None, None]
    B = monomials(exponents(3, geo.order), X)
    c = state.coeffs[:, 0, :].double().cpu().numpy()
    rho_h = np.einsum("nqj,nj->nq", B, c)
    err = rho_h - rho_exact(pts[..., 0], pts[..., 1], pts[..., 2])
    w = t.vol_weights[None, :] * mesh.cell_area[:, None]
    return float(np.sqrt(np.sum(w * err * err)))
