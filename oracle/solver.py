"""Oracle solver driver (TEST INFRASTRUCTURE ONLY).

Restates the reference's residual wrappers and time integration:
  * flows / projection       hodg/flows.py:23-57, hodg/dg.py:549-569
  * face / cell passes       hodg/dg.py:594-663 (C kernels in hodg_oracle.c)
  * dt, min, RK2, residual   hodg/timestepping.py:105-211
  * iteration driver         hodg/timestepping.py:256-357
  * precision control        hodg/precision.py:51-115
  * residual CSV             hodg/output.py:17-28
3D additions (no reference): 5 variables, SSP-RK3, LLF flux option.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _clib
from .geometry import compute_tables


class AdmissibilityError(Exception):
    """Mirror of hodg.physics.AdmissibilityError (hodg/physics.py:59-73)."""

    def __init__(self, message, cell=None, face=None, iteration=None):
        parts = [message]
        if cell is not None:
            parts.append(f"cell {cell}")
        if face is not None:
            parts.append(f"face {face}")
        if iteration is not None:
            parts.append(f"iteration {iteration}")
        super().__init__(", ".join(parts))
        self.cell, self.face, self.iteration = cell, face, iteration


class SolverDivergedError(RuntimeError):
    def __init__(self, iteration, history):
        super().__init__(f"non-finite residual at iteration {iteration}")
        self.iteration, self.history = iteration, history


@dataclass(frozen=True)
class Gas:
    gamma: float = 1.4
    R: float = 1.0
    mu: float = 0.0
    Pr: float = 0.72
    ivis: int = 0  # 1: Navier-Stokes with BR1 viscous terms (2D; hodg/physics.py:76-100)


# ---------------------------------------------------------------------------
# flows (hodg/flows.py)


def freestream_primitive(gas, mach, angle_deg, dim=2):
    rho = 1.0
    T = 1.0
    p = rho * gas.R * T
    a = np.sqrt(gas.gamma * gas.R * T)
    ang = np.deg2rad(angle_deg)
    u = mach * a * np.cos(ang)
    v = mach * a * np.sin(ang)
    return (rho, u, v, 0.0, p) if dim == 3 else (rho, u, v, p)


def freestream_conserved(gas, mach, angle_deg, dim=2):
    if dim == 3:
        rho, u, v, w, p = freestream_primitive(gas, mach, angle_deg, 3)
        e = p / (gas.gamma - 1.0) + 0.5 * rho * (u * u + v * v + w * w)
        return np.array([rho, rho * u, rho * v, rho * w, e])
    rho, u, v, p = freestream_primitive(gas, mach, angle_deg, 2)
    e = p / (gas.gamma - 1.0) + 0.5 * rho * (u * u + v * v)
    return np.array([rho, rho * u, rho * v, e])


def vortex_primitive(gas, mach, angle_deg, beta, x0, y0, t, x, y, dim=2):
    """hodg/flows.py:38-53; in 3D the vortex is a tube along z (w = 0)."""
    inf = freestream_primitive(gas, mach, angle_deg, 2)
    uinf, vinf = inf[1], inf[2]
    xr = np.asarray(x, dtype=np.float64) - x0 - uinf * t
    yr = np.asarray(y, dtype=np.float64) - y0 - vinf * t
    r2 = xr * xr + yr * yr
    g = gas.gamma
    vel_scale = np.sqrt(gas.R)
    env = np.exp(0.5 * (1.0 - r2))
    u = uinf - beta / (2.0 * np.pi) * yr * env * vel_scale
    v = vinf + beta / (2.0 * np.pi) * xr * env * vel_scale
    T = 1.0 - (g - 1.0) * beta * beta / (8.0 * g * np.pi * np.pi) * np.exp(1.0 - r2)
    rho = T ** (1.0 / (g - 1.0))
    p = rho * gas.R * T
    if dim == 3:
        return rho, u, v, np.zeros_like(u), p
    return rho, u, v, p


def pulse_primitive(gas, amplitude, sigma, x0, y0, x, y, mach=0.0, angle_deg=0.0, dim=2):
    """hodg/flows.py:60-73; in 3D a tube along z (w = 0)."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    r2 = (x - x0) ** 2 + (y - y0) ** 2
    p_inf = gas.R
    p = p_inf * (1.0 + amplitude * np.exp(-0.5 * r2 / (sigma * sigma)))
    rho = (p / p_inf) ** (1.0 / gas.gamma)
    if mach > 0.0:
        inf = freestream_primitive(gas, mach, angle_deg, 2)
        u, v = np.full_like(p, inf[1]), np.full_like(p, inf[2])
    else:
        u, v = np.zeros_like(p), np.zeros_like(p)
    if dim == 3:
        return rho, u, v, np.zeros_like(p), p
    return rho, u, v, p


def project_initial(mesh, tab, field, gas):
    """hodg/dg.py:549-569: L2 projection; field(x, y[, z]) -> primitives."""
    xs = [tab.vol_xy[:, :, d].ravel() for d in range(mesh.dim)]
    prim = field(*xs)
    prim = [np.broadcast_to(np.asarray(a, dtype=np.float64), xs[0].shape) for a in prim]
    if mesh.dim == 3:
        rho, u, v, w, p = prim
        if np.any(rho <= 0.0) or np.any(p <= 0.0):
            raise AdmissibilityError("initial field is inadmissible")
        e = p / (gas.gamma - 1.0) + 0.5 * rho * (u * u + v * v + w * w)
        q = np.stack([rho, rho * u, rho * v, rho * w, e], axis=-1)
    else:
        rho, u, v, p = prim
        if np.any(rho <= 0.0) or np.any(p <= 0.0):
            raise AdmissibilityError("initial field is inadmissible")
        e = p / (gas.gamma - 1.0) + 0.5 * rho * (u * u + v * v)
        q = np.stack([rho, rho * u, rho * v, e], axis=-1)
    nv = q.shape[-1]
    q = q.reshape(mesh.n_cells, tab.n_vol_points, nv)
    proj = np.einsum("cq,cqj,cqv->cvj", tab.vol_w, tab.vol_basis, q)
    return np.ascontiguousarray(np.einsum("cjk,cvk->cvj", tab.minv, proj))


# ---------------------------------------------------------------------------
# residual


class Disc:
    """Kernel-ready views of one setup (hodg/dg.py:476-534)."""

    def __init__(self, mesh, tab, gas, qinf, flux_kind=0):
        self.mesh, self.tab, self.gas = mesh, tab, gas
        self.qinf = np.asarray(qinf, dtype=np.float64)
        self.flux_kind = flux_kind
        self.bc = mesh.bc_codes()
        if np.any(self.bc < 0):
            raise ValueError("boundary face without a patch")
        self.nv = 5 if mesh.dim == 3 else 4
        self._per = {}

    def bundle(self, dtype):
        dt = np.dtype(dtype)
        b = self._per.get(dt)
        if b is None:
            b = self.tab.cast(dt)
            b["normal"] = np.ascontiguousarray(self.mesh.face_normal.T, dtype=dt)
            b["qinf"] = self.qinf.astype(dt)
            self._per[dt] = b
        return b

    def flux_pass(self, coeffs, iteration=None):
        m, t = self.mesh, self.tab
        b = self.bundle(coeffs.dtype)
        finv = np.zeros((m.n_faces, t.n_face_points, self.nv), dtype=coeffs.dtype)
        errf = np.zeros(m.n_faces, dtype=np.uint8)
        getattr(_clib.lib(), "ora_flux_pass" + _clib.sfx(coeffs.dtype))(
            m.dim, m.n_faces, t.n_face_points, t.n_basis, _clib.ptr(coeffs), _clib.ptr(b["face_basis_l"]),
            _clib.ptr(b["face_basis_r"]), _clib.ptr(m.face_cells), _clib.ptr(self.bc), _clib.ptr(b["normal"]),
            _clib.ptr(b["qinf"]), self.gas.gamma, self.flux_kind, _clib.ptr(finv), _clib.ptr(errf))
        if errf.any():
            raise AdmissibilityError("inadmissible face trace", face=int(np.nonzero(errf)[0][0]), iteration=iteration)
        return finv

    def rhs_pass(self, coeffs, finv, iteration=None):
        m, t = self.mesh, self.tab
        b = self.bundle(coeffs.dtype)
        res = np.empty((m.n_cells, self.nv, t.n_basis))
        scratch = np.zeros_like(res)
        errc = np.zeros(m.n_cells, dtype=np.uint8)
        getattr(_clib.lib(), "ora_rhs_pass" + _clib.sfx(coeffs.dtype))(
            m.dim, m.n_cells, t.n_basis, t.n_vol_points, t.n_face_points, m.cell_faces.shape[1], _clib.ptr(coeffs),
            _clib.ptr(finv), _clib.ptr(b["vol_w"]), _clib.ptr(b["vol_basis"]), _clib.ptr(b["vol_grad"]),
            _clib.ptr(m.cell_nfaces), _clib.ptr(m.cell_faces), _clib.ptr(m.cell_fsign), _clib.ptr(b["face_w"]),
            _clib.ptr(b["face_basis_l"]), _clib.ptr(b["face_basis_r"]), _clib.ptr(t.minv), self.gas.gamma,
            _clib.ptr(scratch), _clib.ptr(res), _clib.ptr(errc))
        if errc.any():
            raise AdmissibilityError("inadmissible volume state", cell=int(np.nonzero(errc)[0][0]), iteration=iteration)
        return res

    # -- viscous (BR1) terms, hodg/dg.py:572-663 ---------------------------
    def _check_2d_viscous(self):
        if self.mesh.dim != 2:
            raise NotImplementedError("the oracle's viscous terms follow the reference and are 2D")

    def aux_gradient(self, coeffs, iteration=None):
        """compute_aux_gradient (hodg/dg.py:572-591): qhat_pass then aux_pass."""
        self._check_2d_viscous()
        m, t = self.mesh, self.tab
        b = self.bundle(coeffs.dtype)
        L, sf = _clib.lib(), _clib.sfx(coeffs.dtype)
        nqf, nb = t.n_face_points, t.n_basis
        qhat = np.zeros((m.n_faces, nqf, 4), dtype=coeffs.dtype)
        errf = np.zeros(m.n_faces, dtype=np.uint8)
        nrm = b["normal"]
        getattr(L, "ora_qhat_pass" + sf)(
            m.n_faces, nqf, nb, _clib.ptr(coeffs), _clib.ptr(b["face_basis_l"]), _clib.ptr(b["face_basis_r"]),
            _clib.ptr(m.face_cells), _clib.ptr(self.bc), _clib.ptr(nrm[0]), _clib.ptr(nrm[1]), _clib.ptr(b["qinf"]),
            self.gas.gamma, _clib.ptr(qhat), _clib.ptr(errf))
        if errf.any():
            raise AdmissibilityError("inadmissible face trace", face=int(np.nonzero(errf)[0][0]), iteration=iteration)
        aux = np.empty((m.n_cells, 2, 4, nb), dtype=coeffs.dtype)
        scratch = np.zeros_like(aux)
        minv = b.get("minv_cast")
        if minv is None:
            minv = b["minv_cast"] = np.ascontiguousarray(t.minv, dtype=coeffs.dtype)
        g = b["vol_grad"]
        getattr(L, "ora_aux_pass" + sf)(
            m.n_cells, nb, t.n_vol_points, nqf, m.cell_faces.shape[1], _clib.ptr(coeffs), _clib.ptr(qhat),
            _clib.ptr(b["vol_w"]), _clib.ptr(b["vol_basis"]), _clib.ptr(g[0]), _clib.ptr(g[1]),
            _clib.ptr(m.cell_nfaces), _clib.ptr(m.cell_faces), _clib.ptr(m.cell_fsign), _clib.ptr(b["face_w"]),
            _clib.ptr(b["face_basis_l"]), _clib.ptr(b["face_basis_r"]), _clib.ptr(nrm[0]), _clib.ptr(nrm[1]),
            _clib.ptr(minv), _clib.ptr(scratch), _clib.ptr(aux))
        return aux

    def flux_pass_ns(self, coeffs, aux, iteration=None):
        """flux_pass with ivis = 1 (hodg/dg.py:240-351): (finv, fvis, fqhat)."""
        self._check_2d_viscous()
        m, t, gs = self.mesh, self.tab, self.gas
        b = self.bundle(coeffs.dtype)
        shp = (m.n_faces, t.n_face_points, 4)
        finv, fvis, fqhat = (np.zeros(shp, dtype=coeffs.dtype) for _ in range(3))
        errf = np.zeros(m.n_faces, dtype=np.uint8)
        nrm = b["normal"]
        getattr(_clib.lib(), "ora_flux_pass_ns" + _clib.sfx(coeffs.dtype))(
            m.n_faces, t.n_face_points, t.n_basis, _clib.ptr(coeffs), _clib.ptr(aux), _clib.ptr(b["face_basis_l"]),
            _clib.ptr(b["face_basis_r"]), _clib.ptr(m.face_cells), _clib.ptr(self.bc), _clib.ptr(nrm[0]),
            _clib.ptr(nrm[1]), _clib.ptr(b["qinf"]), gs.gamma, gs.R, gs.mu, gs.Pr, _clib.ptr(finv), _clib.ptr(fvis),
            _clib.ptr(fqhat), _clib.ptr(errf))
        if errf.any():
            raise AdmissibilityError("inadmissible face trace", face=int(np.nonzero(errf)[0][0]), iteration=iteration)
        return finv, fvis, fqhat

    def rhs_pass_ns(self, coeffs, aux, finv, fvis, iteration=None):
        """rhs_pass with ivis = 1 (hodg/dg.py:353-460)."""
        self._check_2d_viscous()
        m, t, gs = self.mesh, self.tab, self.gas
        b = self.bundle(coeffs.dtype)
        res = np.empty((m.n_cells, 4, t.n_basis))
        scratch = np.zeros_like(res)
        errc = np.zeros(m.n_cells, dtype=np.uint8)
        g = b["vol_grad"]
        getattr(_clib.lib(), "ora_rhs_pass_ns" + _clib.sfx(coeffs.dtype))(
            m.n_cells, t.n_basis, t.n_vol_points, t.n_face_points, m.cell_faces.shape[1], _clib.ptr(coeffs),
            _clib.ptr(aux), _clib.ptr(finv), _clib.ptr(fvis), _clib.ptr(b["vol_w"]), _clib.ptr(b["vol_basis"]),
            _clib.ptr(g[0]), _clib.ptr(g[1]), _clib.ptr(m.cell_nfaces), _clib.ptr(m.cell_faces),
            _clib.ptr(m.cell_fsign), _clib.ptr(b["face_w"]), _clib.ptr(b["face_basis_l"]),
            _clib.ptr(b["face_basis_r"]), _clib.ptr(t.minv), gs.gamma, gs.R, gs.mu, gs.Pr, _clib.ptr(scratch),
            _clib.ptr(res), _clib.ptr(errc))
        if errc.any():
            raise AdmissibilityError("inadmissible volume state", cell=int(np.nonzero(errc)[0][0]), iteration=iteration)
        return res

    def rhs(self, coeffs, iteration=None):
        coeffs = np.ascontiguousarray(coeffs)
        if self.gas.ivis:
            aux = self.aux_gradient(coeffs, iteration)
            finv, fvis, _ = self.flux_pass_ns(coeffs, aux, iteration)
            return self.rhs_pass_ns(coeffs, aux, finv, fvis, iteration)
        return self.rhs_pass(coeffs, self.flux_pass(coeffs, iteration), iteration)


def make_disc(mesh, order, gas=Gas(), mach=0.5, angle_deg=0.0, flux_kind=0):
    tab = compute_tables(mesh, order)
    return Disc(mesh, tab, gas, freestream_conserved(gas, mach, angle_deg, mesh.dim), flux_kind)


# ---------------------------------------------------------------------------
# time integration (hodg/timestepping.py)


def local_dt_field(disc, coeffs, cfl, order, iteration=None):
    m = disc.mesh
    out = np.empty(m.n_cells)
    errc = np.zeros(m.n_cells, dtype=np.uint8)
    coeffs = np.ascontiguousarray(coeffs)
    getattr(_clib.lib(), "ora_dt_pass" + _clib.sfx(coeffs.dtype))(
        m.dim, m.n_cells, disc.tab.n_basis, _clib.ptr(coeffs), _clib.ptr(disc.tab.basis_mean), _clib.ptr(m.cell_h),
        disc.gas.gamma, disc.gas.mu, cfl, order, _clib.ptr(out), _clib.ptr(errc))
    if errc.any():
        raise AdmissibilityError("inadmissible cell mean", cell=int(np.nonzero(errc)[0][0]), iteration=iteration)
    return out


def min_reduce(values, block_size=256):
    """hodg/timestepping.py:150-162 (exact, so any order agrees)."""
    a = np.ascontiguousarray(values, dtype=np.float64).ravel()
    if a.size == 0:
        raise ValueError("min_reduce of empty array")
    while a.size > 1:
        a = np.minimum.reduceat(a, np.arange(0, a.size, block_size))
    return float(a[0])


def _dtvec(dt, n):
    return np.full(n, float(dt)) if np.ndim(dt) == 0 else np.ascontiguousarray(dt, dtype=np.float64)


def rk2_step(coeffs, dt, rhs_fn):
    """hodg/timestepping.py:192-205 (Heun)."""
    n = coeffs.shape[0]
    per = coeffs.shape[1] * coeffs.shape[2]
    dtc = _dtvec(dt, n)
    L = _clib.lib()
    s = _clib.sfx(coeffs.dtype)
    r0 = rhs_fn(coeffs)
    u1 = np.empty_like(coeffs)
    getattr(L, "ora_axpy" + s)(n, per, _clib.ptr(coeffs), _clib.ptr(r0), _clib.ptr(dtc), _clib.ptr(u1))
    r1 = rhs_fn(u1)
    out = np.empty_like(coeffs)
    getattr(L, "ora_combine" + s)(n, per, _clib.ptr(coeffs), _clib.ptr(u1), _clib.ptr(r1), _clib.ptr(dtc),
                                  _clib.ptr(out))
    return out


def rk3_step(coeffs, dt, rhs_fn):
    """SSP-RK3 (Shu-Osher): u1 = u + dt L(u); u2 = 3/4 u + 1/4 (u1 + dt L(u1));
    u' = 1/3 u + 2/3 (u2 + dt L(u2)).  Stages are a u + b (us + dt r)."""
    n = coeffs.shape[0]
    per = coeffs.shape[1] * coeffs.shape[2]
    dtc = _dtvec(dt, n)
    L = _clib.lib()
    s = _clib.sfx(coeffs.dtype)
    r0 = rhs_fn(coeffs)
    u1 = np.empty_like(coeffs)
    getattr(L, "ora_axpy" + s)(n, per, _clib.ptr(coeffs), _clib.ptr(r0), _clib.ptr(dtc), _clib.ptr(u1))
    r1 = rhs_fn(u1)
    u2 = np.empty_like(coeffs)
    getattr(L, "ora_rk_combo" + s)(n, per, 0.75, 0.25, _clib.ptr(coeffs), _clib.ptr(u1), _clib.ptr(r1),
                                   _clib.ptr(dtc), _clib.ptr(u2))
    r2 = rhs_fn(u2)
    out = np.empty_like(coeffs)
    getattr(L, "ora_rk_combo" + s)(n, per, 1.0 / 3.0, 2.0 / 3.0, _clib.ptr(coeffs), _clib.ptr(u2), _clib.ptr(r2),
                                   _clib.ptr(dtc), _clib.ptr(out))
    return out


def residual_l2(res, cell_area):
    """hodg/timestepping.py:208-211."""
    r0 = res[:, :, 0]
    return np.sqrt(np.sum(cell_area[:, None] * r0 * r0, axis=0))


# ---------------------------------------------------------------------------
# precision control (hodg/precision.py)


class PrecisionController:
    def __init__(self, mode="dp", switch_iter=0, window=200, factor=2.0):
        self.mode, self.switch_iter, self.window, self.factor = mode, switch_iter, window, factor
        self._switched = False

    def decide(self, it, rho_hist):
        if self.mode == "dp":
            return 64
        if self.mode == "sp":
            return 32
        if self._switched:
            return 64
        if self.mode == "mp_fixed":
            if it < self.switch_iter:
                return 32
            self._switched = True
            return 64
        n = len(rho_hist)
        if n >= 2:
            m = min(rho_hist[max(0, n - 1 - self.window): n - 1])
            if m > 0.0 and float(rho_hist[-1]) >= self.factor * m:
                self._switched = True
                return 64
        return 32

    def starts_reduced(self):
        return self.mode in ("sp", "mp_rebound") or (self.mode == "mp_fixed" and self.switch_iter > 0)


# ---------------------------------------------------------------------------
# driver (hodg/timestepping.py:256-357)


@dataclass
class RunSpec:
    mesh: object
    order: int = 1
    gas: Gas = Gas()
    mach: float = 0.3
    angle_deg: float = 0.0
    initial: str = "freestream"  # freestream | vortex | pulse
    beta: float = 5.0
    amplitude: float = 0.2
    sigma: float = 0.1
    x0: float = 0.0
    y0: float = 0.0
    cfl: float = 0.3
    dt_mode: str = "local"
    max_iterations: int = 100
    log_every: int = 1
    precision_mode: str = "dp"
    switch_iter: int = 0
    window: int = 200
    factor: float = 2.0
    dt_floor: float = 0.0
    dt_fixed: float | None = None
    t_final: float | None = None
    scheme: str = "rk2"  # rk2 | rk3
    flux_kind: int = 0  # 0 Roe (Harten-Hyman), 1 LLF
    state_bits_mp: int = 32  # storage width during reduced-precision steps


@dataclass
class History:
    iterations: list = field(default_factory=list)
    res: list = field(default_factory=list)
    dts: list = field(default_factory=list)
    precision: list = field(default_factory=list)
    t_sim: float = 0.0  # simulated time (global dt mode)
    switch: int | None = None  # iteration of the promotion to 64-bit



def initial_state(spec, disc):
    m, gas = spec.mesh, spec.gas
    if spec.initial == "vortex":
        def fld(*xs):
            return vortex_primitive(gas, spec.mach, spec.angle_deg, spec.beta, spec.x0, spec.y0, 0.0, xs[0], xs[1],
                                    dim=m.dim)
    elif spec.initial == "pulse":
        def fld(*xs):
            return pulse_primitive(gas, spec.amplitude, spec.sigma, spec.x0, spec.y0, xs[0], xs[1], spec.mach,
                                   spec.angle_deg, dim=m.dim)
    else:
        w = freestream_primitive(gas, spec.mach, spec.angle_deg, m.dim)

        def fld(*xs):
            return w
    return project_initial(m, disc.tab, fld, gas)


def run(spec: RunSpec):
    m = spec.mesh
    disc = Disc(m, compute_tables(m, spec.order), spec.gas,
                freestream_conserved(spec.gas, spec.mach, spec.angle_deg, m.dim), spec.flux_kind)
    u = initial_state(spec, disc)
    ctrl = PrecisionController(spec.precision_mode, spec.switch_iter, spec.window, spec.factor)
    hist = History()
    if ctrl.starts_reduced():
        u32 = u.astype(np.float32)
        if not np.all(np.isfinite(u32)):
            raise ValueError("demotion to 32-bit overflowed to non-finite values")
        u = u32
    step = rk3_step if spec.scheme == "rk3" else rk2_step
    for it in range(spec.max_iterations):
        bits = ctrl.decide(it, [r[0] for r in hist.res])
        if bits == 64 and hist.switch is None and ctrl._switched:
            hist.switch = it
        if bits == 64 and u.dtype == np.float32:
            u = u.astype(np.float64)
        dts = local_dt_field(disc, u, spec.cfl, spec.order, it)
        # hodg/timestepping.py:328-341: dt floor, fixed dt, t_final clip
        if spec.dt_floor > 0.0:
            np.maximum(dts, spec.dt_floor, out=dts)
        if spec.dt_mode == "global":
            dt = spec.dt_fixed if spec.dt_fixed is not None else min_reduce(dts)
            if spec.t_final is not None:
                if hist.t_sim >= spec.t_final - 1e-14:
                    break
                dt = min(dt, spec.t_final - hist.t_sim)
            dtv = np.full(m.n_cells, dt)
            dt_log = dt
        else:
            dtv = dts
            dt_log = min_reduce(dts)
        first = []

        def rfn(c, _it=it):
            r = disc.rhs(c, _it)
            if not first:
                first.append(r)
            return r

        u = step(u, dtv, rfn)
        if spec.dt_mode == "global":
            hist.t_sim += dt_log
        if spec.log_every and (it % spec.log_every == 0 or it == spec.max_iterations - 1):
            res4 = residual_l2(first[0], m.cell_area)
            if not np.all(np.isfinite(res4)):
                raise SolverDivergedError(it, hist)
            hist.iterations.append(it)
            hist.res.append(tuple(float(r) for r in res4))
            hist.dts.append(float(dt_log))
            hist.precision.append(bits)
    return u, hist, disc


def residual_csv_text(hist, nvar=4):
    """hodg/output.py:17-28 (4 variables); 3D adds res_rhow."""
    head = "iter,res_rho,res_rhou,res_rhov,res_e,dt,precision" if nvar == 4 else \
        "iter,res_rho,res_rhou,res_rhov,res_rhow,res_e,dt,precision"
    lines = [head]
    for it, res, dt, bits in zip(hist.iterations, hist.res, hist.dts, hist.precision):
        lines.append(",".join([str(it)] + [repr(r) for r in res] + [repr(dt), str(bits)]))
    return "\n".join(lines) + "\n"


# ---------------------------------------------------------------------------
# point evaluations (hodg/physics.py:436-479)


def point_flux(qL, qR, normals, gamma=1.4, flux_kind=0, dtype=np.float64):
    qL = np.ascontiguousarray(qL, dtype=dtype)
    qR = np.ascontiguousarray(qR, dtype=dtype)
    nr = np.ascontiguousarray(normals, dtype=dtype)
    n, nv = qL.shape
    out = np.zeros_like(qL)
    ok = np.zeros(n, dtype=np.uint8)
    getattr(_clib.lib(), "ora_point_flux" + _clib.sfx(dtype))(nr.shape[1], n, _clib.ptr(qL), _clib.ptr(qR),
                                                               _clib.ptr(nr), gamma, flux_kind, _clib.ptr(out),
                                                               _clib.ptr(ok))
    return out, ok.astype(bool)


def point_bstate(kind, q, normals, qf, gamma=1.4, dtype=np.float64):
    q = np.ascontiguousarray(q, dtype=dtype)
    nr = np.ascontiguousarray(normals, dtype=dtype)
    qf = np.ascontiguousarray(qf, dtype=dtype)
    out = np.zeros_like(q)
    getattr(_clib.lib(), "ora_point_bstate" + _clib.sfx(dtype))(nr.shape[1], q.shape[0], kind, _clib.ptr(q),
                                                                 _clib.ptr(nr), _clib.ptr(qf), gamma, _clib.ptr(out))
    return out
