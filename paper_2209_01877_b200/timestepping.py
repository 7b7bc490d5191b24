"""Time integration on the B200 (hodg/timestepping.py:1-402).

Two surfaces:

* the reference's functional API -- `local_dt_field`, `min_reduce`,
  `rk2_step(state, dt, rhs_fn)`, `rk3_step`, `residual_l2` -- for drop-in
  use with an arbitrary `rhs_fn` (stage combinations are torch elementwise
  ops on the device there);

* `Stepper`, the fused hot path: per RK stage one face kernel and one
  element kernel that also applies the stage combination, the CFL dt of
  the new state (global min by atomics, no host sync) and the residual-norm
  partials; the state stays in device memory in the reference-element basis
  and one step is captured in a CUDA graph.  `run()` drives it with the
  reference's loop semantics (precision control, logging, divergence and
  admissibility checks).
"""

from __future__ import annotations

import ctypes as C
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .dg import BoundaryConditions, Discretization, DofState, N_VARS, Residual, _get_disc, project_initial
from .geometry import compute_geometry
from .mesh import TetMesh
from .physics import AdmissibilityError, GasModel
from .precision import PrecisionController, PrecisionSchedule

__all__ = [
    "SolverDivergedError",
    "ResidualHistory",
    "local_dt_field",
    "min_reduce",
    "rk2_step",
    "rk3_step",
    "residual_l2",
    "Stepper",
    "RunConfig",
    "RunArtifacts",
    "run",
]

INF_BITS = 0x7FF0000000000000


def _torch():
    import torch

    return torch


class SolverDivergedError(RuntimeError):
    def __init__(self, iteration, history):
        super().__init__(f"non-finite residual at iteration {iteration}")
        self.iteration = iteration
        self.history = history


@dataclass
class ResidualHistory:
    iterations: list = field(default_factory=list)
    res: list = field(default_factory=list)
    dts: list = field(default_factory=list)
    precision: list = field(default_factory=list)

    def append(self, iteration, res5, dt, bits):
        self.iterations.append(int(iteration))
        self.res.append(tuple(float(r) for r in res5))
        self.dts.append(float(dt))
        self.precision.append(int(bits))

    @property
    def res_rho(self):
        return [r[0] for r in self.res]


# ---------------------------------------------------------------------------
# functional API


def local_dt_field(state: DofState, mesh: TetMesh, geo, gas: GasModel, cfl: float, order: int,
                   bcs: BoundaryConditions | None = None):
    """Per-element CFL dt from the cell means, float64 device tensor
    (hodg/timestepping.py:137-147)."""
    from .physics import Conserved

    bcs = bcs or BoundaryConditions(Conserved(1.0, 0.0, 0.0, 0.0, 1.0))
    disc = _get_disc(mesh, geo, gas, bcs)
    if order != geo.order:
        raise ValueError("order does not match the geometry")
    rows = disc.to_reference(state.coeffs)
    out = _torch().empty(disc.n, dtype=_torch().float64, device=disc.device)
    disc.reset_errors()
    _lib.check(disc.L.hodg_local_dt(disc.handle, _lib.ptr(rows), float(cfl), _lib.ptr(out), None,
                                    _lib.ptr(disc.err), _lib.stream_ptr()), "hodg_local_dt")
    disc.raise_errors(state.iteration)
    return out


def min_reduce(values, block_size: int = 256) -> float:
    """Exact global minimum (hodg/timestepping.py:150-162); min is exact, so
    the device reduction equals the reference's block tree bitwise."""
    torch = _torch()
    if block_size < 2:
        raise ValueError("block size must be at least 2")
    x = torch.as_tensor(values, dtype=torch.float64)
    if x.numel() == 0:
        raise ValueError("min_reduce of empty array")
    if not x.is_cuda:
        x = x.to("cuda")
    x = x.contiguous().reshape(-1)
    L = _lib.lib()
    scratch = torch.empty(1024, dtype=torch.float64, device=x.device)
    out = torch.empty(1, dtype=torch.float64, device=x.device)
    _lib.check(L.hodg_min_reduce_f64(_lib.ptr(x), x.numel(), _lib.ptr(scratch), _lib.ptr(out), _lib.stream_ptr()),
               "hodg_min_reduce_f64")
    return float(out.item())


def _dt_tensor(dt, n, device):
    torch = _torch()
    t = torch.as_tensor(dt, dtype=torch.float64, device=device)
    if t.ndim == 0:
        return t.expand(n)
    if tuple(t.shape) != (n,):
        raise ValueError("per-cell dt has wrong length")
    return t


def rk2_step(state: DofState, dt, rhs_fn) -> DofState:
    """Heun: u1 = u + dt R(u); u' = (u + u1 + dt R(u1)) / 2, computed in
    float64 and stored at the state precision (hodg/timestepping.py:192-205).
    rhs_fn is called exactly twice."""
    u = state.coeffs
    d = _dt_tensor(dt, u.shape[0], u.device)[:, None, None]
    r0 = rhs_fn(state)
    u1 = (u.double() + d * r0.res).to(u.dtype)
    r1 = rhs_fn(DofState(u1, state.iteration))
    out = (0.5 * ((u + u1).double() + d * r1.res)).to(u.dtype)
    return DofState(out, state.iteration + 1)


def rk3_step(state: DofState, dt, rhs_fn) -> DofState:
    """SSP-RK3 (Shu-Osher): u1 = u + dt L(u); u2 = 3/4 u + 1/4 (u1 + dt L(u1));
    u' = 1/3 u + 2/3 (u2 + dt L(u2)).  rhs_fn is called exactly three times."""
    u = state.coeffs
    d = _dt_tensor(dt, u.shape[0], u.device)[:, None, None]
    ud = u.double()
    r0 = rhs_fn(state)
    u1 = (ud + d * r0.res).to(u.dtype)
    r1 = rhs_fn(DofState(u1, state.iteration))
    u2 = (0.75 * ud + 0.25 * (u1.double() + d * r1.res)).to(u.dtype)
    r2 = rhs_fn(DofState(u2, state.iteration))
    out = ((1.0 / 3.0) * ud + (2.0 / 3.0) * (u2.double() + d * r2.res)).to(u.dtype)
    return DofState(out, state.iteration + 1)


def residual_l2(residual: Residual, mesh: TetMesh):
    """Per-variable sqrt(sum vol * res[:, v, 0]^2) (hodg/timestepping.py:208-211)."""
    torch = _torch()
    vol = torch.as_tensor(mesh.cell_area, device=residual.res.device)
    r0 = residual.res[:, :, 0]
    return torch.sqrt(torch.sum(vol[:, None] * r0 * r0, dim=0)).cpu().numpy()


# ---------------------------------------------------------------------------
# fused device stepper

SCHEMES = {
    # per stage: (combine, a, b, u0 needed)
    "rk2": [(0, 0.0, 1.0), (1, 0.5, 0.5)],
    "rk3": [(0, 0.0, 1.0), (0, 0.75, 0.25), (0, 1.0 / 3.0, 2.0 / 3.0)],
}


class Stepper:
    """Device-resident RK stepping with fused stage kernels.

    Buffers (n x rs float64, reference basis): A holds u^n and receives
    u^{n+1}; B holds the intermediate stages (written in place).  Global dt
    lives in two device slots (double bits) alternating per step: stage 1
    resets the slot the last stage will atomically min into.
    """

    def __init__(self, disc: Discretization, scheme="rk3", prec=_lib.PREC_F64, dt_mode="global", cfl=0.3,
                 log_norms=True, use_graph=True, layout="auto", shadow=None):
        torch = _torch()
        if layout not in ("auto", "elem", "face"):
            raise ValueError(f"unknown record layout {layout!r}")
        self.layout = layout
        if scheme not in SCHEMES:
            raise ValueError(f"unknown scheme {scheme!r}")
        if dt_mode not in ("local", "global"):
            raise ValueError(f"unknown dt mode {dt_mode!r}")
        self.disc, self.scheme, self.prec, self.dt_mode, self.cfl = disc, scheme, prec, dt_mode, float(cfl)
        self.log_norms = log_norms
        self.use_graph = use_graph
        dev = disc.device
        self.A = disc.new_state()
        self.B = disc.new_state()
        self.hbuf = self._records(prec)
        self.slots = torch.full((2,), INF_BITS, dtype=torch.int64, device=dev)
        self.dtv = [torch.zeros(disc.n, dtype=torch.float64, device=dev) for _ in range(2)]
        self.partial = torch.zeros((disc.nblk, 5), dtype=torch.float64, device=dev)
        self.norms = torch.zeros(5, dtype=torch.float64, device=dev)
        self.parity = 0
        self.steps = 0
        self._graphs = {}
        self._args = []
        # boundary faces concurrent with the interior tail (HODG_OVERLAP_BND=0: serial)
        self._side = torch.cuda.Stream(device=dev) if os.environ.get("HODG_OVERLAP_BND", "1") != "0" else None
        self.capture_mode = "global"
        # mixed precision: the element kernel also writes an FP32 shadow of
        # each stage's state, which the face kernel reads (no per-row FP64 ->
        # FP32 conversion, half the row bytes); off with shadow=False or
        # HODG_SHADOW=0, and for partitioned runs (FP64 ghost rows)
        if shadow is None:
            shadow = os.environ.get("HODG_SHADOW", "1") != "0"
        self.shadow = bool(shadow)
        self.A32 = self.B32 = None

    # -- state in / out ----------------------------------------------------
    def load(self, state: DofState):
        self.disc.to_reference(state.coeffs, out=self.A)
        self.steps = 0
        self.parity = 0
        self.init_dt()
        self._sync_shadow()

    def _uses_shadow(self) -> bool:
        return self.shadow and self.prec == _lib.PREC_MIXED

    def _sync_shadow(self):
        """(Re)build the FP32 shadow of A when the mixed kernels run."""
        if not self._uses_shadow():
            return
        if self.A32 is None:
            self.A32 = self.disc.new_state32()
            self.B32 = self.disc.new_state32()
        self.disc.shadow_of(self.A, self.A32)

    def state(self, iteration=0) -> DofState:
        return DofState(self.disc.from_reference(self.A), iteration)

    def init_dt(self):
        """CFL dt of the loaded state into the current slot / vector."""
        d = self.disc
        d.reset_errors()
        self.slots.fill_(INF_BITS)
        _lib.check(d.L.hodg_local_dt(d.handle, _lib.ptr(self.A), self.cfl, _lib.ptr(self.dtv[self.parity]),
                                     _lib.ptr(self.slots[self.parity:]), _lib.ptr(d.err), _lib.stream_ptr()),
                   "hodg_local_dt")

    def set_dt(self, dt: float):
        """Overwrite the global dt the next step uses (host-chosen dt:
        dt_fixed, dt_floor, the t_final clip; hodg/timestepping.py:328-337)."""
        bits = int(np.array([float(dt)], dtype=np.float64).view(np.int64)[0])
        self.slots[self.parity].fill_(bits)

    def floor_dt(self, dt_floor: float):
        """Per-element dt floor of the next step (local dt mode,
        hodg/timestepping.py:328-329), applied on the device."""
        self.dtv[self.parity].clamp_(min=float(dt_floor))

    def cell_means(self):
        """(n, 5) float64 cell means of the current state (device)."""
        from .refelem import ref_tables

        t = ref_tables(self.disc.order)
        mean = _torch().from_numpy(t.MEAN).to(self.disc.device)
        return self.A[: self.disc.n, : N_VARS * t.nb].reshape(self.disc.n, N_VARS, t.nb) @ mean

    def dt_value(self) -> float:
        """The global dt used by the next step (host read, syncs)."""
        if self.dt_mode == "global":
            bits = int(self.slots[self.parity].item())
            return float(np.array([bits], dtype=np.int64).view(np.float64)[0])
        return min_reduce(self.dtv[self.parity])

    # -- one step ----------------------------------------------------------
    def _records(self, prec):
        """Face flux record buffer: the element-slot layout (one bulk copy per
        element tile, but two record stores per face) or the face-ordered one.
        "auto" takes the faster on the B200: element-slot at P3
        and for mixed precision at P0, face-ordered otherwise (round 2, C1M:
        mixed P1 4.65e10 face vs 4.28e10 element-slot, P2 7.51e10 vs 7.40e10,
        P0 2.34e10 vs 2.53e10)."""
        use_elem = self.layout == "elem" or (
            self.layout == "auto" and (self.disc.order >= 3 or (prec == _lib.PREC_MIXED and self.disc.order == 0)))
        return self.disc.elem_buffer(prec) if use_elem else self.disc.face_buffer(prec)

    def _stage_args(self, k, parity):
        d = self.disc
        combine, a, b = SCHEMES[self.scheme][k]
        last = k == len(SCHEMES[self.scheme]) - 1
        s = _lib.StageArgs()
        s.us = _lib.ptr(self.A if k == 0 else self.B)
        s.u0 = _lib.ptr(self.A)
        s.out = _lib.ptr(self.A if last else self.B)
        s.res = None
        s.a, s.b = a, b
        s.combine = combine
        if self.dt_mode == "global":
            s.dt_is_vector = 0
            s.dt = C.c_void_p(self.slots.data_ptr() + 8 * parity)
        else:
            s.dt_is_vector = 1
            s.dt = _lib.ptr(self.dtv[parity])
        s.norm_partial = _lib.ptr(self.partial) if (k == 0 and self.log_norms) else None
        if last:
            if self.dt_mode == "global":
                s.dt_next = C.c_void_p(self.slots.data_ptr() + 8 * (1 - parity))
            else:
                s.dt_vec_out = _lib.ptr(self.dtv[1 - parity])
        if k == 0 and self.dt_mode == "global":
            s.dt_reset = C.c_void_p(self.slots.data_ptr() + 8 * (1 - parity))
        s.cfl = self.cfl
        if self._uses_shadow():
            s.out32 = _lib.ptr(self.A32 if last else self.B32)
        return s

    def _launch_step(self, parity):
        d = self.disc
        n_st = len(SCHEMES[self.scheme])
        for k in range(n_st):
            us = self.A if k == 0 else self.B
            us32 = (self.A32 if k == 0 else self.B32) if self._uses_shadow() else None
            d.face_flux_split(us, self.prec, self.hbuf, self._side, rows32=us32)
            args = self._stage_args(k, parity)
            self._args.append(args)
            d.stage(self.prec, self.hbuf, args)
            if k == 0 and self.log_norms:
                _lib.check(d.L.hodg_norm_finalize(_lib.ptr(self.partial), d.nblk, _lib.ptr(self.norms),
                                                  _lib.stream_ptr()), "hodg_norm_finalize")

    def warm(self):
        """Run the stage kernels once outside graph capture (first-launch
        attribute setup) without touching the state: residual into B."""
        d = self.disc
        if self._uses_shadow():
            d.face_flux32(self.A32, self.hbuf)
        else:
            d.face_flux(self.A, self.prec, self.hbuf)
        d.residual_rows(self.A, self.hbuf, self.prec, res=self.B)

    def launches_per_step(self) -> int:
        """Kernels one step launches: per stage the face-kernel ranges and the
        element kernel, plus the norm finalize."""
        per_stage = len(self.disc.face_segments()) + 1
        return per_stage * len(SCHEMES[self.scheme]) + (1 if self.log_norms else 0)

    def step(self):
        """Advance one step (asynchronous; no host sync)."""
        torch = _torch()
        p = self.parity
        if self.use_graph:
            g = self._graphs.get(p)
            if g is None:
                self.warm()
                s = torch.cuda.Stream()
                s.wait_stream(torch.cuda.current_stream())
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s, capture_error_mode=self.capture_mode):
                    self._launch_step(p)
                torch.cuda.current_stream().wait_stream(s)
                self._graphs[p] = g
            g.replay()
        else:
            self._launch_step(p)
            self._args.clear()
        self.parity = 1 - p
        self.steps += 1

    def check(self, iteration=None):
        self.disc.raise_errors(iteration)


# ---------------------------------------------------------------------------
# driver


@dataclass
class RunConfig:
    """Subset of the reference's RunConfig (hodg/config.py:28-75) for the
    tetrahedral box generator, plus scheme / flux / renumbering knobs."""

    n: int = 8
    ny: int | None = None
    nz: int | None = None
    extent: tuple = (0.0, 0.0, 0.0, 1.0, 1.0, 1.0)
    bc: object = "far_field"
    perturb: float = 0.0
    perturb_seed: int = 3
    gamma: float = 1.4
    R: float = 1.0
    mach: float = 0.3
    angle_deg: float = 0.0
    initial_kind: str = "freestream"  # freestream | vortex
    vortex_beta: float = 5.0
    initial_x0: float = 0.0
    initial_y0: float = 0.0
    order: int = 1
    cfl: float = 0.3
    dt_mode: str = "local"
    scheme: str = "rk2"
    flux: str = "roe"
    dt_floor: float = 0.0
    dt_fixed: float | None = None
    t_final: float | None = None
    max_iterations: int = 100
    log_every: int = 1
    residual_target: float | None = None
    output_prefix: str | None = None
    output_every: int = 0
    renumber: bool = False
    randomize_cells: int | None = None
    precision_mode: str = "dp"
    switch_iter: int = 0
    window: int = 200
    factor: float = 2.0
    check_every: int = 1

    def __post_init__(self):
        if self.dt_mode not in ("local", "global"):
            raise ValueError(f"unknown dt mode {self.dt_mode!r}")
        if self.dt_floor < 0.0:
            raise ValueError("dt_floor must be non-negative")
        if self.dt_fixed is not None and not self.dt_fixed > 0.0:
            raise ValueError("dt_fixed must be positive")
        if self.max_iterations < 0:
            raise ValueError("max_iterations must be non-negative")
        if self.output_every < 0:
            raise ValueError("output_every must be non-negative")

    def make_mesh(self) -> TetMesh:
        from .mesh import generate_tet_box, perturb_interior_nodes

        m = generate_tet_box(self.n, self.ny, self.nz, self.extent, self.bc)
        if self.perturb > 0.0:
            m = perturb_interior_nodes(m, self.perturb, self.perturb_seed)
        return m

    def gas_model(self) -> GasModel:
        return GasModel(gamma=self.gamma, R=self.R)

    def precision_schedule(self) -> PrecisionSchedule:
        return PrecisionSchedule(self.precision_mode, self.switch_iter, self.window, self.factor)


@dataclass
class RunArtifacts:
    final_state: DofState
    history: ResidualHistory
    events: list
    mesh: TetMesh
    geo: object
    config: RunConfig
    iterations_run: int
    setup_seconds: float
    iterate_seconds: float
    bandwidth_before: int | None = None
    bandwidth_after: int | None = None
    t_sim: float = 0.0
    output_files: list = field(default_factory=list)


def initial_field(cfg: RunConfig, gas: GasModel):
    from .physics import freestream_primitive, vortex_primitive

    if cfg.initial_kind == "vortex":
        return lambda x, y, z: vortex_primitive(gas, cfg.mach, cfg.angle_deg, cfg.vortex_beta, cfg.initial_x0,
                                                cfg.initial_y0, 0.0, x, y)
    w = freestream_primitive(gas, cfg.mach, cfg.angle_deg)
    return lambda x, y, z: w


def run(config: RunConfig, mesh: TetMesh | None = None) -> RunArtifacts:
    """Drive a solve (hodg/timestepping.py:256-402): optional shuffle /
    RCM renumbering, geometry, projection, then the precision-controlled
    loop on the fused stepper, with the reference's order of operations per
    step -- decide / promote, dt (CFL, `dt_floor`, `dt_fixed`, the `t_final`
    clip with 1e-14 slack), the RK step, logging, field output every
    `output_every` steps.  The logged residual is the first stage's, as in
    the reference; errors are checked every `check_every` steps.

    The CFL dt comes from the previous step's fused epilogue (device atomic
    min); a host-chosen dt (dt_fixed, dt_floor, t_final) is written into the
    stepper's dt slot before the step, which costs one small host sync per
    step -- the plain CFL path stays sync-free except for logging."""
    from .output import write_residual_csv, write_vtk
    from .physics import freestream_conserved
    from .renumber import apply_permutation, bandwidth, build_adjacency, random_permutation, rcm

    t0 = time.perf_counter()
    mesh = config.make_mesh() if mesh is None else mesh
    gas = config.gas_model()
    bcs = BoundaryConditions(freestream_conserved(gas, config.mach, config.angle_deg), config.flux)
    bw0 = bw1 = None
    if config.randomize_cells is not None:
        mesh = apply_permutation(mesh, random_permutation(mesh.n_cells, config.randomize_cells))
    if config.renumber:
        g = build_adjacency(mesh)
        perm = rcm(g)
        bw0, bw1 = bandwidth(g), bandwidth(g, perm)
        mesh = apply_permutation(mesh, perm, device="cuda")
    geo = compute_geometry(mesh, config.order)
    state = project_initial(mesh, geo, initial_field(config, gas), gas)
    disc = _get_disc(mesh, geo, gas, bcs)
    sched = config.precision_schedule()
    ctrl = PrecisionController(sched)
    prec = _lib.PREC_MIXED if sched.starts_reduced else _lib.PREC_F64
    stepper = Stepper(disc, config.scheme, prec, config.dt_mode, config.cfl, log_norms=bool(config.log_every))
    stepper.load(state)
    stepper.check(0)
    hist = ResidualHistory()
    events = []
    out_files = []
    written = set()

    def write_field(iteration):
        if config.output_prefix is None or iteration in written:
            return
        path = f"{config.output_prefix}_{iteration:06d}.vtk"
        write_vtk(path, mesh, stepper.cell_means().cpu().numpy(), gas.gamma)
        out_files.append(path)
        written.add(iteration)

    host_dt = config.dt_mode == "global" and (
        config.dt_fixed is not None or config.t_final is not None or config.dt_floor > 0.0)
    setup = time.perf_counter() - t0
    t1 = time.perf_counter()
    it_run = 0
    t_sim = 0.0
    if config.max_iterations == 0:
        write_field(0)
    for it in range(config.max_iterations):
        bits, ev = ctrl.decide(it, hist.res_rho)
        if ev is not None:
            events.append(ev)
        want = _lib.PREC_MIXED if bits == 32 else _lib.PREC_F64
        if want != stepper.prec:
            stepper.prec = want
            stepper.hbuf = stepper._records(want)
            stepper._graphs.clear()
            stepper._sync_shadow()
        log = config.log_every and (it % config.log_every == 0 or it == config.max_iterations - 1)
        if config.dt_mode == "global":
            if host_dt:
                dt = config.dt_fixed if config.dt_fixed is not None else max(stepper.dt_value(), config.dt_floor)
                if config.t_final is not None:
                    if t_sim >= config.t_final - 1e-14:
                        break
                    dt = min(dt, config.t_final - t_sim)
                stepper.set_dt(dt)
                dt_log = dt
            else:
                dt_log = stepper.dt_value() if log else None
        else:
            if config.dt_floor > 0.0:
                stepper.floor_dt(config.dt_floor)
            dt_log = stepper.dt_value() if log else None
        stepper.step()
        it_run = it + 1
        if config.dt_mode == "global" and host_dt:
            t_sim += dt_log
        if config.check_every and (it + 1) % config.check_every == 0:
            stepper.check(it)
        if log:
            res5 = stepper.norms.cpu().numpy()
            if not np.all(np.isfinite(res5)):
                raise SolverDivergedError(it, hist)
            hist.append(it, res5, dt_log, bits)
            if config.residual_target is not None and np.all(res5 < config.residual_target):
                break
        if config.output_every and (it + 1) % config.output_every == 0:
            write_field(it + 1)
    stepper.check(it_run)
    _torch().cuda.synchronize()
    iterate = time.perf_counter() - t1
    if config.max_iterations > 0:
        write_field(it_run)
    if config.output_prefix is not None:
        csv_path = f"{config.output_prefix}_residuals.csv"
        write_residual_csv(csv_path, hist)
        out_files.append(csv_path)
    final = stepper.state(it_run)
    return RunArtifacts(final, hist, events, mesh, geo, config, it_run, setup, iterate, bw0, bw1, t_sim, out_files)
