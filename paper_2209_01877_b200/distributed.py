"""Partitioned multi-GPU stepping: one process per GPU (torch.distributed,
NCCL over NVLink / NVSwitch), element partition by RCB, ghost-row halo
exchange per RK stage overlapped with the interior-face kernel.

Per stage on each rank:
  1. post the halo exchange of the stage state (NCCL send/recv of the owned
     rows the peers hold as ghosts; receives land directly in the ghost
     block of the state array);
  2. face kernel over the interior faces (no ghost dependency) -- runs while
     the exchange is in flight;
  3. wait for the exchange, face kernel over the partition faces;
  4. element kernel over the owned elements (volume + gather + RK + dt).
After the last stage the per-rank CFL dt minimum is all-reduced (MIN, exact)
for the next step; logged residual norms are all-reduced (SUM).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .dg import BoundaryConditions, Discretization, DofState
from .geometry import compute_geometry
from .mesh import TetMesh
from .partition import HaloExchange, HostHaloExchange, LocalPart, NativeHaloExchange, build_local, rcb_partition
from .physics import GasModel
from .timestepping import SCHEMES, Stepper

__all__ = ["DistributedStepper", "setup_partitioned"]


class DistributedStepper(Stepper):
    """halo: "native" -- the library's NCCL exchange (`hodg_halo_*`, its own
    communicator, unique id broadcast over `group`); "torch" -- point-to-point
    ops of the torch.distributed group (the gloo CPU tests); "host" -- rows
    staged through host memory over a gloo group (ranks sharing one GPU:
    tests/test_gpu_multirank.py); "auto" -- native on CUDA devices (override
    with HODG_HALO=torch|host)."""

    def __init__(self, part: LocalPart, disc: Discretization, scheme="rk3", prec=_lib.PREC_F64, cfl=0.3,
                 log_norms=True, group=None, halo="auto", use_graph=None):
        import os

        import torch
        import torch.distributed as dist

        if halo == "auto":
            halo = os.environ.get("HODG_HALO", "native" if torch.device(disc.device).type == "cuda" else "torch")
        # launches: eager by default -- the exchange and the reductions are
        # stream-ordered (no host sync per step), so the host runs ahead of the
        # GPU.  use_graph=True (or HODG_DIST_GRAPH=1) captures the whole step,
        # NCCL exchange and all-reduces included, in one CUDA graph per dt
        # parity (tools/scaling_estimate.py --capture measures both); the host
        # halo never captures (it synchronises with the host).
        if use_graph is None:
            use_graph = os.environ.get("HODG_DIST_GRAPH", "0") == "1"
        if halo == "host":
            use_graph = False
        super().__init__(disc, scheme, prec, "global", cfl, log_norms=log_norms, use_graph=use_graph,
                         shadow=False)
        # NCCL's proxy thread issues CUDA calls while the step is being
        # captured: "global" capture mode would invalidate the capture
        self.capture_mode = "relaxed"
        self.part = part
        self.group = group
        self.native = halo == "native"
        self.own_reduce = halo in ("native", "host")  # the exchange object's allreduce
        if halo == "native":
            rank, world = dist.get_rank(group), dist.get_world_size(group)
            uid = [NativeHaloExchange.unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0, group=group)
            self.halo = NativeHaloExchange(part, disc.rs, rank, world, uid[0], disc.device)
        elif halo == "torch":
            self.halo = HaloExchange(part, disc.device, group)
        elif halo == "host":
            self.halo = HostHaloExchange(part, disc.device, group)
        else:
            raise ValueError(f"unknown halo exchange {halo!r}")
        self.norm_sums = None

    def _allreduce_dt(self, slot_index):
        import torch.distributed as dist

        s = self.slots[slot_index:slot_index + 1]
        # positive doubles order like their int64 bit patterns: MIN is exact
        if self.own_reduce:
            self.halo.allreduce(s, 0)
        else:
            dist.all_reduce(s, op=dist.ReduceOp.MIN, group=self.group)

    def init_dt(self):
        super().init_dt()
        self._allreduce_dt(self.parity)

    def warm(self):
        """First launches outside graph capture on a halo-complete state."""
        self.halo.start(self.A)
        self.halo.wait()
        super().warm()

    def _launch_step(self, parity):
        import torch

        d = self.disc
        n_st = len(SCHEMES[self.scheme])
        # faces are [interior | boundary | partition]: the interior ones
        # overlap the exchange; boundary + partition faces are one launch
        ni = d.geo.n_int0
        for k in range(n_st):
            us = self.A if k == 0 else self.B
            self.halo.start(us)
            d.face_flux(us, self.prec, self.hbuf, f_begin=0, f_end=ni)
            self.halo.wait()
            d.face_flux(us, self.prec, self.hbuf, f_begin=ni, f_end=d.nf)
            args = self._stage_args(k, parity)
            self._args.append(args)
            d.stage(self.prec, self.hbuf, args)
            if k == 0 and self.log_norms:
                self.norm_sums = self.partial.sum(dim=0)
        self._allreduce_dt(1 - parity)
        if self.log_norms:
            import torch.distributed as dist

            if self.own_reduce:
                self.halo.allreduce(self.norm_sums, 1)
            else:
                dist.all_reduce(self.norm_sums, op=dist.ReduceOp.SUM, group=self.group)
            self.norms.copy_(torch.sqrt(self.norm_sums))

    def launches_per_step(self) -> int:
        d = self.disc
        ni = d.geo.n_int0
        per_stage = len(d.face_segments(0, ni)) + len(d.face_segments(ni, d.nf)) + 1
        return per_stage * len(SCHEMES[self.scheme])  # (the norm sums are torch reductions here)

    def close(self):
        """Release the exchange (the native one owns an NCCL communicator);
        call before destroying the process group."""
        import torch

        # captured steps hold NCCL work: drop the graphs before the
        # communicator (destroying it under a live graph exec blocks)
        self._graphs.clear()
        self._args.clear()
        torch.cuda.synchronize()
        close = getattr(self.halo, "close", None)
        if close is not None:
            close()

    def gather_state(self):
        """Global (n_cells, 5, nb) Taylor coefficients on every rank."""
        import torch
        import torch.distributed as dist

        mine = self.disc.from_reference(self.A).contiguous()
        sizes = [None] * self.part.nparts
        dist.all_gather_object(sizes, (self.part.owned.tolist(), mine.shape[0]), group=self.group)
        maxn = max(s[1] for s in sizes)
        pad = torch.zeros((maxn,) + tuple(mine.shape[1:]), dtype=mine.dtype, device=mine.device)
        pad[: mine.shape[0]] = mine
        bufs = [torch.empty_like(pad) for _ in range(self.part.nparts)]
        dist.all_gather(bufs, pad, group=self.group)
        n = sum(s[1] for s in sizes)
        out = torch.empty((n,) + tuple(mine.shape[1:]), dtype=mine.dtype, device=mine.device)
        for (ids, cnt), b in zip(sizes, bufs):
            out[torch.as_tensor(ids, device=mine.device)] = b[:cnt]
        return out


def setup_partitioned(mesh: TetMesh, order: int, gas: GasModel, bcs: BoundaryConditions, rank: int, world: int,
                      device="cuda"):
    """RCB partition of `mesh` over `world` ranks -> (LocalPart, Discretization)."""
    parts = rcb_partition(mesh.cell_centroid, world)
    part = build_local(mesh, parts, rank)
    geo = compute_geometry(part.mesh, order, split=part.n_inner_faces)
    disc = Discretization(part.mesh, geo, gas, bcs, device=device, n_elems=part.n_owned)
    return part, disc


def owned_state(state: DofState, part: LocalPart) -> DofState:
    import torch

    idx = torch.as_tensor(part.owned, device=state.coeffs.device)
    return DofState(state.coeffs.index_select(0, idx).contiguous(), state.iteration)
