"""Partitioning and the multi-rank halo path on CPU (gloo, world size 2 and
3): the RCB map is bit-exact with the oracle restatement, the halo plan is
consistent, and a partitioned SSP-RK3 run (oracle kernels as the compute,
the product's LocalPart / HaloExchange as the plumbing) equals the serial
run bitwise."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from gpu_helpers import to_oracle
from oracle import partition as OP
from oracle import solver as S
from paper_2209_01877_b200 import mesh as M
from paper_2209_01877_b200.partition import HaloExchange, build_local, rcb_partition


def box():
    return M.perturb_interior_nodes(M.generate_tet_box(4, 3, 2, extent=(0.0, 0.0, 0.0, 4.0, 3.0, 1.0),
                                                       bc={"xmin": "far_field", "xmax": "far_field",
                                                           "ymin": "far_field", "ymax": "far_field",
                                                           "zmin": "slip_wall", "zmax": "slip_wall"}), 0.1, 3)


@pytest.mark.parametrize("nparts", [1, 2, 3, 4, 8])
def test_rcb_bitwise_vs_oracle(nparts):
    m = box()
    p = rcb_partition(m.cell_centroid, nparts)
    q = OP.rcb(m.cell_centroid.tolist(), nparts)
    assert np.array_equal(p, np.array(q))
    counts = np.bincount(p, minlength=nparts)
    assert counts.max() - counts.min() <= 1 + m.n_cells // (4 * nparts)


def test_cube_splits_into_octants():
    m = M.generate_tet_box(4)
    p = rcb_partition(m.cell_centroid, 8)
    for k in range(8):
        c = m.cell_centroid[p == k]
        assert np.all(c.max(axis=0) - c.min(axis=0) <= 0.5)


@pytest.mark.parametrize("nparts", [2, 3, 5])
def test_halo_plan_consistent(nparts):
    m = box()
    parts = rcb_partition(m.cell_centroid, nparts)
    locs = [build_local(m, parts, r) for r in range(nparts)]
    for r, L in enumerate(locs):
        assert np.array_equal(L.owned, np.flatnonzero(parts == r))
        assert M.validate(L.mesh)[:0] == []
        # every face of every owned element is local, with global orientation
        for e in range(L.n_owned):
            for s in range(4):
                lf = L.mesh.cell_faces[e, s]
                gf = m.cell_faces[L.owned[e], s]
                assert L.face_gid[lf] == gf
        gl = np.concatenate([L.owned, L.ghosts])
        fc = L.mesh.face_cells
        assert np.array_equal(gl[fc[:, 0]], m.face_cells[L.face_gid, 0])
        ok = fc[:, 1] >= 0
        assert np.array_equal(gl[fc[ok, 1]], m.face_cells[L.face_gid[ok], 1])
        # interior faces never touch a ghost
        inner = fc[: L.n_inner_faces]
        assert np.all(inner[:, 0] < L.n_owned) and np.all(inner[:, 1] < L.n_owned)
        for q, (r0, cnt) in L.recv_range.items():
            send = locs[q].owned[locs[q].send_idx[r]]
            assert np.array_equal(send, gl[r0:r0 + cnt])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class LocalOracle:
    """Oracle kernels restricted to one rank's local problem (owned +
    ghost rows, local faces)."""

    def __init__(self, gdisc, part):
        from oracle import _clib

        self.c = _clib
        t = gdisc.tab
        fg = part.face_gid
        own = part.owned
        self.part = part
        self.gas = gdisc.gas
        self.order = t.order
        self.nb, self.nqf, self.nqv = t.n_basis, t.n_face_points, t.n_vol_points
        self.fbL = np.ascontiguousarray(t.face_basis_l[fg])
        self.fbR = np.ascontiguousarray(t.face_basis_r[fg])
        self.face_w = np.ascontiguousarray(t.face_w[fg])
        self.normal = np.ascontiguousarray(gdisc.mesh.face_normal[fg].T)
        self.fcells = np.ascontiguousarray(part.mesh.face_cells)
        self.bc = np.ascontiguousarray(gdisc.bc[fg])
        self.qinf = gdisc.qinf
        self.vol_w = np.ascontiguousarray(t.vol_w[own])
        self.vol_b = np.ascontiguousarray(t.vol_basis[own])
        self.vol_g = np.ascontiguousarray(t.vol_grad[:, own])
        self.minv = np.ascontiguousarray(t.minv[own])
        self.bmean = np.ascontiguousarray(t.basis_mean[own])
        self.cfaces = np.ascontiguousarray(part.mesh.cell_faces[: part.n_owned])
        self.csign = np.ascontiguousarray(part.mesh.cell_fsign[: part.n_owned])
        self.cnf = np.full(part.n_owned, 4, dtype=np.int8)
        self.h = np.ascontiguousarray(gdisc.mesh.cell_h[own])

    def rhs(self, rows):
        L, p = self.c.lib(), self.c.ptr
        nf = self.fcells.shape[0]
        finv = np.zeros((nf, self.nqf, 5))
        errf = np.zeros(nf, dtype=np.uint8)
        L.ora_flux_pass_f64(3, nf, self.nqf, self.nb, p(rows), p(self.fbL), p(self.fbR), p(self.fcells), p(self.bc),
                            p(self.normal), p(self.qinf), self.gas.gamma, 0, p(finv), p(errf))
        n = self.part.n_owned
        res = np.empty((n, 5, self.nb))
        scratch = np.zeros_like(res)
        errc = np.zeros(n, dtype=np.uint8)
        L.ora_rhs_pass_f64(3, n, self.nb, self.nqv, self.nqf, 4, p(rows), p(finv), p(self.vol_w), p(self.vol_b),
                           p(self.vol_g), p(self.cnf), p(self.cfaces), p(self.csign), p(self.face_w), p(self.fbL),
                           p(self.fbR), p(self.minv), self.gas.gamma, p(scratch), p(res), p(errc))
        assert not errf.any() and not errc.any()
        return res

    def dt_min(self, rows):
        L, p = self.c.lib(), self.c.ptr
        n = self.part.n_owned
        out = np.empty(n)
        errc = np.zeros(n, dtype=np.uint8)
        own = np.ascontiguousarray(rows[:n])
        L.ora_dt_pass_f64(3, n, self.nb, p(own), p(self.bmean), p(self.h), self.gas.gamma, 0.0, 0.3, self.order,
                          p(out), p(errc))
        return float(out.min())


def _rank_main(rank, world, port, steps, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = box()
    parts = rcb_partition(m.cell_centroid, world)
    part = build_local(m, parts, rank)
    gdisc = S.make_disc(to_oracle(m), 1, S.Gas(), 0.5, 0.0)
    u_glob = S.initial_state(S.RunSpec(mesh=gdisc.mesh, order=1, mach=0.5, initial="vortex", x0=2.0, y0=1.5), gdisc)
    lo = LocalOracle(gdisc, part)
    halo = HaloExchange(part, "cpu")
    rows_g = np.concatenate([part.owned, part.ghosts])
    u = np.ascontiguousarray(u_glob[rows_g])
    n = part.n_owned

    def exchange(a):
        t = torch.from_numpy(a.reshape(a.shape[0], -1))
        halo.start(t)
        halo.wait()

    for _ in range(steps):
        d = torch.tensor([lo.dt_min(u)], dtype=torch.float64)
        dist.all_reduce(d, op=dist.ReduceOp.MIN)
        dt = float(d.item())
        exchange(u)
        r0 = lo.rhs(u)
        u1 = u.copy()
        u1[:n] = u[:n] + dt * r0
        exchange(u1)
        r1 = lo.rhs(u1)
        u2 = u.copy()
        u2[:n] = 0.75 * u[:n] + 0.25 * (u1[:n] + dt * r1)
        exchange(u2)
        r2 = lo.rhs(u2)
        un = u.copy()
        un[:n] = (1.0 / 3.0) * u[:n] + (2.0 / 3.0) * (u2[:n] + dt * r2)
        u = un
    out_q.put((rank, part.owned, u[:n]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_rk3_equals_serial_bitwise(world):
    steps = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    m = box()
    gdisc = S.make_disc(to_oracle(m), 1, S.Gas(), 0.5, 0.0)
    u = S.initial_state(S.RunSpec(mesh=gdisc.mesh, order=1, mach=0.5, initial="vortex", x0=2.0, y0=1.5), gdisc)
    for _ in range(steps):
        dt = S.min_reduce(S.local_dt_field(gdisc, u, 0.3, 1))
        u = S.rk3_step(u, dt, lambda x: gdisc.rhs(x))
    got = np.empty_like(u)
    for _, owned, rows in results:
        got[owned] = rows
    assert np.array_equal(got, u)


def _host_halo_main(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2209_01877_b200.partition import HostHaloExchange

    m = box()
    parts = rcb_partition(m.cell_centroid, world)
    part = build_local(m, parts, rank)
    # rows = global id encoded in every column; ghosts start as NaN
    gl = np.concatenate([part.owned, part.ghosts])
    rows = torch.full((part.n_rows, 7), float("nan"), dtype=torch.float64)
    rows[: part.n_owned] = torch.from_numpy(np.repeat(part.owned[:, None].astype(np.float64), 7, axis=1))
    h = HostHaloExchange(part, "cpu")
    h.start(rows)
    h.wait()
    dt = torch.tensor([float(rank + 3)], dtype=torch.float64).view(torch.int64)
    h.allreduce(dt, 0)
    s = torch.tensor([1.0 + rank], dtype=torch.float64)
    h.allreduce(s, 1)
    out_q.put((rank, np.array_equal(rows.numpy(), np.repeat(gl[:, None].astype(np.float64), 7, axis=1)),
               float(dt.view(torch.float64).item()), float(s.item())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_host_staged_halo_exchange(world):
    """HostHaloExchange (the transport of tests/test_gpu_multirank.py) over
    gloo: every ghost row arrives from its owner, the dt MIN and norm SUM
    reductions are exact."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_host_halo_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, ok, dtmin, ssum in res:
        assert ok, rank
        assert dtmin == 3.0
        assert ssum == sum(1.0 + r for r in range(world))
