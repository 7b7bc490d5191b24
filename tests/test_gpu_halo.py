"""The library's NCCL halo exchange (csrc/halo.cu) on one GPU: a 1-rank
communicator whose rank is its own peer.  The two-partition case keeps both
partitions' rows in one buffer and lists the rank twice as a peer (NCCL
matches same-peer sends and receives in issue order), so the exchange fills
both ghost blocks exactly as two ranks would; the partitioned residual must
then equal the serial one bitwise."""

import types

import numpy as np
import pytest

import gpu_helpers
from gpu_helpers import oracle_state

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2209_01877_b200 as P

    P._lib.lib()
    return P


def test_self_exchange_moves_rows(P):
    import torch

    from paper_2209_01877_b200.partition import NativeHaloExchange

    rs, n_owned, n_ghost = 50, 40, 9
    rows = torch.randn(n_owned + n_ghost, rs, dtype=torch.float64, device="cuda")
    send = np.array([3, 17, 5, 39, 0, 22, 8, 30, 11], dtype=np.int32)
    part = types.SimpleNamespace(send_idx={0: send}, recv_range={0: (n_owned, n_ghost)})
    h = NativeHaloExchange(part, rs, 0, 1, NativeHaloExchange.unique_id())
    want = rows[torch.as_tensor(send, dtype=torch.int64, device="cuda")].clone()
    h.start(rows)
    h.wait()
    torch.cuda.synchronize()
    assert torch.equal(rows[n_owned:], want)
    h.close()


def test_two_partitions_through_the_native_exchange(P):
    import torch

    from paper_2209_01877_b200.dg import Discretization, _get_disc
    from paper_2209_01877_b200.geometry import compute_geometry
    from paper_2209_01877_b200.partition import NativeHaloExchange, build_local, rcb_partition

    m = P.perturb_interior_nodes(P.generate_tet_box(5, bc=gpu_helpers.MIXED_BC), 0.1, 4)
    order = 2
    gas = P.GasModel()
    geo = P.compute_geometry(m, order)
    bcs = P.BoundaryConditions(P.freestream_conserved(gas, 0.4, 10.0))
    _, c = oracle_state(m, order)
    full = _get_disc(m, geo, gas, bcs)
    rows_g = full.to_reference(torch.from_numpy(c).cuda())
    ref = full.residual_rows(rows_g, full.face_flux(rows_g, 64), 64)

    parts = rcb_partition(m.cell_centroid, 2)
    lp = [build_local(m, parts, r) for r in range(2)]
    off = [0, lp[0].n_rows]
    rs = full.rs
    big = torch.full((lp[0].n_rows + lp[1].n_rows, rs), float("nan"), dtype=torch.float64, device="cuda")
    for r in range(2):  # owned rows only; ghosts come through the exchange
        own = torch.as_tensor(lp[r].owned, device="cuda")
        big[off[r]:off[r] + lp[r].n_owned] = rows_g.index_select(0, own)
    # one plan, rank 0 listed twice as a peer: part 0 -> part 1, part 1 -> part 0
    plan = types.SimpleNamespace(send_idx={}, recv_range={})
    entries = []
    for src, dst in ((0, 1), (1, 0)):
        send = np.asarray(lp[src].send_idx[dst], dtype=np.int64) + off[src]
        first, cnt = lp[dst].recv_range[src]
        entries.append((send, first + off[dst], cnt))
    import ctypes as C

    from paper_2209_01877_b200 import _lib

    L = _lib.lib()
    peers = np.zeros(2, dtype=np.int32)
    send_count = np.array([e[0].size for e in entries], dtype=np.int64)
    send_rows = np.concatenate([e[0] for e in entries]).astype(np.int32)
    recv_first = np.array([e[1] for e in entries], dtype=np.int64)
    recv_count = np.array([e[2] for e in entries], dtype=np.int64)
    uid = C.create_string_buffer(NativeHaloExchange.unique_id(), 128)
    h = C.c_void_p()
    _lib.check(L.hodg_halo_create(1, 0, uid, 2, peers.ctypes.data, send_count.ctypes.data, send_rows.ctypes.data,
                                  recv_first.ctypes.data, recv_count.ctypes.data, rs, C.byref(h)), "create")
    _lib.check(L.hodg_halo_exchange(h, _lib.ptr(big), _lib.stream_ptr()), "exchange")
    torch.cuda.synchronize()
    L.hodg_halo_destroy(h)
    assert not torch.isnan(big).any()
    for r in range(2):
        part = lp[r]
        d = Discretization(part.mesh, compute_geometry(part.mesh, order, split=part.n_inner_faces), gas, bcs,
                           n_elems=part.n_owned)
        rows = big[off[r]:off[r] + part.n_rows].contiguous()
        gl = torch.as_tensor(np.concatenate([part.owned, part.ghosts]), device="cuda")
        assert torch.equal(rows, rows_g.index_select(0, gl))
        d.reset_errors()
        hb = d.face_buffer(64)
        d.face_flux(rows, 64, hb)
        res = d.residual_rows(rows, hb, 64, res=d.new_state())
        d.raise_errors()
        own = torch.as_tensor(part.owned, device="cuda")
        assert torch.equal(res[: part.n_owned], ref.index_select(0, own)), r


@pytest.mark.timeout(600)
@pytest.mark.parametrize("use_graph", [False, True])
def test_distributed_stepper_native_halo_single_rank(P, use_graph):
    """DistributedStepper on a 1-rank NCCL group with the native exchange (no
    peers): same states as the single-GPU stepper -- launched eagerly, and
    captured in a CUDA graph with the NCCL all-reduces inside (relaxed
    capture mode; close() drops the graphs before the communicator)."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2209_01877_b200.dg import _get_disc
    from paper_2209_01877_b200.distributed import DistributedStepper, owned_state, setup_partitioned
    from paper_2209_01877_b200.timestepping import Stepper

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        m = P.generate_tet_box(4, bc=gpu_helpers.MIXED_BC)
        gas = P.GasModel()
        bcs = P.BoundaryConditions(P.freestream_conserved(gas, 0.4, 10.0))
        geo = P.compute_geometry(m, 1)
        _, c = oracle_state(m, 1)
        st0 = P.DofState(torch.from_numpy(c).cuda())
        part, disc = setup_partitioned(m, 1, gas, bcs, 0, 1)
        ds = DistributedStepper(part, disc, "rk3", 64, 0.3, log_norms=True, halo="native", use_graph=use_graph)
        ds.load(owned_state(st0, part))
        ref = Stepper(_get_disc(m, geo, gas, bcs), "rk3", 64, "global", 0.3, use_graph=False)
        ref.load(st0)
        for _ in range(3):
            ds.step()
            ref.step()
        ds.check()
        ref.check()
        own = torch.as_tensor(part.owned, device="cuda")
        assert torch.equal(ds.state().coeffs, ref.state().coeffs.index_select(0, own))
        assert torch.allclose(ds.norms, ref.norms, rtol=1e-12, atol=0)  # (summation order differs)
        ds.close()
    finally:
        dist.destroy_process_group()

