"""The multi-rank path with the product's CUDA kernels: two processes on the
one GPU of the test box run DistributedStepper (RCB partition, owned +
ghost rows, interior / partition face ranges, owned-only element kernel,
per-stage halo exchange, dt MIN and norm SUM all-reduces) over a gloo group
with the ghost rows staged through host memory (HostHaloExchange), and the
assembled state equals the serial Stepper's bitwise.

Only the halo transport differs from an NVLink run (NCCL send / recv
there): the partition, local numbering, kernels and reduction plumbing are
the ones bench.py --gpus N drives.  Ranks sharing a GPU never run kernels
that wait on each other -- every transfer here is synchronous with the host."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BOX_BC = {"xmin": "far_field", "xmax": "far_field", "ymin": "slip_wall", "ymax": "far_field",
          "zmin": "slip_wall", "zmax": "no_slip_wall"}


def _mesh():
    from paper_2209_01877_b200 import mesh as M

    return M.perturb_interior_nodes(M.generate_tet_box(5, 4, 3, extent=(0.0, 0.0, 0.0, 5.0, 4.0, 3.0), bc=BOX_BC),
                                    0.1, 3)


def _setup(P, m, order):
    gas = P.GasModel()
    bcs = P.BoundaryConditions(P.freestream_conserved(gas, 0.5, 5.0))
    geo = P.compute_geometry(m, order)
    state = P.project_initial(m, geo, lambda x, y, z: P.vortex_primitive(gas, 0.5, 5.0, 5.0, 2.5, 2.0, 0.0, x, y),
                              gas)
    return gas, bcs, geo, state


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, order, prec_bits, steps, out_q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2209_01877_b200 as P
    from paper_2209_01877_b200 import _lib
    from paper_2209_01877_b200.distributed import DistributedStepper, owned_state, setup_partitioned

    m = _mesh()
    gas, bcs, geo, state = _setup(P, m, order)
    part, disc = setup_partitioned(m, order, gas, bcs, rank, world)
    prec = _lib.PREC_F64 if prec_bits == 64 else _lib.PREC_MIXED
    st = DistributedStepper(part, disc, "rk3", prec, 0.3, log_norms=True, halo="host")
    st.load(owned_state(state, part))
    norms = []
    for _ in range(steps):
        st.step()
        norms.append(st.norms.cpu().numpy().copy())
    st.check(steps)
    out = st.state().coeffs.cpu().numpy()
    out_q.put((rank, part.owned, out, np.array(norms), st.dt_value()))
    dist.barrier()
    st.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("order,prec_bits,world", [(2, 64, 2), (1, 64, 2), (2, 32, 2), (2, 64, 3)])
def test_partitioned_cuda_equals_serial_bitwise(order, prec_bits, world):
    import torch
    import torch.multiprocessing as mp

    import paper_2209_01877_b200 as P
    from paper_2209_01877_b200 import _lib
    from paper_2209_01877_b200.dg import _get_disc
    from paper_2209_01877_b200.timestepping import Stepper

    steps = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, order, prec_bits, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0

    m = _mesh()
    gas, bcs, geo, state = _setup(P, m, order)
    prec = _lib.PREC_F64 if prec_bits == 64 else _lib.PREC_MIXED
    st = Stepper(_get_disc(m, geo, gas, bcs), "rk3", prec, "global", 0.3, log_norms=True)
    st.load(state)
    ref_norms = []
    for _ in range(steps):
        st.step()
        ref_norms.append(st.norms.cpu().numpy().copy())
    ref = st.state().coeffs.cpu().numpy()
    got = np.empty_like(ref)
    for _, owned, rows, norms, dt in results:
        got[owned] = rows
        # norms: the same terms summed in a different order across ranks
        np.testing.assert_allclose(norms, np.array(ref_norms), rtol=1e-12)
        assert dt == st.dt_value()
    assert np.array_equal(got, ref)
    torch.cuda.synchronize()
