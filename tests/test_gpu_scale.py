"""Parity at the sizes bench.py reports, built exactly as bench.py builds
them (bench.build_cube: device Kuhn cube, seeded shuffle randomize_cells = 1,
device RCM, device face re-sort, device element records, projected vortex):

* C1M (n = 55, 998,250 tets): the device RCM permutation is bit-exact with
  the oracle's restatement of hodg/renumber.py:171-208 (oracle/rcm_oracle.c);
  three SSP-RK3 steps agree with the oracle (all host cores) -- FP64 state
  and residual history <= 1e-12, mixed precision <= 1e-5 on the state and
  10x that on the residual history (a residual is a small difference of
  O(1) fluxes whose FP32 rounding it inherits);
* C4M (n = 87, 3,951,018 tets), P3: one full SSP-RK3 step on the device
  against the oracle on sampled elements -- the oracle evaluates the same
  step on the sub-mesh of the samples' 3-ring neighbourhoods (each stage
  widens the dependency by one ring), with the device run's global dt, and
  the sampled elements' new states agree to <= 1e-12.  (The oracle's
  per-element tables for all 3.95M P3 elements would need ~110 GB.)
"""

import os
import sys

import numpy as np
import pytest

from gpu_helpers import rel, to_oracle
from oracle import renumber as OR
from oracle import solver as S

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

FP64_TOL = 1e-12
MIXED_TOL = 1e-5


@pytest.fixture(scope="module")
def P():
    import paper_2209_01877_b200 as P

    P._lib.lib()
    from oracle import _clib

    _clib.set_threads(os.cpu_count() or 1)
    return P


def _gpu_steps(P, mesh, geo, gas, bcs, state, prec_bits, steps):
    from paper_2209_01877_b200 import _lib
    from paper_2209_01877_b200.dg import _get_disc
    from paper_2209_01877_b200.timestepping import Stepper

    prec = _lib.PREC_F64 if prec_bits == 64 else _lib.PREC_MIXED
    st = Stepper(_get_disc(mesh, geo, gas, bcs), "rk3", prec, "global", 0.3, log_norms=True)
    st.load(state)
    hist, dts = [], []
    for _ in range(steps):
        dts.append(st.dt_value())
        st.step()
        hist.append(st.norms.cpu().numpy().copy())
    st.check(steps)
    return st.state().coeffs.double().cpu().numpy(), np.array(hist), dts


@pytest.fixture(scope="module")
def c1m(P):
    mesh, gas, geo, bcs, state, bw = bench.build_cube(55, 2)
    assert mesh.n_cells == 998250
    spec = S.RunSpec(mesh=to_oracle(mesh), order=2, mach=0.5, initial="vortex", x0=5.0, y0=5.0, cfl=0.3,
                     dt_mode="global", scheme="rk3", max_iterations=3, log_every=1)
    u_ref, hist, _ = S.run(spec)
    return mesh, gas, geo, bcs, state, u_ref, hist


def test_c1m_device_rcm_bitexact(P):
    m = P.generate_tet_box(55, extent=bench.EXTENT, bc=bench.CUBE_BC, device="cuda")
    shuffled = P.apply_permutation(m, P.random_permutation(m.n_cells, 1))
    perm = P.rcm(P.build_adjacency(shuffled))
    om = to_oracle(shuffled)
    fwd, inv = OR.rcm(OR.adjacency(om))
    assert np.array_equal(perm.forward, fwd) and np.array_equal(perm.inverse, inv)


@pytest.mark.parametrize("prec_bits", [64, 32])
def test_c1m_three_steps_against_oracle(P, c1m, prec_bits):
    mesh, gas, geo, bcs, state, u_ref, hist = c1m
    got, ghist, dts = _gpu_steps(P, mesh, geo, gas, bcs, state, prec_bits, 3)
    tol = FP64_TOL if prec_bits == 64 else MIXED_TOL
    assert rel(got, u_ref) <= tol, rel(got, u_ref)
    assert rel(ghist, np.array(hist.res)) <= (tol if prec_bits == 64 else 10 * tol)
    if prec_bits == 64:
        np.testing.assert_allclose(dts, hist.dts, rtol=1e-13)


def _rings(mesh, seeds, depth):
    """Element sets within `depth` face-neighbour steps of the seeds."""
    cur = np.unique(seeds)
    allset = set(cur.tolist())
    for _ in range(depth):
        nb = mesh.cell_neighbors[cur].ravel()
        nb = np.unique(nb[nb >= 0])
        new = np.array(sorted(set(nb.tolist()) - allset), dtype=np.int64)
        allset.update(new.tolist())
        cur = new
    return np.array(sorted(allset), dtype=np.int64)


def _sub_patches(mesh, remap, tets):
    """The full mesh's boundary triangles that bound the sub-mesh, plus the
    cut faces as far field (they only reach ring 3, never the samples)."""
    from collections import Counter

    cnt = Counter(tuple(sorted(int(x) for x in t[list(f)])) for t in tets
                  for f in ((1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2)))
    outer = {k for k, c in cnt.items() if c == 1}
    specs, used = [], set()
    for p in mesh.patches:
        tris = [tuple(int(remap[x]) for x in mesh.face_nodes[f]) for f in p.face_ids]
        tris = [t for t in tris if min(t) >= 0 and tuple(sorted(t)) in outer]
        used.update(tuple(sorted(t)) for t in tris)
        specs.append((p.name, p.kind, tris))
    specs.append(("cut", "far_field", sorted(outer - used)))
    return specs


def test_c4m_p3_step_sampled_against_oracle(P):
    mesh, gas, geo, bcs, state, bw = bench.build_cube(87, 3)
    assert mesh.n_cells == 3951018
    got, _, dts = _gpu_steps(P, mesh, geo, gas, bcs, state, 64, 1)
    rng = np.random.default_rng(7)
    # samples in the vortex core, near walls / far field and at random
    bnd = np.flatnonzero((mesh.cell_neighbors < 0).any(axis=1))
    seeds = np.concatenate([rng.choice(mesh.n_cells, 40, replace=False), rng.choice(bnd, 24, replace=False)])
    sub = _rings(mesh, seeds, 3)
    # sub-mesh: its elements' nodes renumbered in ascending order (element
    # vertex order kept) and the full mesh's boundary triangles it contains
    nodes = np.unique(mesh.cell_nodes[sub])
    remap = np.full(mesh.n_nodes, -1, dtype=np.int64)
    remap[nodes] = np.arange(nodes.size)
    tets = remap[mesh.cell_nodes[sub]]
    specs = _sub_patches(mesh, remap, tets)
    from oracle import mesh as OM

    om = OM.build_tet_mesh(mesh.node_xy[nodes], tets, specs)
    disc = S.make_disc(om, 3, S.Gas(), 0.5, 0.0)
    c0 = state.coeffs.double().cpu().numpy()[sub]
    u = S.rk3_step(np.ascontiguousarray(c0), dts[0], lambda x: disc.rhs(x))
    pos = np.searchsorted(sub, np.unique(seeds))
    assert rel(got[np.unique(seeds)], u[pos]) <= FP64_TOL
