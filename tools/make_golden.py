"""Regenerate tests/golden/ from the reference itself.

Runs ONLY in the build container, where the read-only reference is at
/root/reference (it does not exist on the GPU box).  It imports the
reference package `hodg` (numba) and writes:

  residuals_dp.csv, residuals_mp.csv   the reference's 150-step fixture runs
                                       (pkg/tests/test_fixtures.py:43-58),
                                       asserted equal to pkg/fixtures/*
  spy_before.mtx, spy_after.mtx,       RCM spy fixtures
  spy_path3.mtx                        (pkg/tests/test_fixtures.py:31-40)
  ref_rhs2d.npz                        dg.rhs of perturbed projected states on
                                       the reference test corpus
                                       (pkg/tests/conftest.py:47-61), orders 0-2
  ref_flux.npz                         roe_flux / boundary_state on 2000 seeded
                                       random states (pkg/tests/test_physics.py)
  ref_rcm.npz                          rcm permutations of seeded random graphs,
                                       including disconnected ones
  ref_ns2d.npz                         the viscous (ivis = 1, BR1) passes on the
                                       corpus: aux gradient, qhat, finv, fvis,
                                       fqhat and the residual, orders 0-2, at
                                       float64 and float32
  field_tri_perturbed_p2.vtk           reference write_vtk of a corpus state
  mesh_quad_perturbed.hodg,            reference save_mesh output (HODG-MESH v1)
  mesh_tri_perturbed.hodg              of two corpus meshes
  residuals_ns_dp.csv,                 reference Navier-Stokes runs: a viscous
  residuals_ns_mp.csv                  vortex (order 2) and a small version of
                                       the c07 pulse case (mp_fixed switch)

Usage:  python tools/make_golden.py
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
os.environ.setdefault("NUMBA_NUM_THREADS", "16")
REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))

import numpy as np  # noqa: E402

import hodg  # noqa: E402,F401  (sets NUMBA_NUM_THREADS before numba import)
from hodg import dg, flows  # noqa: E402
from hodg import mesh as M  # noqa: E402
from hodg.config import RunConfig  # noqa: E402
from hodg.geometry import compute_geometry  # noqa: E402
from hodg.output import write_residual_csv  # noqa: E402
from hodg.perf import MachineModel, PerfSample, emit_roofline_csv, emit_timing_csv  # noqa: E402
from hodg.physics import Conserved, GasModel, boundary_state, roe_flux  # noqa: E402
from hodg.renumber import AdjacencyGraph, apply_permutation, build_adjacency, export_spy, random_permutation, rcm  # noqa: E402
from hodg.timestepping import run  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def corpus():
    # pkg/tests/conftest.py:47-61
    return [
        ("quad_4x4", M.generate_quad_grid(4, 4)),
        ("quad_stretched", M.generate_quad_grid(3, 3, (0.0, 0.0, 2.0, 0.7))),
        ("tri_4x3", M.generate_tri_grid(4, 3)),
        ("quad_perturbed", M.perturb_interior_nodes(M.generate_quad_grid(6, 5), 0.15, seed=3)),
        ("tri_perturbed", M.perturb_interior_nodes(M.generate_tri_grid(5, 4), 0.12, seed=7)),
    ]


def main():
    os.makedirs(OUT, exist_ok=True)
    for name, mode, kw in [("residuals_dp.csv", "dp", {}), ("residuals_mp.csv", "mp_fixed", {"switch_iter": 60})]:
        cfg = RunConfig(gen_kind="quad", gen_nx=16, gen_ny=16, gen_extent=(0.0, 0.0, 10.0, 10.0),
                        initial_kind="vortex", initial_x0=5.0, initial_y0=5.0, mach=0.5, order=1,
                        max_iterations=150, log_every=1, precision_mode=mode, **kw)
        path = os.path.join(OUT, name)
        write_residual_csv(path, run(cfg).history)
        assert open(path, "rb").read() == open(os.path.join(REF, "fixtures", name), "rb").read()

    mesh = M.generate_quad_grid(63, 64)
    shuffled = apply_permutation(mesh, random_permutation(mesh.n_cells, seed=4))
    graph = build_adjacency(shuffled)
    export_spy(graph, None, os.path.join(OUT, "spy_before.mtx"))
    export_spy(graph, rcm(graph), os.path.join(OUT, "spy_after.mtx"))
    export_spy(AdjacencyGraph.from_edges(3, [(0, 1), (1, 2)]), None, os.path.join(OUT, "spy_path3.mtx"))
    for n in ("spy_before.mtx", "spy_after.mtx", "spy_path3.mtx"):
        assert open(os.path.join(OUT, n), "rb").read() == open(os.path.join(REF, "fixtures", n), "rb").read()

    # synthetic perf fixtures (pkg/tests/test_fixtures.py:61-78)
    samples = [
        ("grid4", PerfSample(wall_seconds=0.020, flops=4.0e8, dram_bytes=3.2e9, iterations=1)),
        ("grid5", PerfSample(wall_seconds=0.085, flops=1.6e9, dram_bytes=1.28e10, iterations=1)),
        ("dense", PerfSample(wall_seconds=0.010, flops=5.0e9, dram_bytes=2.0e8, iterations=1)),
    ]
    machines = [MachineModel("cpu-node", 3.0e12, 2.0e11), MachineModel("gpu-node", 7.0e12, 9.0e11)]
    emit_roofline_csv(samples, machines, os.path.join(OUT, "roofline.csv"))
    emit_timing_csv([("grid4", 1, 0.0400), ("grid4", 2, 0.0215), ("grid4", 8, 0.0095),
                     ("grid5", 1, 0.1660), ("grid5", 2, 0.0890), ("grid5", 8, 0.0410)], os.path.join(OUT, "timing.csv"))
    for n in ("roofline.csv", "timing.csv"):
        assert open(os.path.join(OUT, n), "rb").read() == open(os.path.join(REF, "fixtures", n), "rb").read()

    # residuals of perturbed freestream / vortex projections on the corpus
    gas = GasModel()
    arrays = {}
    for name, m in corpus():
        for order in (0, 1, 2):
            geo = compute_geometry(m, order)
            bcs = dg.BoundaryConditions(flows.freestream_conserved(gas, 0.4, 10.0))
            st = dg.project_initial(m, geo, lambda x, y: flows.vortex_primitive(
                gas, 0.4, 10.0, 2.0, 0.5, 0.4, 0.0, x, y), gas)
            rng = np.random.default_rng(order + 11)
            st.coeffs[:, :, 0] *= 1.0 + 0.01 * rng.random(st.coeffs.shape[:2])
            r = dg.rhs(st, m, geo, bcs, gas)
            arrays[f"{name}_p{order}_coeffs"] = st.coeffs
            arrays[f"{name}_p{order}_res"] = r.res
            # reduced-precision (float32) residual of the same state
            st32 = dg.DofState(st.coeffs.astype(np.float32))
            arrays[f"{name}_p{order}_res32"] = dg.rhs(st32, m, geo, bcs, gas).res
    np.savez_compressed(os.path.join(OUT, "ref_rhs2d.npz"), **arrays)

    # HODG-MESH v1 files written by the reference, and a VTK field of a
    # corpus state (hodg/output.py:54-83)
    from hodg.output import write_vtk

    for name, m in corpus():
        if name in ("quad_perturbed", "tri_perturbed"):
            M.save_mesh(m, os.path.join(OUT, f"mesh_{name}.hodg"))
        if name == "tri_perturbed":
            geo = compute_geometry(m, 2)
            st = dg.DofState(np.load(os.path.join(OUT, "ref_rhs2d.npz"))[f"{name}_p2_coeffs"])
            write_vtk(os.path.join(OUT, "field_tri_perturbed_p2.vtk"), m, st, geo, gas)

    # viscous passes (pkg/tests/test_dg.py:12, mu = 0.02)
    ns = GasModel(mu_dyn=0.02, ivis=1)
    arrays = {}
    for name, m in corpus():
        for order in (0, 1, 2):
            geo = compute_geometry(m, order)
            bcs = dg.BoundaryConditions(flows.freestream_conserved(ns, 0.4, 10.0))
            st = dg.project_initial(m, geo, lambda x, y: flows.vortex_primitive(
                ns, 0.4, 10.0, 2.0, 0.5, 0.4, 0.0, x, y), ns)
            rng = np.random.default_rng(order + 23)
            st.coeffs[:, :, 0] *= 1.0 + 0.01 * rng.random(st.coeffs.shape[:2])
            arrays[f"{name}_p{order}_coeffs"] = st.coeffs
            for tag, s_ in (("", st), ("32", dg.DofState(st.coeffs.astype(np.float32)))):
                aux = dg.compute_aux_gradient(s_, m, geo, bcs, ns)
                buf = dg.face_flux_pass(s_, aux, m, geo, bcs, ns)
                arrays[f"{name}_p{order}_aux{tag}"] = aux.z
                arrays[f"{name}_p{order}_finv{tag}"] = buf.inviscid
                arrays[f"{name}_p{order}_fvis{tag}"] = buf.viscous
                arrays[f"{name}_p{order}_fqhat{tag}"] = buf.qhat
                arrays[f"{name}_p{order}_res{tag}"] = dg.accumulate_rhs(s_, aux, buf, m, geo, bcs, ns).res
    np.savez_compressed(os.path.join(OUT, "ref_ns2d.npz"), **arrays)
    for name, kw in [
        ("residuals_ns_dp.csv", dict(gen_kind="quad", gen_nx=12, gen_ny=12, gen_extent=(0.0, 0.0, 10.0, 10.0),
                                     initial_kind="vortex", initial_x0=5.0, initial_y0=5.0, mach=0.5, order=2,
                                     ivis=1, mu_dyn=0.01, max_iterations=60)),
        ("residuals_ns_mp.csv", dict(gen_kind="quad", gen_nx=96, gen_ny=4, gen_extent=(0.0, 0.0, 12.0, 0.5),
                                     initial_kind="pulse", initial_x0=6.0, initial_y0=0.25, pulse_amplitude=0.2,
                                     pulse_sigma=0.3, mach=0.4, order=1, cfl=0.5, ivis=1, mu_dyn=0.002,
                                     max_iterations=120, precision_mode="mp_fixed", switch_iter=70)),
    ]:
        cfg = RunConfig(log_every=1, **kw)
        write_residual_csv(os.path.join(OUT, name), run(cfg).history)

    # point fluxes: Roe and boundary states on random admissible states
    rng = np.random.default_rng(2024)
    n = 2000
    qs = []
    for _ in range(2 * n):
        rho = rng.uniform(0.2, 3.0)
        u, v = rng.uniform(-2.0, 2.0, 2)
        p = rng.uniform(0.2, 3.0)
        qs.append((rho, rho * u, rho * v, p / 0.4 + 0.5 * rho * (u * u + v * v)))
    qs = np.array(qs)
    ang = rng.uniform(0, 2 * np.pi, n)
    nrm = np.stack([np.cos(ang), np.sin(ang)], axis=1)
    fs = Conserved(1.0, 0.5 * np.sqrt(1.4), 0.0, 1.0 / 0.4 + 0.5 * 0.25 * 1.4)
    roe = np.array([roe_flux(Conserved(*qs[i]), Conserved(*qs[n + i]), nrm[i], gas) for i in range(n)])
    bnd = {k: np.array([boundary_state(Conserved(*qs[i]), k, nrm[i], fs, gas).__dict__ and
                        [getattr(boundary_state(Conserved(*qs[i]), k, nrm[i], fs, gas), a)
                         for a in ("rho", "rho_u", "rho_v", "e")] for i in range(n)])
           for k in ("far_field", "slip_wall", "no_slip_wall")}
    np.savez_compressed(os.path.join(OUT, "ref_flux.npz"), q=qs, normal=nrm, roe=roe,
                        freestream=np.array([fs.rho, fs.rho_u, fs.rho_v, fs.e]),
                        far=bnd["far_field"], slip=bnd["slip_wall"], noslip=bnd["no_slip_wall"])

    # RCM permutations of random graphs (connected and disconnected)
    rng = np.random.default_rng(7)
    graphs = {}
    for t in range(60):
        nv = int(rng.integers(1, 400))
        ne = int(rng.integers(0, 3 * nv))
        e = rng.integers(0, nv, size=(ne, 2))
        e = e[e[:, 0] != e[:, 1]]
        g = AdjacencyGraph.from_edges(nv, e)
        graphs[f"g{t}_n"] = np.array([nv])
        graphs[f"g{t}_edges"] = e
        graphs[f"g{t}_fwd"] = rcm(g).forward
    np.savez_compressed(os.path.join(OUT, "ref_rcm.npz"), **graphs)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
