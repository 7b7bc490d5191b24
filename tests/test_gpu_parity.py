"""CUDA residual path vs the CPU oracle (which is pinned to the reference's
golden files).  North-star tolerances: FP64 relative L2 <= 1e-12, mixed
precision <= 1e-5."""

import numpy as np
import pytest

import gpu_helpers
from gpu_helpers import meshes, oracle_state, rel, to_oracle
from oracle import solver as S

pytestmark = pytest.mark.gpu

FP64_TOL = 1e-12
MIXED_TOL = 1e-5


@pytest.fixture(scope="module")
def P():
    import paper_2209_01877_b200 as P

    P._lib.lib()  # fail loudly if the CUDA library / device is missing
    return P


def gpu_setup(P, m, order, mach=0.4, angle=10.0, flux="roe"):
    gas = P.GasModel()
    geo = P.compute_geometry(m, order)
    bcs = P.BoundaryConditions(P.freestream_conserved(gas, mach, angle), flux)
    return gas, geo, bcs


@pytest.mark.parametrize("order", [0, 1, 2, 3])
@pytest.mark.parametrize("flux,kind", [("roe", 0), ("llf", 1)])
def test_rhs_fp64_matches_oracle(P, order, flux, kind):
    import torch

    for name, m in meshes():
        disc, c = oracle_state(m, order, flux_kind=kind)
        gas, geo, bcs = gpu_setup(P, m, order, flux=flux)
        r = P.rhs(P.DofState(torch.from_numpy(c).cuda()), m, geo, bcs, gas).res.cpu().numpy()
        ref = disc.rhs(c)
        assert rel(r, ref) <= FP64_TOL, (name, order, flux, rel(r, ref))


@pytest.mark.parametrize("order", [1, 2, 3])
def test_face_flux_fp64_matches_oracle(P, order):
    import torch

    for name, m in meshes():
        disc, c = oracle_state(m, order)
        gas, geo, bcs = gpu_setup(P, m, order)
        buf = P.face_flux_pass(P.DofState(torch.from_numpy(c).cuda()), None, m, geo, bcs, gas)
        f = buf.inviscid.cpu().numpy()
        ref = disc.flux_pass(c)
        assert f.shape == ref.shape
        assert rel(f, ref) <= FP64_TOL, (name, order, rel(f, ref))
        # accumulate_rhs on the oracle's own face buffer
        res = P.accumulate_rhs(P.DofState(torch.from_numpy(c).cuda()), None,
                               P.FaceFluxBuffer(torch.from_numpy(ref).cuda()), m, geo, bcs, gas)
        assert rel(res.res.cpu().numpy(), disc.rhs_pass(c, ref)) <= FP64_TOL


@pytest.mark.parametrize("order", [1, 2, 3])
def test_rhs_mixed_matches_oracle(P, order):
    import torch

    for name, m in meshes():
        disc, c = oracle_state(m, order)
        gas, geo, bcs = gpu_setup(P, m, order)
        st = P.DofState(torch.from_numpy(c).cuda().to(torch.float32))
        r = P.rhs(st, m, geo, bcs, gas).res.cpu().numpy()
        ref = disc.rhs(np.ascontiguousarray(c.astype(np.float32).astype(np.float64)))  # FP64 oracle, same state
        ref32 = disc.rhs(np.ascontiguousarray(c.astype(np.float32)))  # the reference's own MP kernels
        # the residual is a small difference of O(1) fluxes, so FP32 flux
        # rounding shows at ~1e-6..1e-5 of its norm; the solution after N
        # steps is held to 1e-5 (test_run_mixed_matches_fp64_oracle)
        assert rel(r, ref) <= 5 * MIXED_TOL, (name, order, rel(r, ref))
        assert rel(r, ref32) <= 5 * MIXED_TOL, (name, order, rel(r, ref32))


@pytest.mark.parametrize("order", [0, 1, 2, 3])
def test_freestream_preserved(P, order):
    import torch

    for name, m in meshes():
        if "mixed_bc" in name:  # walls are not aligned with the freestream: not a steady state
            continue
        gas, geo, bcs = gpu_setup(P, m, order, mach=0.3)
        w = P.freestream_primitive(gas, 0.3, 10.0)
        st = P.project_initial(m, geo, lambda x, y, z: w, gas)
        r = P.rhs(st, m, geo, bcs, gas).res
        scale = 1e-11 * (10.0 ** order)
        assert float(r.abs().max()) < scale, (name, order, float(r.abs().max()))


def test_projection_matches_oracle(P):
    for order in (1, 2, 3):
        for name, m in meshes():
            disc, _ = oracle_state(m, order)
            gas, geo, bcs = gpu_setup(P, m, order)
            f = lambda x, y, z: P.vortex_primitive(gas, 0.4, 10.0, 2.0, 1.0, 0.5, 0.0, x, y)  # noqa: E731
            c = P.project_initial(m, geo, f, gas).coeffs.cpu().numpy()
            om = disc.mesh
            ref = S.project_initial(om, disc.tab, lambda x, y, z: S.vortex_primitive(
                S.Gas(), 0.4, 10.0, 2.0, 1.0, 0.5, 0.0, x, y, dim=3), S.Gas())
            assert rel(c, ref) <= 1e-12, (name, order, rel(c, ref))


def test_local_dt_and_min_reduce(P):
    import torch

    for order in (1, 2):
        for name, m in meshes():
            disc, c = oracle_state(m, order)
            gas, geo, bcs = gpu_setup(P, m, order)
            dt = P.local_dt_field(P.DofState(torch.from_numpy(c).cuda()), m, geo, gas, 0.3, order, bcs)
            ref = S.local_dt_field(disc, c, 0.3, order)
            assert rel(dt.cpu().numpy(), ref) <= 1e-13
            assert P.min_reduce(dt) == float(np.min(dt.cpu().numpy()))


@pytest.mark.parametrize("scheme", ["rk2", "rk3"])
@pytest.mark.parametrize("dt_mode", ["global", "local"])
def test_run_history_matches_oracle(P, scheme, dt_mode):
    """10 steps of the fused stepper vs the oracle's RK loop: residual
    history and final state within 1e-12 (BASELINE config 1 shape)."""
    m = P.perturb_interior_nodes(P.generate_tet_box(4, extent=(0.0, 0.0, 0.0, 10.0, 10.0, 2.5),
                                                    bc={"xmin": "far_field", "xmax": "far_field",
                                                        "ymin": "far_field", "ymax": "far_field",
                                                        "zmin": "slip_wall", "zmax": "slip_wall"}), 0.1, 3)
    cfg = P.RunConfig(order=1, mach=0.5, initial_kind="vortex", initial_x0=5.0, initial_y0=5.0, cfl=0.3,
                      dt_mode=dt_mode, scheme=scheme, max_iterations=10, log_every=1)
    art = P.run(cfg, mesh=m)
    spec = S.RunSpec(mesh=to_oracle(m), order=1, mach=0.5, initial="vortex", x0=5.0, y0=5.0, cfl=0.3,
                     dt_mode=dt_mode, scheme=scheme, max_iterations=10, log_every=1)
    u, hist, _ = S.run(spec)
    assert rel(art.final_state.coeffs.cpu().numpy(), u) <= FP64_TOL
    assert rel(np.array(art.history.res), np.array(hist.res)) <= FP64_TOL
    assert rel(np.array(art.history.dts), np.array(hist.dts)) <= FP64_TOL


def test_rk_functional_api_matches_fused(P):
    import torch

    m = P.generate_tet_box(3)
    gas, geo, bcs = gpu_setup(P, m, 2)
    disc, c = oracle_state(m, 2)
    st = P.DofState(torch.from_numpy(c).cuda())
    dt = P.min_reduce(P.local_dt_field(st, m, geo, gas, 0.3, 2, bcs))
    calls = []

    def fn(s):
        calls.append(1)
        return P.rhs(s, m, geo, bcs, gas)

    out = P.rk3_step(st, dt, fn)
    assert len(calls) == 3
    ref = S.rk3_step(c, dt, lambda x: disc.rhs(x))
    assert rel(out.coeffs.cpu().numpy(), ref) <= FP64_TOL
    out2 = P.rk2_step(st, dt, fn)
    ref2 = S.rk2_step(c, dt, lambda x: disc.rhs(x))
    assert rel(out2.coeffs.cpu().numpy(), ref2) <= FP64_TOL


def test_admissibility_error_carries_cell_and_iteration(P):
    import torch

    m = P.generate_tet_box(3)
    gas, geo, bcs = gpu_setup(P, m, 1)
    w = P.freestream_primitive(gas, 0.3, 10.0)
    st = P.project_initial(m, geo, lambda x, y, z: w, gas)
    st.coeffs[4, 0, 0] = -1.0
    st.iteration = 17
    with pytest.raises(P.AdmissibilityError) as err:
        P.rhs(st, m, geo, bcs, gas)
    assert "17" in str(err.value)
    assert err.value.face is not None or err.value.cell == 4


def test_deterministic_bitwise(P):
    import torch

    m = P.perturb_interior_nodes(P.generate_tet_box(5), 0.1, 2)
    gas, geo, bcs = gpu_setup(P, m, 2)
    _, c = oracle_state(m, 2)
    st = P.DofState(torch.from_numpy(c).cuda())
    r1 = P.rhs(st, m, geo, bcs, gas).res.clone()
    r2 = P.rhs(st, m, geo, bcs, gas).res
    assert torch.equal(r1, r2)


@pytest.mark.parametrize("order", [1, 2])
def test_run_mixed_matches_fp64_oracle(P, order):
    """Mixed precision (FP32 flux / quadrature, FP64 state and accumulation):
    10 SSP-RK3 steps within the stated 1e-5 of the FP64 oracle."""
    m = P.perturb_interior_nodes(P.generate_tet_box(4, extent=(0.0, 0.0, 0.0, 10.0, 10.0, 2.5),
                                                    bc={"xmin": "far_field", "xmax": "far_field",
                                                        "ymin": "far_field", "ymax": "far_field",
                                                        "zmin": "slip_wall", "zmax": "slip_wall"}), 0.1, 3)
    cfg = P.RunConfig(order=order, mach=0.5, initial_kind="vortex", initial_x0=5.0, initial_y0=5.0, cfl=0.3,
                      dt_mode="global", scheme="rk3", max_iterations=10, log_every=1, precision_mode="sp")
    art = P.run(cfg, mesh=m)
    spec = S.RunSpec(mesh=to_oracle(m), order=order, mach=0.5, initial="vortex", x0=5.0, y0=5.0, cfl=0.3,
                     dt_mode="global", scheme="rk3", max_iterations=10, log_every=1)
    u, hist, _ = S.run(spec)
    assert all(b == 32 for b in art.history.precision)
    assert rel(art.final_state.coeffs.cpu().numpy(), u) <= MIXED_TOL
    assert rel(np.array(art.history.res), np.array(hist.res)) <= 10 * MIXED_TOL


@pytest.mark.parametrize("nparts", [2, 3])
def test_partitioned_residual_bitwise_on_one_gpu(P, nparts):
    """The partitioned device path (ghost rows, face ranges, owned-only
    element kernel) emulated on one GPU: partitions run one after the other
    with the halo filled by copies -- no kernels wait on each other.  The
    owned residual rows equal the single-partition residual bitwise."""
    import torch

    from paper_2209_01877_b200.dg import Discretization, _get_disc
    from paper_2209_01877_b200.geometry import compute_geometry
    from paper_2209_01877_b200.partition import build_local, rcb_partition

    m = P.perturb_interior_nodes(P.generate_tet_box(5, bc=gpu_helpers.MIXED_BC), 0.1, 4)
    order = 2
    gas, geo, bcs = gpu_setup(P, m, order)
    disc_g, c = oracle_state(m, order)
    full = _get_disc(m, geo, gas, bcs)
    rows_g = full.to_reference(torch.from_numpy(c).cuda())
    ref = full.residual_rows(rows_g, full.face_flux(rows_g, 64), 64)
    parts = rcb_partition(m.cell_centroid, nparts)
    for r in range(nparts):
        part = build_local(m, parts, r)
        d = Discretization(part.mesh, compute_geometry(part.mesh, order, split=part.n_inner_faces), gas, bcs,
                           n_elems=part.n_owned)
        gl = torch.as_tensor(np.concatenate([part.owned, part.ghosts]), device="cuda")
        rows = rows_g.index_select(0, gl).contiguous()  # owned + ghost rows (the halo)
        own = torch.as_tensor(part.owned, device="cuda")
        for hb in (d.face_buffer(64), d.elem_buffer(64)):  # both record layouts
            d.reset_errors()
            d.face_flux(rows, 64, hb, f_begin=0, f_end=part.n_inner_faces)
            d.face_flux(rows, 64, hb, f_begin=part.n_inner_faces, f_end=d.nf)
            res = d.residual_rows(rows, hb, 64, res=d.new_state())
            d.raise_errors()
            assert torch.equal(res[: part.n_owned], ref.index_select(0, own)), (r, hb.dim())


@pytest.mark.parametrize("order", [0, 1, 2, 3])
@pytest.mark.parametrize("prec", [64, 32])
def test_element_slot_layout_bitwise(P, order, prec):
    """The stepper's element-slot record path (hodg_face_flux_range_es +
    hodg_elem_stage_es) gives the same residual bits as the face-ordered
    path: same values, same summation order, different placement."""
    import torch

    from paper_2209_01877_b200.dg import _get_disc

    for name, m in meshes():
        disc_o, c = oracle_state(m, order)
        gas, geo, bcs = gpu_setup(P, m, order)
        d = _get_disc(m, geo, gas, bcs)
        rows = d.to_reference(torch.from_numpy(c).cuda())
        p = P._lib.PREC_F64 if prec == 64 else P._lib.PREC_MIXED
        d.reset_errors()
        ref = d.residual_rows(rows, d.face_flux(rows, p, d.face_buffer(p)), p)
        eb = d.elem_buffer(p)
        eb.fill_(float("nan"))  # every slot must be written
        got = d.residual_rows(rows, d.face_flux(rows, p, eb), p)
        d.raise_errors()
        assert torch.equal(got, ref), (name, order, prec)


@pytest.mark.parametrize("order", [1, 2, 3])
@pytest.mark.parametrize("prec", [64, 32])
def test_stepper_layouts_identical_trajectories(P, order, prec):
    """Fused SSP-RK3 steps (CUDA graphs) with the face-ordered and the
    element-slot record layouts give bit-identical states and dt."""
    import torch

    from paper_2209_01877_b200.dg import _get_disc
    from paper_2209_01877_b200.timestepping import Stepper

    name, m = meshes()[-1]
    disc_o, c = oracle_state(m, order)
    gas, geo, bcs = gpu_setup(P, m, order)
    d = _get_disc(m, geo, gas, bcs)
    p = P._lib.PREC_F64 if prec == 64 else P._lib.PREC_MIXED
    out = []
    for layout in ("face", "elem"):
        st = Stepper(d, "rk3", p, "global", 0.3, log_norms=True, use_graph=True, layout=layout)
        st.load(P.DofState(torch.from_numpy(c).cuda()))
        for _ in range(4):
            st.step()
        st.check()
        out.append((st.state().coeffs.clone(), st.dt_value(), st.norms.clone()))
    assert torch.equal(out[0][0], out[1][0]), (order, prec)
    assert out[0][1] == out[1][1]
    assert torch.equal(out[0][2], out[1][2])


_C_BC = {"xmin": "far_field", "xmax": "far_field", "ymin": "far_field", "ymax": "far_field",
         "zmin": "slip_wall", "zmax": "slip_wall"}


def test_config0_against_fixture(P):
    """BASELINE config 0 on the GPU against the committed oracle fixture
    (tests/golden/config0_*, tools/make_golden_3d.py): residual history per
    entry and final state within 1e-12."""
    from conftest import golden_path

    m = P.perturb_interior_nodes(P.generate_tet_box(4, extent=(0.0, 0.0, 0.0, 10.0, 10.0, 2.5), bc=_C_BC), 0.1, 3)
    cfg = P.RunConfig(order=1, mach=0.5, initial_kind="vortex", initial_x0=5.0, initial_y0=5.0, cfl=0.3,
                      dt_mode="global", scheme="rk3", max_iterations=10, log_every=1)
    art = P.run(cfg, mesh=m)
    rows = [r.split(",") for r in open(golden_path("config0_residuals.csv")).read().strip().splitlines()[1:]]
    ref = np.array([[float(x) for x in r[1:7]] for r in rows])
    got = np.column_stack([np.array(art.history.res), np.array(art.history.dts)])
    assert np.max(np.abs(got - ref) / np.abs(ref)) <= FP64_TOL
    u = np.load(golden_path("config0_state.npz"))["coeffs"]
    assert rel(art.final_state.coeffs.cpu().numpy(), u) <= FP64_TOL


@pytest.mark.parametrize("prec", [64, 32])
def test_c200k_against_oracle(P, prec):
    """BASELINE config 1 at its full size (C200k: Kuhn cube n = 32, 196,608
    tets, P2): freestream preserved to 1e-11, and three SSP-RK3 steps of the
    vortex agree with the oracle (16 host threads) -- FP64 1e-12, mixed 1e-5
    on the state."""
    import torch

    m = P.generate_tet_box(32, extent=(0.0, 0.0, 0.0, 10.0, 10.0, 10.0), bc=_C_BC, device="cuda")
    assert m.n_cells == 196608
    gas = P.GasModel()
    geo = P.compute_geometry(m, 2)
    bcs = P.BoundaryConditions(P.freestream_conserved(gas, 0.5, 0.0))
    fs = P.project_initial(m, geo, lambda x, y, z: P.freestream_primitive(gas, 0.5, 0.0), gas)
    if prec == 64:
        r = P.rhs(fs, m, geo, bcs, gas).res
        assert float(r.abs().max()) < 1e-11
    om = to_oracle(m)
    spec = S.RunSpec(mesh=om, order=2, mach=0.5, initial="vortex", x0=5.0, y0=5.0, cfl=0.3, dt_mode="global",
                     scheme="rk3", max_iterations=3, log_every=1, precision_mode="dp")
    u_ref, hist, _ = S.run(spec)
    cfg = P.RunConfig(order=2, mach=0.5, initial_kind="vortex", initial_x0=5.0, initial_y0=5.0, cfl=0.3,
                      dt_mode="global", scheme="rk3", max_iterations=3, log_every=1,
                      precision_mode="dp" if prec == 64 else "sp")
    art = P.run(cfg, mesh=m)
    got = art.final_state.coeffs.double().cpu().numpy()
    tol = FP64_TOL if prec == 64 else MIXED_TOL
    assert rel(got, u_ref) <= tol, rel(got, u_ref)
    if prec == 64:
        assert rel(np.array(art.history.res), np.array(hist.res)) <= tol


def test_wing_against_oracle(P):
    """BASELINE config 4's wedge-wing geometry (generate_wing_box; slip walls
    on the wing and the symmetry plane): watertight, and two SSP-RK3 steps of
    the incident freestream (P1, FP64) match the oracle to 1e-12."""
    m = P.generate_wing_box(12, thickness=0.3, device="cuda")
    bnd = m.face_cells[:, 1] < 0
    closure = (m.face_normal[bnd] * m.face_length[bnd][:, None]).sum(axis=0)
    assert np.abs(closure).max() < 1e-13
    assert {p.name: p.kind for p in m.patches} == {"far": "far_field", "symmetry": "slip_wall",
                                                    "wing": "slip_wall"}
    assert m.patches[2].face_ids.size > 0
    cfg = P.RunConfig(order=1, mach=0.5, angle_deg=3.0, initial_kind="freestream", cfl=0.3, dt_mode="global",
                      scheme="rk3", max_iterations=2, log_every=1)
    art = P.run(cfg, mesh=m)
    spec = S.RunSpec(mesh=to_oracle(m), order=1, mach=0.5, angle_deg=3.0, initial="freestream", cfl=0.3,
                     dt_mode="global", scheme="rk3", max_iterations=2, log_every=1)
    u, hist, _ = S.run(spec)
    assert rel(art.final_state.coeffs.cpu().numpy(), u) <= FP64_TOL
    assert rel(np.array(art.history.res), np.array(hist.res)) <= FP64_TOL


@pytest.mark.parametrize("order", [1, 2, 3])
def test_mixed_fp32_shadow_bitwise(P, order):
    """The mixed-precision stepper's FP32 state shadow (element kernel writes
    it, face kernel reads it) rounds each coefficient once instead of at
    every (face, side): the steps are bitwise those of the FP64-row path."""
    import torch

    from paper_2209_01877_b200 import _lib
    from paper_2209_01877_b200.dg import _get_disc
    from paper_2209_01877_b200.timestepping import Stepper

    m = P.perturb_interior_nodes(P.generate_tet_box(4, bc=gpu_helpers.MIXED_BC), 0.1, 3)
    gas, geo, bcs = gpu_setup(P, m, order)
    _, c = oracle_state(m, order)
    out = []
    for shadow in (True, False):
        st = Stepper(_get_disc(m, geo, gas, bcs), "rk3", _lib.PREC_MIXED, "global", 0.3, shadow=shadow)
        st.load(P.DofState(torch.from_numpy(c).cuda()))
        for _ in range(3):
            st.step()
        st.check(3)
        out.append((st.A.clone(), st.norms.clone(), st.dt_value()))
        assert (st.A32 is not None) == shadow
    assert torch.equal(out[0][0], out[1][0]) and torch.equal(out[0][1], out[1][1]) and out[0][2] == out[1][2]
