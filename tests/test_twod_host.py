"""2D host setup of the product (paper_2209_01877_b200.twod) is bitwise the
oracle's (which is pinned to the reference): meshes and geometry tables."""

import numpy as np
import pytest

from oracle import geometry as OG
from oracle import mesh as OM
from paper_2209_01877_b200 import twod


def test_mesh_and_tables_bitwise():
    pairs = [
        (twod.generate_quad_grid(16, 16, (0.0, 0.0, 10.0, 10.0)), OM.quad_grid(16, 16, (0.0, 0.0, 10.0, 10.0))),
        (twod.perturb_interior_nodes(twod.generate_tri_grid(5, 4), 0.12, seed=7),
         OM.perturb_2d(OM.tri_grid(5, 4), 0.12, seed=7)),
    ]
    for a, b in pairs:
        assert np.array_equal(a.node_xy, b.node_xy)
        assert np.array_equal(a.face_cells, b.face_cells)
        assert np.array_equal(a.face_normal, b.face_normal)
        assert np.array_equal(a.cell_area, b.cell_area)
        for order in (0, 1, 2):
            ta, tb = twod.compute_geometry_2d(a, order), OG.tables_2d(b, order)
            assert np.array_equal(ta.vol_basis, tb.vol_basis)
            assert np.array_equal(ta.vol_gx, tb.vol_grad[0]) and np.array_equal(ta.vol_gy, tb.vol_grad[1])
            assert np.array_equal(ta.minv, tb.minv)
            assert np.array_equal(ta.fbl, tb.face_basis_l) and np.array_equal(ta.fbr, tb.face_basis_r)


def test_mu_from_reynolds_and_pulse_field():
    """hodg/config.py:102-111 and hodg/flows.py:60-73 (pkg/tests/test_config.py:56-66)."""
    from paper_2209_01877_b200 import twod

    cfg = twod.RunConfig2D(gen_nx=2, gen_ny=2, ivis=1, mach=0.3, reynolds=5000.0)
    assert cfg.mu() == pytest.approx(0.3 * 1.4 ** 0.5 / 5000.0)
    assert twod.RunConfig2D(ivis=1, mach=0.3, reynolds=5000.0, mu_dyn=0.01).mu() == 0.01
    assert twod.RunConfig2D(ivis=0, reynolds=5000.0).mu() == 0.0
    x = np.linspace(-1, 1, 7)
    rho, u, v, p = twod.pulse_2d(1.4, 1.0, 0.2, 0.3, 0.0, 0.0, x, 0 * x, 0.4, 10.0)
    from oracle import solver as S
    ref = S.pulse_primitive(S.Gas(), 0.2, 0.3, 0.0, 0.0, x, 0 * x, 0.4, 10.0)
    for a, b in zip((rho, u, v, p), ref):
        assert np.array_equal(a, b)


def test_hodg_mesh_v1_roundtrip_with_reference_files(tmp_path):
    """load_mesh_2d reads the reference's own save_mesh output
    (tests/golden/mesh_*.hodg) into the same mesh the generators build, and
    save_mesh_2d writes it back byte for byte (hodg/mesh.py:431-560)."""
    from conftest import golden_path
    from paper_2209_01877_b200.mesh import MeshParseError

    gens = {"quad_perturbed": lambda: twod.perturb_interior_nodes(twod.generate_quad_grid(6, 5), 0.15, seed=3),
            "tri_perturbed": lambda: twod.perturb_interior_nodes(twod.generate_tri_grid(5, 4), 0.12, seed=7)}
    for name, gen in gens.items():
        path = golden_path(f"mesh_{name}.hodg")
        m = twod.load_mesh_2d(path)
        g = gen()
        for f in ("node_xy", "cell_nodes", "cell_faces", "cell_fsign", "face_nodes", "face_cells", "face_normal",
                  "face_length", "face_patch"):
            assert np.array_equal(getattr(m, f), getattr(g, f)), (name, f)
        out = tmp_path / f"{name}.hodg"
        twod.save_mesh_2d(m, out)
        assert out.read_bytes() == open(path, "rb").read()
    bad = tmp_path / "bad.hodg"
    bad.write_text("hodg-mesh 1\nnodes 2\n0 0\n1 x\n")
    with pytest.raises(MeshParseError) as e:
        twod.load_mesh_2d(bad)
    assert e.value.line_no == 4


def test_vtk_field_matches_reference_file(tmp_path):
    """write_vtk_2d writes the reference's legacy-VTK cell-mean field byte
    for byte (hodg/output.py:54-83; tests/golden/field_tri_perturbed_p2.vtk
    from tools/make_golden.py)."""
    from conftest import golden_path

    m = twod.perturb_interior_nodes(twod.generate_tri_grid(5, 4), 0.12, seed=7)
    t = twod.compute_geometry_2d(m, 2)
    c = np.load(golden_path("ref_rhs2d.npz"))["tri_perturbed_p2_coeffs"]
    out = tmp_path / "f.vtk"
    twod.write_vtk_2d(out, m, t, c, 1.4)
    assert out.read_bytes() == open(golden_path("field_tri_perturbed_p2.vtk"), "rb").read()
