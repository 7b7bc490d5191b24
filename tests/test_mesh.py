"""Tetrahedral mesh builder: agreement with the oracle's independent
builder, invariants (the 3D analogue of pkg/tests/test_mesh.py), I/O."""

import numpy as np
import pytest

from oracle import mesh as OM
from paper_2209_01877_b200 import mesh as M


def to_oracle(m):
    nodes, elems, specs = m.raw()
    return OM.build_tet_mesh(nodes, elems, specs)


@pytest.mark.parametrize("n,kw", [(1, {}), (2, {}), (3, {"ny": 2, "nz": 4}), (5, {})])
def test_box_counts_and_agreement(n, kw):
    m = M.generate_tet_box(n, **kw, bc="slip_wall")
    ny, nz = kw.get("ny", n), kw.get("nz", n)
    N = 6 * n * ny * nz
    B = 4 * (n * ny + ny * nz + n * nz)
    assert m.n_cells == N
    assert int((m.face_cells[:, 1] < 0).sum()) == B
    assert m.n_faces == (4 * N + B) // 2
    assert np.isclose(m.cell_area.sum(), 1.0, rtol=1e-13)
    assert M.validate(m) == []
    o = OM.kuhn_box(n, ny=ny, nz=nz, bc="slip_wall")
    for a, b in [("cell_nodes", "cell_nodes"), ("cell_faces", "cell_faces"), ("cell_fsign", "cell_fsign"),
                 ("cell_neighbors", "cell_neighbors"), ("face_nodes", "face_nodes"), ("face_cells", "face_cells"),
                 ("face_patch", "face_patch")]:
        assert np.array_equal(getattr(m, a), getattr(o, b)), a
    assert np.allclose(m.face_normal, o.face_normal, rtol=0, atol=1e-15)
    assert np.allclose(m.face_length, o.face_length, rtol=1e-15)
    assert np.array_equal(m.node_xy, o.node_xy)


def test_perturbed_agrees_with_oracle():
    m = M.perturb_interior_nodes(M.generate_tet_box(4), 0.12, seed=3)
    o = OM.perturb_3d(OM.kuhn_box(4), 0.12, seed=3)
    assert np.array_equal(m.node_xy, o.node_xy)
    assert np.array_equal(m.face_cells, o.face_cells)
    assert M.validate(m) == []


def test_slots_and_orientation():
    m = M.perturb_interior_nodes(M.generate_tet_box(3), 0.1, seed=1)
    for side in (0, 1):
        ok = m.face_cells[:, side] >= 0
        c = m.face_cells[ok, side]
        s = m.face_slots[ok, side]
        assert np.array_equal(m.cell_faces[c, s], np.flatnonzero(ok))
    # left-to-right normal points away from the left element's centroid
    fc = m.face_cells
    mid = m.node_xy[m.face_nodes].mean(axis=1)
    assert np.all(np.einsum("fd,fd->f", m.face_normal, mid - m.cell_centroid[fc[:, 0]]) > 0)


def test_save_load_roundtrip(tmp_path):
    m = M.perturb_interior_nodes(M.generate_tet_box(2, bc={"xmin": "far_field", "xmax": "far_field",
                                                           "ymin": "slip_wall", "ymax": "slip_wall",
                                                           "zmin": "no_slip_wall", "zmax": "slip_wall"}), 0.1)
    p = tmp_path / "box.mesh"
    M.save_mesh(m, p)
    r = M.load_mesh(p)
    assert np.array_equal(r.node_xy, m.node_xy)
    assert np.array_equal(r.face_cells, m.face_cells)
    assert [(x.name, x.kind) for x in r.patches] == [(x.name, x.kind) for x in m.patches]
    assert np.array_equal(r.boundary_kind_codes(), m.boundary_kind_codes())


def test_parse_error_has_line_number(tmp_path):
    p = tmp_path / "bad.mesh"
    p.write_text("hodg-mesh 1\ndim 3\nnodes 1\n0.0 zero 0.0\n")
    with pytest.raises(M.MeshParseError) as e:
        M.load_mesh(p)
    assert e.value.line_no == 4


def test_rejects_bad_topology():
    X = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 1, 1.0]])
    with pytest.raises(M.TopologyError):
        M.build_tet_mesh(X, [[0, 1, 2, 2]])
    with pytest.raises(M.TopologyError):
        M.build_tet_mesh(np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0], [3, 0, 0.0]]), [[0, 1, 2, 3]])
    # three elements on one face: non-manifold
    X2 = np.vstack([X, [[-1, -1, -1.0]]])
    with pytest.raises(M.TopologyError):
        M.build_tet_mesh(X2, [[0, 1, 2, 3], [0, 1, 2, 4], [0, 1, 2, 5]])
