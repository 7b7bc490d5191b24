"""2D host setup of the product (paper_2209_01877_b200.twod) is bitwise the
oracle's (which is pinned to the reference): meshes and geometry tables."""

import numpy as np

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
