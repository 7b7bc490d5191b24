"""Helpers shared by the GPU parity tests: the same mesh and state fed to
the CUDA path and to the CPU oracle."""

import numpy as np

from oracle import mesh as OM
from oracle import solver as S
from paper_2209_01877_b200 import mesh as M

MIXED_BC = {"xmin": "far_field", "xmax": "far_field", "ymin": "slip_wall", "ymax": "far_field",
            "zmin": "no_slip_wall", "zmax": "slip_wall"}


def meshes():
    return [
        ("box2", M.generate_tet_box(2)),
        ("box3_stretched", M.generate_tet_box(3, extent=(0.0, 0.0, 0.0, 2.0, 0.7, 1.3))),
        ("box4_perturbed", M.perturb_interior_nodes(M.generate_tet_box(4), 0.12, seed=3)),
        ("box3x2x4_mixed_bc", M.perturb_interior_nodes(M.generate_tet_box(3, 2, 4, bc=MIXED_BC), 0.1, seed=5)),
    ]


def to_oracle(m):
    nodes, elems, specs = m.raw()
    return OM.build_tet_mesh(nodes, elems, specs)


def oracle_state(m, order, mach=0.4, angle=10.0, flux_kind=0, seed=11, beta=2.0):
    """(oracle disc, physical-basis coefficients): projected vortex tube
    with a 1% random density perturbation (pkg/tests/test_dg.py:155-160)."""
    om = to_oracle(m)
    disc = S.make_disc(om, order, S.Gas(), mach, angle, flux_kind)
    cx = 0.5 * (m.node_xy[:, 0].min() + m.node_xy[:, 0].max())
    cy = 0.5 * (m.node_xy[:, 1].min() + m.node_xy[:, 1].max())
    c = S.project_initial(om, disc.tab, lambda x, y, z: S.vortex_primitive(
        S.Gas(), mach, angle, beta, cx, cy, 0.0, x, y, dim=3), S.Gas())
    rng = np.random.default_rng(seed + order)
    c[:, :, 0] *= 1.0 + 0.01 * rng.random(c.shape[:2])
    return disc, np.ascontiguousarray(c)


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))
