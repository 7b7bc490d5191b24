"""Device mesh setup (csrc/setup.cu) against the
host builder: integer connectivity bit-identical, geometry equal (h to the
libm-vs-CUDA cbrt ulp), on boxes, perturbed and shuffled meshes; errors on
non-manifold input."""

import time

import numpy as np
import pytest

from paper_2209_01877_b200 import mesh as M

pytestmark = pytest.mark.gpu

INT_FIELDS = ("cell_nodes", "cell_faces", "cell_fsign", "cell_neighbors", "face_nodes", "face_cells", "face_slots",
              "face_patch")
FLOAT_FIELDS = ("cell_centroid", "cell_area", "face_normal", "face_length")


def _same(a, b):
    for f in INT_FIELDS:
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    for f in FLOAT_FIELDS:
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert np.allclose(a.cell_h, b.cell_h, rtol=4e-16, atol=0.0)
    assert [(p.name, p.kind) for p in a.patches] == [(p.name, p.kind) for p in b.patches]
    for p, q in zip(a.patches, b.patches):
        assert np.array_equal(p.face_ids, q.face_ids)


@pytest.mark.parametrize("dims", [(1, 1, 1), (3, 2, 4), (6, 6, 6)])
def test_device_build_equals_host(dims):
    host = M.generate_tet_box(*dims, bc={"xmin": "far_field", "xmax": "far_field", "ymin": "slip_wall",
                                         "ymax": "slip_wall", "zmin": "no_slip_wall", "zmax": "far_field"})
    dev = M.generate_tet_box(*dims, bc={"xmin": "far_field", "xmax": "far_field", "ymin": "slip_wall",
                                        "ymax": "slip_wall", "zmin": "no_slip_wall", "zmax": "far_field"},
                             device="cuda")
    _same(host, dev)


def test_device_build_perturbed_and_shuffled():
    base = M.perturb_interior_nodes(M.generate_tet_box(5, 4, 3), 0.15, seed=9)
    nodes, elems, specs = base.raw()
    rng = np.random.default_rng(4)
    elems = elems[rng.permutation(elems.shape[0])]
    elems = np.take_along_axis(elems, rng.permuted(np.tile(np.arange(4), (elems.shape[0], 1)), axis=1), axis=1)
    _same(M.build_tet_mesh(nodes, elems, specs), M.build_tet_mesh(nodes, elems, specs, device="cuda"))


def test_device_build_rejects_non_manifold():
    nodes = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [0, 0, -1], [1, 1, 1]], dtype=float)
    tets = [[0, 1, 2, 3], [0, 1, 2, 4], [0, 1, 2, 5]]  # face (0,1,2) shared three times
    with pytest.raises(M.TopologyError):
        M.build_tet_mesh(nodes, tets, device="cuda")


def test_device_setup_c1m_time():
    """C1M (998,250 tets): host build vs device build wall time."""
    import torch

    torch.cuda.synchronize()
    M.generate_tet_box(8, device="cuda")  # warm
    t0 = time.perf_counter()
    host = M.generate_tet_box(55)
    t1 = time.perf_counter()
    dev = M.generate_tet_box(55, device="cuda")
    t2 = time.perf_counter()
    print(f"C1M build: host {t1 - t0:.2f} s, device {t2 - t1:.2f} s ({host.n_cells} tets, {host.n_faces} faces)")
    assert dev.n_faces == host.n_faces == 2014650
    assert np.array_equal(dev.cell_faces, host.cell_faces)


@pytest.mark.parametrize("order", [1, 2, 3])
def test_device_element_records_equal_host(order):
    """hodg_element_records vs compute_geometry's numpy/LAPACK build: fc, h,
    vol and J/h bit-identical, J^-1 (adjugate vs LU) to a few ulp; face
    layout identical; an FP64 residual through either geometry agrees."""
    import torch

    import paper_2209_01877_b200 as P

    m = M.perturb_interior_nodes(M.generate_tet_box(5, 4, 3, bc={"xmin": "far_field", "xmax": "far_field",
                                                                 "ymin": "slip_wall", "ymax": "slip_wall",
                                                                 "zmin": "no_slip_wall", "zmax": "far_field"}),
                                 0.15, seed=3)
    host = P.compute_geometry(m, order)
    dev = P.compute_geometry(m, order, device="cuda")
    assert dev.egeo is None and dev.econv is None
    for k in ("efaces", "fcells", "finfo", "fnrm", "face_perm", "face_inv"):
        assert np.array_equal(getattr(host, k), getattr(dev, k)), k
    assert (host.n_int0, host.n_bnd) == (dev.n_int0, dev.n_bnd)
    d = dev.device("cuda")
    from paper_2209_01877_b200.geometry import TILE

    T = TILE[order]
    eg = d["egeo"].cpu().numpy().reshape(-1, 16, T)
    hg = host.egeo.reshape(-1, 16, T)
    assert np.array_equal(eg[:, 9:, :], hg[:, 9:, :])
    scale = np.abs(hg[:, :9, :]).max(axis=1, keepdims=True)  # per element (0 on padding lanes)
    assert np.all(np.abs(eg[:, :9, :] - hg[:, :9, :]) <= 1e-14 * scale)
    ec = d["econv"].cpu().numpy()
    assert np.array_equal(ec[:, :9], host.econv[:, :9])
    assert np.allclose(ec[:, 9:], host.econv[:, 9:], rtol=0, atol=1e-14 * np.abs(host.econv[:, 9:]).max())
    assert dev.constant_count() == host.constant_count()
    gas = P.GasModel()
    bcs = P.BoundaryConditions(P.freestream_conserved(gas, 0.4, 10.0))
    rng = np.random.default_rng(order)
    st = P.project_initial(m, host, lambda x, y, z: P.vortex_primitive(gas, 0.4, 10.0, 0.5, 0.5, 0.5, 0.0, x, y), gas)
    c = st.coeffs.cpu().numpy() * (1.0 + 0.01 * rng.standard_normal(st.coeffs.shape))
    r_h = P.rhs(P.DofState(torch.from_numpy(c).cuda()), m, host, bcs, gas).res.cpu().numpy()
    r_d = P.rhs(P.DofState(torch.from_numpy(c).cuda()), m, dev, bcs, gas).res.cpu().numpy()
    assert np.linalg.norm(r_d - r_h) <= 1e-13 * np.linalg.norm(r_h)


def test_device_element_records_reject_degenerate():
    import paper_2209_01877_b200 as P
    from paper_2209_01877_b200.geometry import GeometryError

    m = M.generate_tet_box(2, 2, 2)
    m.node_xy[:, 2] = 0.0  # flatten every element
    with pytest.raises(GeometryError):
        P.compute_geometry(m, 1, device="cuda")
