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
