"""The reference's own fixture runs on the GPU (2D table-driven path,
csrc/hodg_2d.cu): 150 RK2 steps of the 16x16 quad vortex case
(pkg/tests/test_fixtures.py:43-58) against the reference's golden residual
histories.  FP64 within 1e-12 relative per entry (typically identical: the
kernels keep the reference's expression trees, -fmad=false; only CUDA's
pow can differ from glibc's by an ulp); mixed precision within 1e-5."""

import numpy as np
import pytest

from conftest import golden_path

pytestmark = pytest.mark.gpu


def read_csv(text):
    rows = [r.split(",") for r in text.strip().splitlines()[1:]]
    return np.array([[float(x) for x in r[1:6]] for r in rows]), [int(r[6]) for r in rows]


@pytest.mark.parametrize("name,mode,kw,tol", [
    ("residuals_dp.csv", "dp", {}, 1e-12),
    ("residuals_mp.csv", "mp_fixed", {"switch_iter": 60}, 1e-5),
])
def test_fixture_history_on_gpu(name, mode, kw, tol):
    from paper_2209_01877_b200 import twod

    cfg = twod.RunConfig2D(gen_kind="quad", gen_nx=16, gen_ny=16, gen_extent=(0.0, 0.0, 10.0, 10.0),
                           initial_kind="vortex", initial_x0=5.0, initial_y0=5.0, mach=0.5, order=1,
                           max_iterations=150, log_every=1, precision_mode=mode, **kw)
    _, hist, _, _ = twod.run2d(cfg)
    text = twod.residual_csv_text(hist)
    with open(golden_path(name)) as fh:
        ref_text = fh.read()
    got, bits = read_csv(text)
    ref, rbits = read_csv(ref_text)
    assert bits == rbits
    relerr = np.abs(got - ref) / np.abs(ref)
    print(f"{name}: max rel diff {relerr.max():.3e}, identical bytes: {text == ref_text}")
    assert relerr.max() <= tol


def test_2d_residual_matches_reference_corpus():
    """GPU 2D residuals of perturbed vortex states on the reference test
    corpus, orders 0-2, FP64 and FP32 states, vs reference-generated vectors."""
    import torch

    from conftest import corpus_2d
    from paper_2209_01877_b200 import twod

    z = np.load(golden_path("ref_rhs2d.npz"))
    specs = {
        "quad_4x4": lambda: twod.generate_quad_grid(4, 4),
        "quad_stretched": lambda: twod.generate_quad_grid(3, 3, (0.0, 0.0, 2.0, 0.7)),
        "tri_4x3": lambda: twod.generate_tri_grid(4, 3),
        "quad_perturbed": lambda: twod.perturb_interior_nodes(twod.generate_quad_grid(6, 5), 0.15, seed=3),
        "tri_perturbed": lambda: twod.perturb_interior_nodes(twod.generate_tri_grid(5, 4), 0.12, seed=7),
    }
    _, qinf = twod.freestream_2d(1.4, 1.0, 0.4, 10.0)
    worst = 0.0
    for name, mk in specs.items():
        m = mk()
        for order in (0, 1, 2):
            t = twod.compute_geometry_2d(m, order)
            dev = twod.Device2D(m, t, 1.4, qinf)
            c = z[f"{name}_p{order}_coeffs"]
            r = dev.rhs(torch.from_numpy(c).cuda()).cpu().numpy()
            ref = z[f"{name}_p{order}_res"]
            e = np.linalg.norm(r - ref) / np.linalg.norm(ref)
            worst = max(worst, e)
            assert e <= 1e-12, (name, order, e)
            r32 = dev.rhs(torch.from_numpy(c.astype(np.float32)).cuda()).cpu().numpy()
            e32 = np.linalg.norm(r32 - z[f"{name}_p{order}_res32"]) / np.linalg.norm(ref)
            assert e32 <= 1e-5, (name, order, e32)
    print("worst FP64 relative error", worst)
