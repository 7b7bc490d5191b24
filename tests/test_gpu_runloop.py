"""The 3D run loop's step control and precision switch against the oracle
(reference hodg/timestepping.py:305-357, hodg/precision.py:81-93):
dt_fixed, dt_floor, the t_final clip with its 1e-14 slack, output_every
field files, and an mp_rebound promotion on the device path."""

import os

import numpy as np
import pytest

from gpu_helpers import rel, to_oracle
from oracle import solver as S

pytestmark = pytest.mark.gpu

FP64_TOL = 1e-12
MIXED_TOL = 1e-5
BOX_BC = {"xmin": "far_field", "xmax": "far_field", "ymin": "far_field", "ymax": "far_field",
          "zmin": "slip_wall", "zmax": "slip_wall"}


@pytest.fixture(scope="module")
def P():
    import paper_2209_01877_b200 as P

    P._lib.lib()
    return P


def _mesh(P):
    return P.perturb_interior_nodes(P.generate_tet_box(4, extent=(0.0, 0.0, 0.0, 10.0, 10.0, 2.5), bc=BOX_BC),
                                    0.1, 3)


def _pair(P, m, order=1, **kw):
    """The same run on the device and in the oracle."""
    common = dict(order=order, mach=0.5, cfl=0.3, scheme="rk3", log_every=1)
    cfg = P.RunConfig(initial_kind="vortex", initial_x0=5.0, initial_y0=5.0, **common, **kw)
    art = P.run(cfg, mesh=m)
    okw = {k: v for k, v in kw.items() if k not in ("output_prefix", "output_every")}
    spec = S.RunSpec(mesh=to_oracle(m), initial="vortex", x0=5.0, y0=5.0, **common, **okw)
    u, hist, _ = S.run(spec)
    return art, u, hist


def test_dt_fixed(P):
    m = _mesh(P)
    art, u, hist = _pair(P, m, dt_mode="global", dt_fixed=0.01, max_iterations=6)
    assert art.history.dts == [0.01] * 6 == hist.dts
    assert rel(art.final_state.coeffs.cpu().numpy(), u) <= FP64_TOL
    assert rel(np.array(art.history.res), np.array(hist.res)) <= FP64_TOL


def test_t_final_clip(P):
    """The last step is clipped to land on t_final; the loop stops there
    even though max_iterations allows more."""
    m = _mesh(P)
    art, u, hist = _pair(P, m, dt_mode="global", t_final=0.3, max_iterations=50)
    assert art.iterations_run == len(hist.iterations) < 50
    assert abs(art.t_sim - 0.3) <= 1e-14 and abs(hist.t_sim - 0.3) <= 1e-14
    np.testing.assert_allclose(art.history.dts, hist.dts, rtol=1e-12)
    assert art.history.dts[-1] < art.history.dts[0]  # the clipped step
    assert rel(art.final_state.coeffs.cpu().numpy(), u) <= FP64_TOL


@pytest.mark.parametrize("dt_mode", ["global", "local"])
def test_dt_floor(P, dt_mode):
    """A floor above the CFL dt of most cells changes every step's dt."""
    m = _mesh(P)
    art0, _, _ = _pair(P, m, dt_mode=dt_mode, max_iterations=1)
    floor = 1.05 * art0.history.dts[0]
    art, u, hist = _pair(P, m, dt_mode=dt_mode, dt_floor=floor, max_iterations=4)
    assert min(art.history.dts) >= floor
    np.testing.assert_allclose(art.history.dts, hist.dts, rtol=1e-12)
    assert rel(art.final_state.coeffs.cpu().numpy(), u) <= FP64_TOL


def test_output_every(P, tmp_path):
    m = _mesh(P)
    prefix = str(tmp_path / "run")
    cfg = P.RunConfig(order=1, mach=0.5, initial_kind="vortex", initial_x0=5.0, initial_y0=5.0, scheme="rk3",
                      dt_mode="global", max_iterations=5, log_every=1, output_prefix=prefix, output_every=2)
    art = P.run(cfg, mesh=m)
    names = sorted(os.path.basename(f) for f in art.output_files)
    assert names == ["run_000002.vtk", "run_000004.vtk", "run_000005.vtk", "run_residuals.csv"]
    from paper_2209_01877_b200.output import read_residual_csv

    it, res, dts, bits = read_residual_csv(prefix + "_residuals.csv")
    assert list(it) == list(range(5)) and np.allclose(res, np.array(art.history.res), rtol=0, atol=0)
    # the last field file holds the final state's cell means
    with open(prefix + "_000005.vtk") as fh:
        text = fh.read()
    assert f"CELL_DATA {m.n_cells}" in text


def test_mp_rebound_promotes_like_oracle(P):
    """mp_rebound on the device: mixed kernels until the density residual
    rebounds by `factor` over its trailing minimum, then FP64.  The vortex
    history bottoms out near step 30 and first exceeds 1.01x its minimum at
    step 34 (next-lower ratio 1.0086), so the promotion is at iteration 35
    in both paths; the history stays within the mixed tolerance of the
    FP64 oracle."""
    m = _mesh(P)
    art, u_mp, hist_mp = _pair(P, m, dt_mode="global", max_iterations=40, precision_mode="mp_rebound",
                               window=200, factor=1.01)
    assert hist_mp.switch == 35
    assert [(e.iteration, e.reason) for e in art.events] == [(35, "rebound")]
    assert art.history.precision == [32] * 35 + [64] * 5 == hist_mp.precision
    spec = S.RunSpec(mesh=to_oracle(m), order=1, mach=0.5, initial="vortex", x0=5.0, y0=5.0, cfl=0.3,
                     dt_mode="global", scheme="rk3", max_iterations=40, log_every=1)
    u64, hist64, _ = S.run(spec)
    assert rel(art.final_state.coeffs.cpu().numpy(), u64) <= MIXED_TOL
    assert rel(np.array(art.history.res), np.array(hist64.res)) <= 10 * MIXED_TOL
