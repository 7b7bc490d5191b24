"""tests/golden/config0_*: BASELINE.json config 0 ("small tetrahedral box
mesh, 3D Euler P1 DG, uniform freestream + isentropic vortex, FP64, 10 RK3
steps on CPU (oracle)") -- the oracle's residual history (CSV, the
reference's format with the w-momentum column) and final state.  The
reference has no tetrahedral path, so these are oracle outputs; the oracle
itself is pinned to the reference's 2D fixtures (tests/test_oracle_golden.py).

Usage:  python tools/make_golden_3d.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import mesh as OM  # noqa: E402
from oracle import solver as S  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
BC = {"xmin": "far_field", "xmax": "far_field", "ymin": "far_field", "ymax": "far_field",
      "zmin": "slip_wall", "zmax": "slip_wall"}


def config0_mesh():
    return OM.perturb_3d(OM.kuhn_box(4, (0.0, 0.0, 0.0, 10.0, 10.0, 2.5), bc=BC), 0.1, 3)


def config0_spec(mesh):
    return S.RunSpec(mesh=mesh, order=1, mach=0.5, initial="vortex", x0=5.0, y0=5.0, cfl=0.3, dt_mode="global",
                     scheme="rk3", max_iterations=10, log_every=1)


def main():
    u, hist, _ = S.run(config0_spec(config0_mesh()))
    with open(os.path.join(OUT, "config0_residuals.csv"), "w") as fh:
        fh.write(S.residual_csv_text(hist, nvar=5))
    np.savez_compressed(os.path.join(OUT, "config0_state.npz"), coeffs=u)
    print("wrote config0 fixtures")


if __name__ == "__main__":
    main()
