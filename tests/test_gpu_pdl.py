"""Programmatic dependent launch (HODG_PDL, csrc/hodg_kernels.cuh) changes
only when a kernel's prologue runs, never what it computes: a CUDA-graph
stepper run with the face and element kernels launched as programmatic
dependents equals the same run with ordinary launches bit for bit (FP64 and
mixed precision, both record layouts).  The launch mode is fixed when the
library loads, so each mode runs in its own process."""

import hashlib
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import hashlib, sys
sys.path.insert(0, sys.argv[1])
import torch
import paper_2209_01877_b200 as P
from paper_2209_01877_b200.dg import _get_disc
from paper_2209_01877_b200.timestepping import Stepper
m = P.perturb_interior_nodes(P.generate_tet_box(6, 5, 4, bc={"xmin": "far_field", "xmax": "far_field",
    "ymin": "far_field", "ymax": "far_field", "zmin": "slip_wall", "zmax": "slip_wall"}), 0.1, 5)
gas = P.GasModel()
bcs = P.BoundaryConditions(P.freestream_conserved(gas, 0.5, 5.0))
h = hashlib.sha256()
for order, prec, layout in ((2, 64, "face"), (2, 32, "elem"), (3, 64, "elem"), (1, 32, "face")):
    geo = P.compute_geometry(m, order)
    st0 = P.project_initial(m, geo, lambda x, y, z: P.vortex_primitive(gas, 0.5, 5.0, 0.5, 0.5, 0.5, 0.0, x, y), gas)
    st = Stepper(_get_disc(m, geo, gas, bcs), "rk3", prec, "global", 0.3, use_graph=True, layout=layout)
    st.load(st0)
    for _ in range(8):
        st.step()
    torch.cuda.synchronize()
    st.check()
    h.update(st.A.cpu().numpy().tobytes())
    h.update(st.norms.cpu().numpy().tobytes())
print(h.hexdigest())
"""


def _run(pdl_max):
    env = dict(os.environ, HODG_PDL_MAX_ELEMS=str(pdl_max))
    out = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout.strip().splitlines()[-1]


def test_pdl_launches_bitwise_equal_ordinary_launches():
    assert _run(10**9) == _run(0)
