"""paper_2209_01877_b200 -- B200-native DG Euler residual + RK stepping.

The hot path of arXiv 2209.01877's `hodg` solver (explicit modal-DG
residual and Runge-Kutta stage update) rebuilt for tetrahedral meshes on
NVIDIA B200 (sm_100a): hand-written CUDA kernels behind a C ABI
(include/hodg_b200.h, libhodg_b200.so), driven from Python with the
reference's API (DofState, rhs, face_flux_pass, accumulate_rhs, rk2_step,
local_dt_field, min_reduce, run, rcm, apply_permutation, ...).
"""

from .mesh import (BC_KINDS, BoundaryPatch, MeshError, MeshParseError, TetMesh, TopologyError, build_tet_mesh,
                   generate_tet_box, generate_wing_box, load_mesh, perturb_interior_nodes, save_mesh, validate)
from .physics import (AdmissibilityError, Conserved, GasModel, Primitive, freestream_conserved,
                      freestream_primitive, vortex_primitive)
from .geometry import DeviceGeometry, compute_geometry
from .dg import (BoundaryConditions, DofState, FaceFluxBuffer, Residual, accumulate_rhs, cell_means,
                 face_flux_pass, project_initial, rhs)
from .precision import PrecisionController, PrecisionSchedule, demote, promote
from .timestepping import (RunConfig, Stepper, SolverDivergedError, local_dt_field, min_reduce, residual_l2,
                           rk2_step, rk3_step, run)
from .renumber import (AdjacencyGraph, Permutation, apply_permutation, bandwidth, build_adjacency, export_spy,
                       random_permutation, rcm)

__version__ = "0.1.0"
