"""Per-rank compute of the partitioned C1M P2 step, measured on one GPU.

Only one GPU is available to this build, so the strong-scaling run cannot be
timed end to end.  This runs, for P = 1, 2, 4, 8 RCB parts, the exact local
problem of the most loaded rank (owned elements + ghost rows, interior and
partition faces) through the fused stepper on one GPU -- the ghost rows are
filled once and not exchanged -- and reports its step time against t1 / P,
plus the halo bytes per stage that the NCCL exchange moves while the
interior-face kernel runs.

usage: python tools/scaling_estimate.py [--n 55] [--steps 20]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2209_01877_b200 as P
from paper_2209_01877_b200.dg import Discretization, _get_disc
from paper_2209_01877_b200.geometry import compute_geometry
from paper_2209_01877_b200.partition import build_local, rcb_partition
from paper_2209_01877_b200.timestepping import Stepper


def time_steps(st, steps):
    for _ in range(3):
        st.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        st.step()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=55)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--order", type=int, default=2)
    args = ap.parse_args()
    bc = {"xmin": "far_field", "xmax": "far_field", "ymin": "far_field", "ymax": "far_field",
          "zmin": "slip_wall", "zmax": "slip_wall"}
    mesh = P.generate_tet_box(args.n, extent=(0.0, 0.0, 0.0, 10.0, 10.0, 10.0), bc=bc, device="cuda")
    gas = P.GasModel()
    bcs = P.BoundaryConditions(P.freestream_conserved(gas, 0.5, 0.0))
    geo = P.compute_geometry(mesh, args.order)
    st0 = P.project_initial(mesh, geo, lambda x, y, z: P.vortex_primitive(gas, 0.5, 0.0, 5.0, 5.0, 5.0, 0.0, x, y),
                            gas)
    full = _get_disc(mesh, geo, gas, bcs)
    rows_g = full.to_reference(st0.coeffs)
    stepper = Stepper(full, "rk3", 64, "global", 0.3, use_graph=True)
    stepper.load(st0)
    t1 = time_steps(stepper, args.steps)
    out = [{"parts": 1, "owned": mesh.n_cells, "faces": mesh.n_faces, "step_ms": t1, "ideal_ms": t1,
            "compute_efficiency": 1.0, "halo_rows": 0, "halo_mb_per_stage": 0.0}]
    rs = full.rs
    for nparts in (2, 4, 8):
        parts = rcb_partition(mesh.cell_centroid, nparts)
        counts = np.bincount(parts, minlength=nparts)
        r = int(np.argmax(counts))  # the most loaded rank
        part = build_local(mesh, parts, r)
        lgeo = compute_geometry(part.mesh, args.order, split=part.n_inner_faces)
        d = Discretization(part.mesh, lgeo, gas, bcs, n_elems=part.n_owned)
        st = Stepper(d, "rk3", 64, "global", 0.3, use_graph=True)
        # the DistributedStepper's schedule: boundary + partition faces after
        # the interior ones (they wait for the halo), not on a side stream
        st._side = None
        gl = torch.as_tensor(np.concatenate([part.owned, part.ghosts]), device="cuda")
        st.A.copy_(rows_g.index_select(0, gl))
        st.init_dt()
        tp = time_steps(st, args.steps)
        sent = sum(len(v) for v in part.send_idx.values())
        out.append({"parts": nparts, "rank": r, "owned": int(part.n_owned), "ghosts": int(part.ghosts.size),
                    "faces": int(part.n_faces), "partition_faces": int(part.n_faces - part.n_inner_faces),
                    "step_ms": tp, "ideal_ms": t1 / nparts, "compute_efficiency": (t1 / nparts) / tp,
                    "halo_rows": int(part.ghosts.size + sent),
                    "halo_mb_per_stage": (part.ghosts.size + sent) * rs * 8 / 1e6})
    for row in out:
        print(json.dumps(row))
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/scaling_estimate_n{args.n}_p{args.order}.json", "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
