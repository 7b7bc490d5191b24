"""Per-rank step time of the partitioned C1M P2 run, measured on one GPU
through the shipped distributed schedule.

Only one GPU is available to this build, so the strong-scaling run cannot be
timed end to end.  For P = 1, 2, 4, 8 RCB parts this takes the local problem
of the most loaded rank (owned elements + ghost rows, interior and partition
faces) and steps it with DistributedStepper exactly as bench.py --gpus P
does -- per stage the NCCL halo exchange (pack kernel + grouped send / recv
on the communication stream) posted before the interior-face kernel, the
wait, the boundary + partition faces, the owned-element kernel; per step the
dt MIN and norm SUM all-reduces -- over a 1-rank NCCL communicator whose rank
is its own peer (tests/test_gpu_halo.py).  The halo therefore moves the
rank's real ghost-row byte count, but as one device-local message instead
of NVLink transfers to 3-7 peers; the NVLink time is added separately from
the measured 770 GB/s peer bandwidth (B200_PROFILING.md) and is hidden
behind the interior faces whenever it is shorter.

Reported per P: the eager schedule (the default, host-launched),
optionally the same step captured in a CUDA graph (--capture), the
compute-only graph-captured local step (no exchange), and the halo bytes per
stage for ghost rows vs face traces (the alternative exchange north_star
names).

usage: python tools/scaling_estimate.py [--n 55] [--order 2] [--steps 20] [--capture]
"""
import argparse
import json
import os
import sys
import types

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2209_01877_b200 as P  # noqa: E402
from paper_2209_01877_b200 import _lib  # noqa: E402
from paper_2209_01877_b200.dg import Discretization, _get_disc  # noqa: E402
from paper_2209_01877_b200.distributed import DistributedStepper  # noqa: E402
from paper_2209_01877_b200.geometry import compute_geometry  # noqa: E402
from paper_2209_01877_b200.partition import build_local, rcb_partition  # noqa: E402
from paper_2209_01877_b200.timestepping import Stepper  # noqa: E402

NVLINK_GBS = 770.0  # measured peer copy bandwidth per direction (B200_PROFILING.md)


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


def self_plan(part):
    """The rank's halo as one self-message of its real ghost-row count."""
    sends = np.concatenate([np.asarray(part.send_idx[q], dtype=np.int64) for q in sorted(part.send_idx)])
    ng = int(part.ghosts.size)
    rows = np.resize(sends, ng).astype(np.int32)
    return types.SimpleNamespace(send_idx={0: rows}, recv_range={0: (int(part.n_owned), ng)},
                                 nparts=1, owned=part.owned)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=55)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--order", type=int, default=2)
    ap.add_argument("--capture", action="store_true", help="also time the graph-captured distributed step")
    ap.add_argument("--parts", default="2,4,8")
    args = ap.parse_args()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
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
    stepper = Stepper(full, "rk3", _lib.PREC_F64, "global", 0.3, use_graph=True)
    stepper.load(st0)
    t1 = time_steps(stepper, args.steps)
    print(f"P=1 {t1:.3f} ms", flush=True)
    nqf, rs = full.nqf, full.rs
    out = [{"parts": 1, "owned": mesh.n_cells, "faces": mesh.n_faces, "step_ms": t1, "ideal_ms": t1,
            "efficiency": 1.0}]
    for nparts in [int(x) for x in args.parts.split(",")]:
        parts = rcb_partition(mesh.cell_centroid, nparts)
        counts = np.bincount(parts, minlength=nparts)
        r = int(np.argmax(counts))  # the most loaded rank
        part = build_local(mesh, parts, r)
        lgeo = compute_geometry(part.mesh, args.order, split=part.n_inner_faces)
        d = Discretization(part.mesh, lgeo, gas, bcs, n_elems=part.n_owned)
        gl = torch.as_tensor(np.concatenate([part.owned, part.ghosts]), device="cuda")
        local_rows = rows_g.index_select(0, gl)
        row = {"parts": nparts, "rank": r, "owned": int(part.n_owned), "ghosts": int(part.ghosts.size),
               "faces": int(part.n_faces), "partition_faces": int(part.n_faces - part.n_inner_faces),
               "ideal_ms": t1 / nparts}
        # compute only: the local step in a CUDA graph, ghosts filled once
        st = Stepper(d, "rk3", _lib.PREC_F64, "global", 0.3, use_graph=True)
        st._side = None
        st.A.copy_(local_rows)
        st.init_dt()
        row["compute_only_ms"] = time_steps(st, args.steps)
        print(f"P={nparts} compute-only {row['compute_only_ms']:.3f} ms", flush=True)
        del st
        # the shipped schedule: DistributedStepper with the native NCCL halo
        for mode in (["eager", "graph"] if args.capture else ["eager"]):
            ds = DistributedStepper(self_plan(part), d, "rk3", _lib.PREC_F64, 0.3, log_norms=True,
                                    halo="native", use_graph=(mode == "graph"))
            ds.A.copy_(local_rows)
            ds.init_dt()
            print(f"P={nparts} {mode}: stepping", flush=True)
            row[f"{mode}_ms"] = time_steps(ds, args.steps)
            print(f"P={nparts} {mode} {row[f'{mode}_ms']:.3f} ms", flush=True)
            ds.close()
            del ds
        # halo bytes per stage and direction: ghost rows (shipped) vs face traces
        ghost_b = part.ghosts.size * rs * 8
        trace_b = (part.n_faces - part.n_inner_faces) * nqf * 5 * 8
        row["halo_mb_per_stage"] = {"ghost_rows": ghost_b / 1e6, "face_traces": trace_b / 1e6}
        row["nvlink_us_per_stage"] = ghost_b / (NVLINK_GBS * 1e3)
        best = min(row[k] for k in ("eager_ms", "graph_ms") if k in row)
        row["efficiency"] = (t1 / nparts) / best
        out.append(row)
    for row in out:
        print(json.dumps(row))
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/scaling_estimate_n{args.n}_p{args.order}.json", "w") as fh:
        json.dump(out, fh, indent=1)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
