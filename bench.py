"""Benchmark: DOF-updates/s per RK stage, FP64 P2 Euler, SSP-RK3, on the
synthetic ~1M-tet Kuhn cube (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--n 55] [--order 2] [--prec 64|32] [--no-renumber]

One JSON line on rank 0.  `value` = whole-job DOF-updates/s per stage with
the state resident in HBM (CUDA-event timed, max over ranks);  `e2e` = the
same metric through the public stepping API with the state uploaded from
pinned host memory, the residual norms / error word read back every step
(the reference's per-iteration logging and admissibility check) and the
final state copied back, all inside the timed region.  `--impl reference`
times the CPU oracle (the C restatement of the reference's numba kernels,
OpenMP on all host cores) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NB = {0: 1, 1: 4, 2: 10, 3: 20}
RBAR = 5.0 / 3.0  # mean state reads per SSP-RK3 stage


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=55, help="Kuhn cube size: 6 n^3 tets (55 -> 998,250)")
    ap.add_argument("--order", type=int, default=2)
    ap.add_argument("--prec", type=int, default=64, choices=[64, 32])
    ap.add_argument("--no-renumber", action="store_true")
    ap.add_argument("--case", default="cube", choices=["cube", "wing"],
                    help="cube: the C1M-class Kuhn cube (headline); wing: BASELINE config 4's wedge-wing mesh")
    ap.add_argument("--layout", default="auto", choices=["auto", "elem", "face"], help="face flux record layout")
    ap.add_argument("--partitioned", action="store_true",
                    help="use the partitioned (NCCL halo) stepper even at one rank")
    return ap.parse_args()


def algorithmic_bytes_per_stage(n_elem, n_faces, order):
    """N[(rbar+1) 8 nvar nb + G_e] + F G_f, G_e = 112, G_f = 44."""
    return n_elem * ((RBAR + 1.0) * 8 * 5 * NB[order] + 112) + n_faces * 44


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def build_case(n, order, renumber, device, case="cube"):
    import paper_2209_01877_b200 as P

    if case == "wing":
        # BASELINE config 4: swept wedge wing cut out of the unit cube (slip
        # walls on the wing and the symmetry plane, far field elsewhere),
        # freestream at Mach 0.5 and 3 degrees incidence
        mesh = P.generate_wing_box(n, device=device)
        gas = P.GasModel()
        geo = P.compute_geometry(mesh, order, device=device)
        bcs = P.BoundaryConditions(P.freestream_conserved(gas, 0.5, 3.0))
        state = P.project_initial(mesh, geo, lambda x, y, z: P.freestream_primitive(gas, 0.5, 3.0), gas)
        return P, mesh, gas, geo, bcs, state, None
    mesh = P.generate_tet_box(n, extent=(0.0, 0.0, 0.0, 10.0, 10.0, 10.0),
                              bc={"xmin": "far_field", "xmax": "far_field", "ymin": "far_field",
                                  "ymax": "far_field", "zmin": "slip_wall", "zmax": "slip_wall"},
                              device=device)  # connectivity + geometry on the GPU (bit-identical)
    bw = None
    if renumber:
        # shuffled input (randomize_cells = 1), then device RCM + face re-sort
        mesh = P.apply_permutation(mesh, P.random_permutation(mesh.n_cells, 1))
        g = P.build_adjacency(mesh)
        perm = P.rcm(g)
        bw = (P.bandwidth(g), P.bandwidth(g, perm))
        mesh = P.apply_permutation(mesh, perm, device="cuda")  # face re-sort on the GPU
    gas = P.GasModel()
    geo = P.compute_geometry(mesh, order, device=device)  # element records on the GPU
    bcs = P.BoundaryConditions(P.freestream_conserved(gas, 0.5, 0.0))
    state = P.project_initial(mesh, geo, lambda x, y, z: P.vortex_primitive(gas, 0.5, 0.0, 5.0, 5.0, 5.0, 0.0, x, y),
                              gas)
    return P, mesh, gas, geo, bcs, state, bw


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist_mode = world > 1 or args.partitioned
    if dist_mode:
        os.environ.setdefault("NCCL_DEBUG", "WARN")  # keep stdout to the one JSON line
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        dist.init_process_group("nccl", init_method="env://", rank=rank, world_size=world)
    P, mesh, gas, geo, bcs, state, bw = build_case(args.n, args.order, not args.no_renumber, "cuda", args.case)
    from paper_2209_01877_b200 import _lib
    from paper_2209_01877_b200.dg import _get_disc
    from paper_2209_01877_b200.timestepping import Stepper

    prec = _lib.PREC_F64 if args.prec == 64 else _lib.PREC_MIXED
    if dist_mode:
        # strong scaling: the same mesh partitioned (RCB) over the ranks,
        # NCCL halo exchange per stage overlapped with interior faces
        from paper_2209_01877_b200.distributed import DistributedStepper, owned_state, setup_partitioned

        part, disc = setup_partitioned(mesh, args.order, gas, bcs, rank, world)
        st = DistributedStepper(part, disc, "rk3", prec, 0.3, log_norms=True)
        state_in = owned_state(state, part)
    else:
        disc = _get_disc(mesh, geo, gas, bcs)
        st = Stepper(disc, "rk3", prec, "global", 0.3, log_norms=True, use_graph=True, layout=args.layout)
        state_in = state
    st.load(state_in)
    st.check(0)
    n_st = 3
    dofs = mesh.n_cells * 5 * NB[args.order]

    def barrier():
        if world > 1:
            dist.barrier()

    # warmup (includes graph capture)
    l0 = _lib.launch_count()
    for _ in range(max(args.warmup, 3)):
        st.step()
    kernels_per_step = st.launches_per_step()
    torch.cuda.synchronize()
    st.check()

    # ---- device-resident timed region ----
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        st.step()
    e1.record()
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    st.check(args.steps)
    value = dofs * n_st * args.steps / (ms * 1e-3)  # whole job: the global mesh

    # ---- per-kernel durations (events around each launch, no graph) ----
    hb = st.hbuf
    t_face, t_elem = [], []
    for k in range(3 * n_st):
        stage = k % n_st
        us = st.A if stage == 0 else st.B
        a = st._stage_args(stage, st.parity)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        disc.face_flux(us, prec, hb)
        ev[1].record()
        disc.stage(prec, hb, a)
        ev[2].record()
        torch.cuda.synchronize()
        t_face.append(ev[0].elapsed_time(ev[1]))
        t_elem.append(ev[1].elapsed_time(ev[2]))
        if stage == n_st - 1:
            st.parity = 1 - st.parity
    tf, te = float(np.mean(t_face)), float(np.mean(t_elem))

    # ---- end to end through the public stepping API ----
    host = state_in.coeffs.cpu().pin_memory()
    out_host = torch.empty_like(host).pin_memory()
    norms = torch.empty(5, dtype=torch.float64).pin_memory()
    errh = torch.empty(4, dtype=torch.int32).pin_memory()

    def e2e_pass():
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev_state = P.DofState(host.to("cuda", non_blocking=True))
        st.load(dev_state)
        for _ in range(args.steps):
            # (distributed: every rank reads its norms / error word each step)
            st.step()
            norms.copy_(st.norms, non_blocking=True)
            errh.copy_(disc.err, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            if np.any(errh.numpy().astype(np.uint32) != 0xFFFFFFFF) or not np.all(np.isfinite(norms.numpy())):
                raise RuntimeError("solver error during e2e run")
        out_host.copy_(st.state().coeffs, non_blocking=True)
        torch.cuda.synchronize()
        return time.perf_counter() - t0

    e2e_pass()  # untimed warm-up pass (the caching allocator's first 400 MB blocks)
    e2e_s = e2e_pass()
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = dofs * n_st * args.steps / e2e_s
    state_bytes = host.numel() * 8

    wc = workload_config(args)
    if args.case == "cube":
        assert (wc["elements"], wc["faces"]) == (mesh.n_cells, mesh.n_faces), "Kuhn cube counts"
    else:
        wc.update(elements=mesh.n_cells, faces=mesh.n_faces, dofs=dofs)
    peaks, peak_kind = measured_peaks()
    alg = algorithmic_bytes_per_stage(mesh.n_cells, mesh.n_faces, args.order)
    achieved = alg / ((tf + te) * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as fh:
                tr = json.load(fh).get(f"n{args.n}_p{args.order}_prec{args.prec}")
            traffic = tr
        except Exception:
            traffic = None
    # the FP64 roof: the stage is FP64-pipe bound; algorithmic
    # FP64-pipe operations per stage (perf.count_flops_and_bytes, FMA = 1)
    from paper_2209_01877_b200 import perf as PF

    ops_step, _ = PF.count_flops_and_bytes(mesh, args.order, "rk3", args.prec)
    ops_stage = ops_step / n_st
    fp64_ops = PF.FP64_PIPE_OPS_PER_S
    line = {
        "metric": "DOF-updates/sec per RK stage (P2, 1M tets)",
        "value": value,
        "unit": "DOF-updates/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(args.warmup, 3),
        "ms_per_step": ms / args.steps,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": dtype_name(args),
        "data": ("synthetic Kuhn-cube tetrahedral mesh (random-shuffled then device-RCM renumbered), "
                 "projected isentropic vortex tube") if args.case == "cube" else
                "synthetic wedge-wing tetrahedral mesh, freestream Mach 0.5 at 3 degrees incidence",
        "config": dict(wc, renumbered=args.case == "cube" and not args.no_renumber, rcm_bandwidth=bw,
                       l2="inputs larger than L2 (state alone is %.0f MB)" % (state_bytes / 1e6),
                       parallelism=f"RCB element partition x{world}, NCCL halo" if world > 1 else "single GPU"),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                     "kernel": "RK stage = face_flux_kernel + elem_stage_kernel",
                     "algorithmic_bytes_per_stage": alg, "stage_ms": tf + te, "face_ms": tf, "elem_ms": te,
                     "peak_source": peak_kind,
                     "fp64": {"achieved": ops_stage / ((tf + te) * 1e-3) / 1e12, "peak": fp64_ops / 1e12,
                              "unit": "T FP64-pipe ops/s (FMA = 1 op)",
                              "frac": ops_stage / ((tf + te) * 1e-3) / fp64_ops,
                              "ops_per_stage": ops_stage,
                              "peak_source": "profiles/fp64_peaks.md (measured DFMA 36.3 TFLOP/s)",
                              "note": "FP64 applies to --prec 64; in mixed precision the traces and fluxes "
                                      "run on the FP32 pipe"}},
        "clocks": clk,
        "gpu_launches": kernels_per_step * args.steps,
        "e2e": {"value": e2e, "unit": "DOF-updates/s", "h2d_bytes_per_step": state_bytes / args.steps,
                "d2h_bytes_per_step": 56 + state_bytes / args.steps},
    }
    if rank == 0:
        line["cpu_baseline"] = cpu_baseline(args)
        print(json.dumps(line), flush=True)
    if dist_mode:
        torch.cuda.synchronize()
        st.close()  # the library's NCCL communicator before the process group
        dist.destroy_process_group()


def cpu_sample(args, n_sample=None, steps=2):
    """The oracle (C restatement of the reference kernels, OpenMP on all host
    cores) on a bounded sample of the workload: same order / scheme /
    precision, smaller cube."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle import _clib
    from oracle import mesh as OM
    from oracle import solver as S

    cores = os.cpu_count() or 1
    _clib.set_threads(cores)
    n = n_sample or (16 if args.order >= 2 else 24)
    m = OM.kuhn_box(n, (0.0, 0.0, 0.0, 10.0, 10.0, 10.0),
                    bc={"xmin": "far_field", "xmax": "far_field", "ymin": "far_field", "ymax": "far_field",
                        "zmin": "slip_wall", "zmax": "slip_wall"})
    disc = S.make_disc(m, args.order, S.Gas(), 0.5, 0.0)
    c = S.project_initial(m, disc.tab, lambda x, y, z: S.vortex_primitive(S.Gas(), 0.5, 0.0, 5.0, 5.0, 5.0, 0.0,
                                                                          x, y, dim=3), S.Gas())
    if args.prec == 32:
        c = np.ascontiguousarray(c.astype(np.float32))
    dt = S.min_reduce(S.local_dt_field(disc, c, 0.3, args.order))
    S.rk3_step(c, dt, lambda x: disc.rhs(x))  # warm
    t0 = time.perf_counter()
    for _ in range(steps):
        c = S.rk3_step(c, dt, lambda x: disc.rhs(x))
    sec = time.perf_counter() - t0
    dofs = m.n_cells * 5 * NB[args.order]
    return dofs * 3 * steps / sec, cores, f"oracle on {m.n_cells}-tet cube (n={n}), P{args.order}, {steps} SSP-RK3 steps"


def cpu_baseline(args):
    v, cores, sample = cpu_sample(args)
    return {"value": v, "unit": "DOF-updates/s", "cores": cores, "kind": "port", "sample": sample}


def dtype_name(args):
    return "f64" if args.prec == 64 else "f32-flux/f64-state"


def workload_config(args):
    """The workload both arms name: Kuhn cube of n^3 cells, 6 tets each
    (N = 6n^3, F = 12n^3 + 6n^2)."""
    n = args.n
    if getattr(args, "case", "cube") == "wing":
        return {"workload": f"config 4 wedge wing: Kuhn unit cube n={n} minus a swept diamond-section wing, "
                            f"P{args.order}, SSP-RK3, global CFL dt, {'FP64' if args.prec == 64 else 'mixed'}",
                "order": args.order}
    ne, nf = 6 * n ** 3, 12 * n ** 3 + 6 * n ** 2
    return {"workload": f"C1M-class cube n={n}: {ne} tets, {nf} faces, P{args.order} ({NB[args.order]} modes x 5 "
                        f"vars), SSP-RK3, global CFL dt, {'FP64' if args.prec == 64 else 'mixed FP32-flux/FP64'}",
            "elements": ne, "faces": nf, "order": args.order, "dofs": ne * 5 * NB[args.order]}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    steps = max(1, min(args.steps, 4))
    for _ in range(min(args.warmup, 1)):
        cpu_sample(args, steps=1)
    v, cores, sample = cpu_sample(args, steps=steps)
    line = {
        "impl": "reference",
        "metric": "DOF-updates/sec per RK stage (P2, 1M tets)",
        "value": v,
        "unit": "DOF-updates/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": steps,
        "warmup": args.warmup,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": dtype_name(args),
        "data": "synthetic Kuhn-cube tetrahedral mesh, projected isentropic vortex tube" if args.case == "cube" else
                "synthetic wedge-wing tetrahedral mesh, freestream Mach 0.5 at 3 degrees incidence",
        "config": workload_config(args),
        "cpu_baseline": {"value": v, "unit": "DOF-updates/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": "DOF-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
