"""Benchmark: DOF-updates/s per RK stage, FP64 P2 Euler, SSP-RK3, on the
synthetic ~1M-tet Kuhn cube (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--n 55] [--order 2] [--prec 64|32] [--no-renumber] [--no-sub] [--no-cpu]

One JSON line on rank 0.

* `value`: whole-job DOF-updates/s per stage of the headline workload (C1M,
  P2, FP64, RCM order) with the state resident in HBM (CUDA-event timed,
  max over ranks).
* `e2e`: the same metric through the public stepping API with the state
  uploaded from pinned host memory, the residual norms / error word read
  back every step (the reference's per-iteration logging and admissibility
  check) and the final state copied back, all inside the timed region.
* `sub`: device-timed lines for the other BASELINE configs on one GPU --
  the unrenumbered (seeded-shuffle) C1M order, mixed precision at C1M, and
  C4M at P3 (N = 1 only; `--no-sub` skips them).
* `cpu_baseline` / `--impl reference`: the CPU oracle (the C restatement of
  the reference's numba kernels, OpenMP on all host cores) on the SAME C1M
  workload, timed dual-phase as the reference's perf harness does
  (hodg/perf.py:83-100).
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NB = {0: 1, 1: 4, 2: 10, 3: 20}
RBAR = 5.0 / 3.0  # mean state reads per SSP-RK3 stage
METRIC = "DOF-updates/sec per RK stage (P2, 1M tets)"
CUBE_BC = {"xmin": "far_field", "xmax": "far_field", "ymin": "far_field", "ymax": "far_field",
           "zmin": "slip_wall", "zmax": "slip_wall"}
EXTENT = (0.0, 0.0, 0.0, 10.0, 10.0, 10.0)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=55, help="Kuhn cube size: 6 n^3 tets (55 -> 998,250)")
    ap.add_argument("--order", type=int, default=2)
    ap.add_argument("--prec", type=int, default=64, choices=[64, 32])
    ap.add_argument("--no-renumber", action="store_true",
                    help="time the seeded-shuffle order (randomize_cells = 1) without RCM")
    ap.add_argument("--case", default="cube", choices=["cube", "wing"],
                    help="cube: the C1M-class Kuhn cube (headline); wing: BASELINE config 4's wedge-wing mesh")
    ap.add_argument("--layout", default="auto", choices=["auto", "elem", "face"], help="face flux record layout")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg (A/B runs)")
    ap.add_argument("--no-sub", action="store_true", help="skip the sub-records (A/B runs)")
    ap.add_argument("--roofline-csv", default=None, help="also write the reference-format roofline CSV here")
    ap.add_argument("--partitioned", action="store_true",
                    help="use the partitioned (NCCL halo) stepper even at one rank")
    return ap.parse_args()


def algorithmic_bytes_per_stage(n_elem, n_faces, order, state_bytes=8):
    """N[(rbar+1) 8 nvar nb + G_e] + F G_f, G_e = 112, G_f = 44."""
    return n_elem * ((RBAR + 1.0) * state_bytes * 5 * NB[order] + 112) + n_faces * 44


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


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


def build_cube(n, order, renumber=True, shuffle=True, device="cuda"):
    """The C1M-class workload: Kuhn cube on the device, shuffled with the
    reference's randomize_cells = 1 (numpy PCG64 seed 1), then device RCM +
    face re-sort unless renumber is False.  Projected isentropic vortex tube."""
    import paper_2209_01877_b200 as P

    mesh = P.generate_tet_box(n, extent=EXTENT, bc=CUBE_BC, device=device)
    bw = None
    if shuffle:
        mesh = P.apply_permutation(mesh, P.random_permutation(mesh.n_cells, 1))
    if renumber:
        g = P.build_adjacency(mesh)
        perm = P.rcm(g)
        bw = (P.bandwidth(g), P.bandwidth(g, perm))
        mesh = P.apply_permutation(mesh, perm, device="cuda")  # face re-sort on the GPU
    elif shuffle:
        g = P.build_adjacency(mesh)
        bw = (P.bandwidth(g), P.bandwidth(g))
    gas = P.GasModel()
    geo = P.compute_geometry(mesh, order, device=device)  # element records on the GPU
    bcs = P.BoundaryConditions(P.freestream_conserved(gas, 0.5, 0.0))
    state = P.project_initial(mesh, geo, lambda x, y, z: P.vortex_primitive(gas, 0.5, 0.0, 5.0, 5.0, 5.0, 0.0, x, y),
                              gas)
    return mesh, gas, geo, bcs, state, bw


def build_case(args, device="cuda"):
    import paper_2209_01877_b200 as P

    if args.case == "wing":
        # BASELINE config 4: swept wedge wing cut out of the unit cube (slip
        # walls on the wing and the symmetry plane, far field elsewhere),
        # freestream at Mach 0.5 and 3 degrees incidence
        mesh = P.generate_wing_box(args.n, device=device)
        gas = P.GasModel()
        geo = P.compute_geometry(mesh, args.order, device=device)
        bcs = P.BoundaryConditions(P.freestream_conserved(gas, 0.5, 3.0))
        state = P.project_initial(mesh, geo, lambda x, y, z: P.freestream_primitive(gas, 0.5, 3.0), gas)
        return mesh, gas, geo, bcs, state, None
    return build_cube(args.n, args.order, renumber=not args.no_renumber, device=device)


def time_steps(st, steps):
    """ms for `steps` fused steps, CUDA events on the launching stream."""
    import torch

    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        st.step()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def kernel_times(st, disc, prec, n_st=3, reps=3):
    """Mean face-kernel and element-kernel ms per stage: events around each
    launch, outside the graph."""
    import torch

    hb = st.hbuf
    t_face, t_elem = [], []
    for k in range(reps * n_st):
        stage = k % n_st
        us = st.A if stage == 0 else st.B
        a = st._stage_args(stage, st.parity)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        if st._uses_shadow():  # mixed: the face kernel reads the FP32 shadow rows
            disc.face_flux32(st.A32 if stage == 0 else st.B32, hb)
        else:
            disc.face_flux(us, prec, hb)
        ev[1].record()
        disc.stage(prec, hb, a)
        ev[2].record()
        torch.cuda.synchronize()
        t_face.append(ev[0].elapsed_time(ev[1]))
        t_elem.append(ev[1].elapsed_time(ev[2]))
        if stage == n_st - 1:
            st.parity = 1 - st.parity
    return float(np.mean(t_face)), float(np.mean(t_elem))


def sub_record(label, mesh, geo, gas, bcs, state, order, prec_bits, steps, warmup, bw=None, peaks=None):
    """Device-timed line of one more BASELINE config on this GPU."""
    from paper_2209_01877_b200 import _lib
    from paper_2209_01877_b200.dg import _get_disc
    from paper_2209_01877_b200.timestepping import Stepper

    prec = _lib.PREC_F64 if prec_bits == 64 else _lib.PREC_MIXED
    disc = _get_disc(mesh, geo, gas, bcs)
    st = Stepper(disc, "rk3", prec, "global", 0.3, log_norms=True, use_graph=True)
    st.load(state)
    for _ in range(max(warmup, 3)):
        st.step()
    st.check()
    ms = time_steps(st, steps)
    st.check(steps)
    tf, te = kernel_times(st, disc, prec, reps=1)
    dofs = mesh.n_cells * 5 * NB[order]
    alg = algorithmic_bytes_per_stage(mesh.n_cells, mesh.n_faces, order)
    rec = {"workload": label, "elements": mesh.n_cells, "faces": mesh.n_faces, "order": order,
           "dtype": "f64" if prec_bits == 64 else "f32-flux/f64-state", "steps": steps,
           "value": dofs * 3 * steps / (ms * 1e-3), "unit": "DOF-updates/s", "ms_per_step": ms / steps,
           "face_ms": tf, "elem_ms": te,
           "hbm_frac": alg / ((tf + te) * 1e-3) / (peaks["hbm_gbs"] * 1e9) if peaks else None}
    if bw is not None:
        rec["rcm_bandwidth"] = bw
    return rec


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
    import paper_2209_01877_b200 as P
    from paper_2209_01877_b200 import _lib
    from paper_2209_01877_b200 import perf as PF
    from paper_2209_01877_b200.dg import _get_disc
    from paper_2209_01877_b200.timestepping import Stepper

    mesh, gas, geo, bcs, state, bw = build_case(args)
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
    for _ in range(max(args.warmup, 3)):
        st.step()
    kernels_per_step = st.launches_per_step()
    torch.cuda.synchronize()
    st.check()

    # ---- device-resident timed region ----
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    ms = time_steps(st, args.steps)
    barrier()
    clk = clocks.stop()
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    st.check(args.steps)
    value = dofs * n_st * args.steps / (ms * 1e-3)  # whole job: the global mesh

    # ---- per-kernel durations (events around each launch, no graph) ----
    tf, te = kernel_times(st, disc, prec)

    # ---- end to end through the public stepping API ----
    host = state_in.coeffs.cpu().pin_memory()
    out_host = torch.empty_like(host).pin_memory()
    # per-step reads into a two-slot pinned ring: step k's norms / error word
    # are copied right after its launch and checked on the host while step
    # k + 1 runs (every step is read and checked; the GPU never waits on it)
    norms = [torch.empty(5, dtype=torch.float64).pin_memory() for _ in range(2)]
    errh = [torch.empty(4, dtype=torch.int32).pin_memory() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]

    def read_ok(k):
        done[k % 2].synchronize()
        return not (np.any(errh[k % 2].numpy().astype(np.uint32) != 0xFFFFFFFF)
                    or not np.all(np.isfinite(norms[k % 2].numpy())))

    def e2e_pass():
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev_state = P.DofState(host.to("cuda", non_blocking=True))
        st.load(dev_state)
        for k in range(args.steps):
            # (distributed: every rank reads its norms / error word each step)
            st.step()
            norms[k % 2].copy_(st.norms, non_blocking=True)
            errh[k % 2].copy_(disc.err, non_blocking=True)
            done[k % 2].record()
            if k > 0 and not read_ok(k - 1):
                raise RuntimeError(f"solver error during e2e run (step {k - 1})")
        if not read_ok(args.steps - 1):
            raise RuntimeError("solver error during e2e run (last step)")
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
    stage_s = (tf + te) * 1e-3
    achieved = alg / stage_s / 1e9
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as fh:
                tj = json.load(fh)
            key = f"n{args.n}_p{args.order}_prec{args.prec}"
            traffic = tj.get(key)
            traffic_src = tj.get("_source", {}).get(key) if traffic is not None else None
        except Exception:
            traffic = None
    # FP64 rooflines: (1) the §8(d) algorithmic flops in the reference's
    # convention, independent of the implementation; (2) the FP64-pipe
    # operations the kernels issue (FMA = 1), i.e. pipe utilisation
    n_bnd = int(np.count_nonzero(np.asarray(mesh.face_cells)[:, 1] < 0))
    flops_stage = PF.algorithmic_flops_per_stage(mesh.n_cells, mesh.n_faces, n_bnd, args.order)
    ops_step, _ = PF.count_flops_and_bytes(mesh, args.order, "rk3", args.prec)
    ops_stage = ops_step / n_st
    line = {
        "metric": METRIC,
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
        "data": ("synthetic Kuhn-cube tetrahedral mesh (seeded shuffle, then device-RCM renumbered), "
                 "projected isentropic vortex tube") if args.case == "cube" else
                "synthetic wedge-wing tetrahedral mesh, freestream Mach 0.5 at 3 degrees incidence",
        "config": dict(wc, renumbered=args.case == "cube" and not args.no_renumber, rcm_bandwidth=bw,
                       l2="inputs larger than L2 (state alone is %.0f MB)" % (state_bytes / 1e6),
                       parallelism=f"RCB element partition x{world}, NCCL halo" if world > 1 else "single GPU"),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / peaks["hbm_gbs"], "traffic": traffic, "traffic_source": traffic_src,
                     "kernel": "RK stage = face_flux_kernel + element stage kernel",
                     "algorithmic_bytes_per_stage": alg, "stage_ms": tf + te, "face_ms": tf, "elem_ms": te,
                     "peak_source": peak_kind,
                     "fp64_alg": {"achieved": flops_stage / stage_s / 1e12, "peak": PF.FP64_FLOPS_PER_S / 1e12,
                                  "unit": "TFLOP/s", "frac": flops_stage / stage_s / PF.FP64_FLOPS_PER_S,
                                  "flops_per_stage": flops_stage,
                                  "convention": "SURVEY.md §8(d), reference hodg/perf.py (add/mul/div/sqrt = 1)",
                                  "peak_source": "profiles/fp64_peaks.md (measured DFMA 36.3 TFLOP/s)"},
                     "fp64_pipe": {"achieved": ops_stage / stage_s / 1e12, "peak": PF.FP64_PIPE_OPS_PER_S / 1e12,
                                   "unit": "T FP64-pipe ops/s (FMA = 1 op)",
                                   "frac": ops_stage / stage_s / PF.FP64_PIPE_OPS_PER_S, "ops_per_stage": ops_stage,
                                   "note": "the kernels' own operation count: pipe utilisation"}},
        "clocks": clk,
        "gpu_launches": kernels_per_step * args.steps,
        "e2e": {"value": e2e, "unit": "DOF-updates/s", "h2d_bytes_per_step": state_bytes / args.steps,
                "d2h_bytes_per_step": 56 + state_bytes / args.steps},
    }
    if rank == 0 and not dist_mode and not args.no_sub and args.case == "cube":
        del st
        torch.cuda.empty_cache()
        sub = {}
        # BASELINE config 2: the same C1M mesh, mixed precision (FP32 flux, FP64 state)
        sub["c1m_p2_mixed"] = sub_record(f"C1M n={args.n} P2 mixed, RCM", mesh, geo, gas, bcs, state, args.order, 32,
                                         args.steps, args.warmup, bw, peaks)
        # config 2: unrenumbered = the seeded shuffle without RCM
        m2, g2, ge2, b2, s2, bw2 = build_cube(args.n, args.order, renumber=False)
        sub["c1m_p2_unrenumbered"] = sub_record(f"C1M n={args.n} P2 FP64, shuffled order (no RCM)", m2, ge2, g2, b2,
                                                s2, args.order, 64, args.steps, args.warmup, bw2, peaks)
        del m2, ge2, s2
        # config 3 on one GPU: C4M (n = 87), P3
        m3, g3, ge3, b3, s3, bw3 = build_cube(87, 3)
        sub["c4m_p3_fp64"] = sub_record("C4M n=87 P3 FP64, RCM", m3, ge3, g3, b3, s3, 3, 64, max(3, args.steps // 4),
                                        args.warmup, bw3, peaks)
        del m3, ge3, s3
        torch.cuda.empty_cache()
        # config 4 on one GPU: the 8M-tet wedge-wing mesh, P2 (wall + far field)
        wa = argparse.Namespace(**dict(vars(args), case="wing", n=110, order=2))
        m4, g4, ge4, b4, s4, _ = build_case(wa)
        sub["wing_c8m_p2_fp64"] = sub_record(f"config 4 wedge wing, n=110 ({m4.n_cells} tets), P2 FP64", m4, ge4, g4,
                                             b4, s4, 2, 64, max(3, args.steps // 4), args.warmup, None, peaks)
        del m4, ge4, s4
        torch.cuda.empty_cache()
        line["sub"] = sub
    if rank == 0:
        line["cpu_baseline"] = None if (args.no_cpu or dist_mode) else cpu_baseline(args)
        if args.roofline_csv:
            # the reference's roofline CSV (hodg/perf.py:208-238) fed by this
            # run's times, the algorithmic flops and the measured DRAM bytes
            samples = [("c1m_stage_alg_bytes", PF.PerfSample(stage_s, flops_stage, alg, 1))]
            if traffic:
                samples.append(("c1m_stage_ncu_bytes", PF.PerfSample(stage_s, flops_stage, float(traffic), 1)))
            machine = PF.MachineModel("b200-measured", PF.FP64_FLOPS_PER_S, peaks["hbm_gbs"] * 1e9)
            PF.emit_roofline_csv(samples, [machine], args.roofline_csv)
        print(json.dumps(line), flush=True)
    if dist_mode:
        torch.cuda.synchronize()
        st.close()  # the library's NCCL communicator before the process group
        dist.destroy_process_group()


def oracle_case(args):
    """The oracle on the same workload as our arm (same mesh generator,
    shuffle seed and RCM, same initial state)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle import _clib
    from oracle import mesh as OM
    from oracle import renumber as OR
    from oracle import solver as S

    cores = os.cpu_count() or 1
    _clib.set_threads(cores)
    m = OM.kuhn_box(args.n, EXTENT, bc=CUBE_BC)
    # randomize_cells = 1, then RCM unless --no-renumber (host restatement)
    m = OR.apply_permutation(m, *OR.random_permutation(m.n_cells, 1))
    if not args.no_renumber:
        m = OR.apply_permutation(m, *OR.rcm(OR.adjacency(m)))
    disc = S.make_disc(m, args.order, S.Gas(), 0.5, 0.0)
    c = S.project_initial(m, disc.tab, lambda x, y, z: S.vortex_primitive(S.Gas(), 0.5, 0.0, 5.0, 5.0, 5.0, 0.0,
                                                                          x, y, dim=3), S.Gas())
    if args.prec == 32:
        c = np.ascontiguousarray(c.astype(np.float32))
    return m, disc, c, cores


def oracle_dual_phase(args, n1, n2, warm=1):
    """Seconds per SSP-RK3 step of the oracle, dual phase: run n1 and n2
    steps and difference the totals (hodg/perf.py:83-100)."""
    from oracle import solver as S

    m, disc, c0, cores = oracle_case(args)
    dt = S.min_reduce(S.local_dt_field(disc, c0, 0.3, args.order))

    def run(n):
        c = c0
        t0 = time.perf_counter()
        for _ in range(n):
            c = S.rk3_step(c, dt, lambda x: disc.rhs(x))
        return time.perf_counter() - t0

    for _ in range(warm):
        run(1)
    reps = 1 if m.n_cells >= 100000 else 3  # small samples: min of 3 per phase
    t1 = min(run(n1) for _ in range(reps))
    t2 = min(run(n2) for _ in range(reps))
    per_step = (t2 - t1) / (n2 - n1)
    if not per_step > 0.0:  # timer noise on a tiny sample
        per_step = t2 / n2
    return per_step, m.n_cells, cores


def cpu_baseline(args):
    n1, n2 = 1, 3
    per_step, ncell, cores = oracle_dual_phase(args, n1, n2)
    dofs = ncell * 5 * NB[args.order]
    return {"value": dofs * 3 / per_step, "unit": "DOF-updates/s", "cores": cores, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"oracle (C restatement of the reference kernels, OpenMP) on the full workload "
                      f"({ncell} tets, P{args.order}), dual phase {n1} vs {n2} SSP-RK3 steps"}


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
    order_txt = "seeded shuffle, no RCM" if getattr(args, "no_renumber", False) else "seeded shuffle + RCM"
    return {"workload": f"C1M-class cube n={n}: {ne} tets, {nf} faces, P{args.order} ({NB[args.order]} modes x 5 "
                        f"vars), SSP-RK3, global CFL dt, {'FP64' if args.prec == 64 else 'mixed FP32-flux/FP64'}, "
                        f"{order_txt}",
            "elements": ne, "faces": nf, "order": args.order, "dofs": ne * 5 * NB[args.order]}


def run_reference(args):
    """The reference arm: the CPU oracle on the same workload, all host
    cores; `steps` timed SSP-RK3 steps after `warmup`, dual phase against a
    shorter run (hodg/perf.py:83-100)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if args.case != "cube":
        print(json.dumps({"impl": "reference", "unavailable": "the CPU arm runs the cube workloads only"}))
        return
    n2 = max(2, args.steps)
    n1 = max(1, n2 // 4)
    per_step, ncell, cores = oracle_dual_phase(args, n1, n2, warm=max(1, min(args.warmup, 2)))
    dofs = ncell * 5 * NB[args.order]
    v = dofs * 3 / per_step
    sample = (f"oracle (C restatement of the reference kernels, OpenMP) on the full workload ({ncell} tets, "
              f"P{args.order}), dual phase {n1} vs {n2} SSP-RK3 steps")
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": v,
        "unit": "DOF-updates/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": n2,
        "warmup": args.warmup,
        "ms_per_step": per_step * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": dtype_name(args),
        "data": "synthetic Kuhn-cube tetrahedral mesh (seeded shuffle, RCM), projected isentropic vortex tube",
        "config": workload_config(args),
        "cpu_baseline": {"value": v, "unit": "DOF-updates/s", "cores": cores, "kind": "port",
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": v, "unit": "DOF-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
