"""Performance measurement and modelling (hodg/perf.py:1-246) for the
tetrahedral B200 path.

* `dual_phase(run_fn, n1, n2)` -- per-iteration cost isolated by running the
  whole application twice and differencing (hodg/perf.py:83-100);
  `device_dual_phase` does the same with CUDA-event timing of the fused
  stepper.
* `count_flops_and_bytes` -- per-step algorithmic DRAM bytes by SURVEY.md
  §8(d) (state reads/writes + compact geometry; tables, face buffers and
  halos are implementation cost and excluded) and FP64-pipe operations of
  the kernels as written (counted from the kernel structure; Roe ~250 ops
  per Riemann solve as measured by tools/microbench/roe_rate.cu).
* `emit_roofline_csv` / `emit_timing_csv` -- the reference's CSV formats
  (consumed by its viz package); they regenerate the reference's
  fixtures/roofline.csv and timing.csv byte for byte (tests/test_perf.py).
"""

from __future__ import annotations

from dataclasses import dataclass

from .refelem import ref_tables

__all__ = ["PerfSample", "MachineModel", "dual_phase", "device_dual_phase", "count_flops_and_bytes",
           "roofline_attainable", "emit_roofline_csv", "emit_timing_csv", "B200"]

ROE_OPS = 250  # FP64-pipe ops per Riemann solve (measured, see module doc)
PRIM_FLUX_OPS = 30  # primitives + physical flux per volume point
STAGES = {"rk2": 2, "rk3": 3}
RBAR = {"rk2": 1.5, "rk3": 5.0 / 3.0}


@dataclass(frozen=True)
class PerfSample:
    wall_seconds: float
    flops: float
    dram_bytes: float
    iterations: int

    def __post_init__(self):
        if min(self.wall_seconds, self.flops, self.dram_bytes, self.iterations) < 0:
            raise ValueError("performance sample fields must be non-negative")

    @property
    def achieved_flops(self) -> float:
        return self.flops / self.wall_seconds if self.wall_seconds > 0 else 0.0

    @property
    def arithmetic_intensity(self) -> float:
        return self.flops / self.dram_bytes if self.dram_bytes > 0 else 0.0


@dataclass(frozen=True)
class MachineModel:
    label: str
    peak_flops: float
    peak_bandwidth: float

    def __post_init__(self):
        if self.peak_flops <= 0 or self.peak_bandwidth <= 0:
            raise ValueError("machine peaks must be positive")


# measured on this pool's B200s: DFMA 36.3 TFLOP/s = 18.15 T FP64-pipe
# instructions/s (profiles/fp64_peaks.md; DMMA shares the same budget), copy
# bandwidth 6551 GB/s (MEASURED_PEAKS.json).  count_flops_and_bytes counts
# an FMA as one operation, so the machine model's peak is in the same unit.
FP64_PIPE_OPS_PER_S = 36.3e12 / 2
B200 = MachineModel("b200-fp64", FP64_PIPE_OPS_PER_S, 6551.4e9)


def dual_phase(run_fn, n1: int, n2: int) -> PerfSample:
    """Run the full application for n1 and n2 iterations and difference the
    totals, removing everything that does not scale with the iterations."""
    if n1 < 1 or n2 <= n1:
        raise ValueError("need n2 > n1 >= 1")
    a, b = run_fn(n1), run_fn(n2)
    k = n2 - n1
    return PerfSample((b.wall_seconds - a.wall_seconds) / k, (b.flops - a.flops) / k,
                      (b.dram_bytes - a.dram_bytes) / k, 1)


def device_dual_phase(stepper, n1: int, n2: int) -> float:
    """Seconds per step of a fused Stepper, CUDA-event timed, dual phase."""
    import torch

    def timed(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(n):
            stepper.step()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e-3

    if n1 < 1 or n2 <= n1:
        raise ValueError("need n2 > n1 >= 1")
    return (timed(n2) - timed(n1)) / (n2 - n1)


def count_flops_and_bytes(mesh, order: int, scheme: str = "rk3", precision_bits: int = 64, detail: bool = False):
    """Per-step FP64-pipe operations (flops: FMA counted once) and
    algorithmic DRAM bytes of the tetrahedral path."""
    t = ref_tables(order)
    nb, nqv, nqf = t.nb, t.nqv, t.nqf
    n, f = mesh.n_cells, mesh.n_faces
    nd = int(sum(1 for i in range(nb) for d in range(3) if t.E[i][d] > 0))  # nonzero derivative pairs
    st = STAGES[scheme]
    face = f * (2 * 5 * nb * nqf + nqf * ROE_OPS)
    vol = n * nqv * (5 * nb + PRIM_FLUX_OPS + 5 * (9 + nd))
    gather = n * 5 * 4 * (nqf * nb + nb)
    solve = n * 5 * nb * nb
    rk = n * 5 * nb * 3
    per_stage = face + vol + gather + solve + rk
    flops = st * per_stage
    bytes_stage = n * ((RBAR[scheme] + 1.0) * (precision_bits // 8) * 5 * nb + 112) + f * 44
    if detail:
        return flops, st * bytes_stage, {"face_pass": face, "volume": vol, "gather": gather, "solve": solve,
                                         "rk": rk}
    return flops, st * bytes_stage


# SURVEY.md §8(d) constants, hand-counted from the 3D scalar code in the
# reference's convention (add / mul / div / sqrt = 1 flop, hodg/perf.py:1-49):
# Roe with Harten-Hyman, primitive recovery, inviscid flux, boundary state
ROE3, PRIM3, INV3, BND3 = 225, 15, 16, 95
RK_FLOPS_PER_DOF = {"rk2": 3.5, "rk3": 4.0}  # mean per stage: u+dt r (2), combos (5)
FP64_FLOPS_PER_S = 36.3e12  # measured DFMA peak (FMA = 2 flops), profiles/fp64_peaks.md


def algorithmic_flops_per_stage(n_cells: int, n_faces: int, n_bnd_faces: int, order: int, scheme: str = "rk3"):
    """Algorithmic flops of one RK stage, the reference's convention restated
    for tetrahedra (hodg/perf.py:130-158):
      flux   F_int nqf (10 trace + ROE3) + F_bnd nqf (5 trace + PRIM3 + BND3 + ROE3)
      volume N nqv (5 trace + PRIM3 + INV3 + 33 nb)
      gather (2 F_int + F_bnd) nqf (3 + 11 nb)
      solve  N 10 nb^2;  RK  N 5 nb (flops per DOF);  dt  N (10 nb + 25) per step
    with trace = 2 nb flops per variable.  Independent of how the kernels are
    written (unlike count_flops_and_bytes, which counts the implementation's
    own FP64-pipe operations)."""
    t = ref_tables(order)
    nb, nqv, nqf = t.nb, t.nqv, t.nqf
    tr = 2 * nb
    fi, fb = n_faces - n_bnd_faces, n_bnd_faces
    flux = fi * nqf * (10 * tr + ROE3) + fb * nqf * (5 * tr + PRIM3 + BND3 + ROE3)
    vol = n_cells * nqv * (5 * tr + PRIM3 + INV3 + 33 * nb)
    gather = (2 * fi + fb) * nqf * (3 + 11 * nb)
    solve = n_cells * 10 * nb * nb
    rk = n_cells * 5 * nb * RK_FLOPS_PER_DOF[scheme]
    dt = n_cells * (10 * nb + 25) / STAGES[scheme]
    return float(flux + vol + gather + solve + rk + dt)


def roofline_attainable(machine: MachineModel, ai: float) -> float:
    if ai < 0:
        raise ValueError("arithmetic intensity must be non-negative")
    return min(machine.peak_flops, machine.peak_bandwidth * ai)


def emit_roofline_csv(samples, machines, path, check: bool = False) -> None:
    """Rows (label, ai, achieved_flops, machine, attainable_flops, bound) in
    the reference's format (hodg/perf.py:208-238)."""
    samples, machines = list(samples), list(machines)
    if not samples or not machines:
        raise ValueError("need at least one sample and one machine model")
    out = ["# analytic ideal-traffic byte model: every float array is counted once per pass, so ai is an upper bound",
           "label,ai,achieved_flops,machine,attainable_flops,bound"]
    for label, s in samples:
        ai, got = s.arithmetic_intensity, s.achieved_flops
        for m in machines:
            roof = roofline_attainable(m, ai)
            if check and got > roof * (1 + 1e-9):
                raise ValueError(f"sample {label!r} achieves {got:.3e} above the {m.label} roof {roof:.3e}")
            bound = "memory" if m.peak_bandwidth * ai < m.peak_flops else "compute"
            out.append(f"{label},{float(ai)!r},{float(got)!r},{m.label},{float(roof)!r},{bound}")
    with open(path, "w") as fh:
        fh.write("\n".join(out) + "\n")


def emit_timing_csv(rows, path) -> None:
    with open(path, "w") as fh:
        fh.write("label,workers,seconds_per_iter\n")
        fh.writelines(f"{label},{int(w)},{float(sec)!r}\n" for label, w, sec in rows)
