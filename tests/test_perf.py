"""Performance tooling (hodg/perf.py restated): CSV formats regenerate the
reference's perf fixtures byte for byte; dual-phase arithmetic; the
analytic model's stage bytes equal SURVEY.md §8(d)."""

import pytest

from conftest import golden_path
from paper_2209_01877_b200 import perf
from paper_2209_01877_b200.mesh import generate_tet_box


def test_roofline_and_timing_csv_bytewise(tmp_path):
    S = perf.PerfSample
    samples = [("grid4", S(0.020, 4.0e8, 3.2e9, 1)), ("grid5", S(0.085, 1.6e9, 1.28e10, 1)),
               ("dense", S(0.010, 5.0e9, 2.0e8, 1))]
    machines = [perf.MachineModel("cpu-node", 3.0e12, 2.0e11), perf.MachineModel("gpu-node", 7.0e12, 9.0e11)]
    perf.emit_roofline_csv(samples, machines, tmp_path / "roofline.csv")
    perf.emit_timing_csv([("grid4", 1, 0.0400), ("grid4", 2, 0.0215), ("grid4", 8, 0.0095),
                          ("grid5", 1, 0.1660), ("grid5", 2, 0.0890), ("grid5", 8, 0.0410)], tmp_path / "timing.csv")
    for n in ("roofline.csv", "timing.csv"):
        with open(golden_path(n)) as fh:
            assert (tmp_path / n).read_text() == fh.read()


def test_dual_phase_differences():
    calls = []

    def run(n):
        calls.append(n)
        return perf.PerfSample(1.0 + 0.5 * n, 10.0 + 3.0 * n, 100.0 + 7.0 * n, n)

    s = perf.dual_phase(run, 2, 6)
    assert calls == [2, 6]
    assert (s.wall_seconds, s.flops, s.dram_bytes) == (0.5, 3.0, 7.0)
    with pytest.raises(ValueError):
        perf.dual_phase(run, 3, 3)


def test_stage_bytes_match_survey_model():
    m = generate_tet_box(3)
    _, b = perf.count_flops_and_bytes(m, 2, "rk3")
    per_stage = m.n_cells * ((5.0 / 3.0 + 1.0) * 8 * 5 * 10 + 112) + m.n_faces * 44
    assert abs(b / 3 - per_stage) < 1e-6 * per_stage
    f, _, d = perf.count_flops_and_bytes(m, 2, "rk3", detail=True)
    assert f == 3 * sum(d.values())


def test_roofline_attainable():
    mm = perf.MachineModel("x", 10.0, 2.0)
    assert perf.roofline_attainable(mm, 1.0) == 2.0
    assert perf.roofline_attainable(mm, 100.0) == 10.0


def test_algorithmic_flops_reference_convention():
    """~16.8k flops per element per stage at C1M P2 in the
    reference's convention (add / mul / div / sqrt = 1), independent of the
    kernels; P1 < P2 < P3 per element."""
    from paper_2209_01877_b200 import perf

    n, f, fb = 998250, 2014650, 36300
    per = {p: perf.algorithmic_flops_per_stage(n, f, fb, p) / n for p in (1, 2, 3)}
    assert 16500 < per[2] < 17200
    assert per[1] < per[2] < per[3]
    # rk2 stages carry fewer RK flops per DOF than rk3 stages
    assert perf.algorithmic_flops_per_stage(n, f, fb, 2, "rk2") > 0
