"""bench.py's JSON contract on CPU: the reference arm (the oracle on the
host cores) prints one line with the keys the driver reads, naming the same
workload as the GPU arm."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1", "--n", "12"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "DOF-updates/s"
    # (a small cube keeps the CPU suite fast; the default is C1M, n = 55)
    assert d["config"]["elements"] == 6 * 12 ** 3 and d["config"]["faces"] == 12 * 12 ** 3 + 6 * 12 ** 2
    assert "workload" in d["cpu_baseline"]["sample"] or "tets" in d["cpu_baseline"]["sample"]
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0


def test_workload_config_counts():
    sys.path.insert(0, ROOT)
    import argparse

    import bench

    for n in (16, 32, 55):
        wc = bench.workload_config(argparse.Namespace(n=n, order=2, prec=64, case="cube"))
        assert wc["elements"] == 6 * n ** 3 and wc["faces"] == 12 * n ** 3 + 6 * n ** 2
