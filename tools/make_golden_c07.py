"""tests/golden/c07_levels.json: the reference's acceptance-c07 runs
(pkg/tests/test_acceptance.py:263-310) -- residual histories' tail levels and
full density-residual histories for dp / sp / mp_late / mp_early.  Runs only
in the build container (imports the reference from /root/reference).

Usage:  python tools/make_golden_c07.py
"""
import json
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
os.environ.setdefault("NUMBA_NUM_THREADS", "16")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import hodg  # noqa: E402,F401
from hodg.config import RunConfig  # noqa: E402
from hodg.timestepping import run  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "c07_levels.json")
base = dict(gen_kind="quad", gen_nx=2016, gen_ny=8, gen_extent=(0.0, 0.0, 252.0, 1.0), initial_kind="pulse",
            initial_x0=126.0, initial_y0=0.5, pulse_amplitude=0.2, pulse_sigma=0.3, dt_mode="local",
            max_iterations=2200, log_every=25, workers=16, mach=0.4, order=1, cfl=0.5, ivis=1, mu_dyn=0.002)
out = {}
for tag, kw in (("dp", dict(precision_mode="dp")), ("sp", dict(precision_mode="sp")),
                ("mp_late", dict(precision_mode="mp_fixed", switch_iter=1950)),
                ("mp_early", dict(precision_mode="mp_fixed", switch_iter=1500))):
    art = run(RunConfig(**base, **kw))
    res = np.array(art.history.res)[:, 0]
    k = max(1, int(len(res) * 0.1))
    out[tag] = {"tail_level": float(res[-k:].mean()), "res_rho": [float(x) for x in res],
                "iterations": [int(i) for i in art.history.iterations]}
    print(tag, out[tag]["tail_level"], flush=True)
with open(OUT, "w") as fh:
    json.dump(out, fh)
print("wrote", OUT)
