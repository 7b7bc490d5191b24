"""Where the end-to-end time goes (bench.py's e2e leg, phase by phase).

    python tools/e2e_breakdown.py [--n 55] [--steps 20]

Times each phase of the e2e region with CUDA events on the current stream:
pinned host -> device upload, Taylor -> reference transform + initial dt,
the K steps with their per-step norm / error-word reads, the reference ->
Taylor transform, and the device -> pinned host download.
"""

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=55)
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    P, mesh, gas, geo, bcs, state, _ = bench.build_case(a.n, 2, True, "cuda")
    from paper_2209_01877_b200 import _lib
    from paper_2209_01877_b200.dg import _get_disc
    from paper_2209_01877_b200.timestepping import Stepper

    disc = _get_disc(mesh, geo, gas, bcs)
    st = Stepper(disc, "rk3", _lib.PREC_F64, "global", 0.3, log_norms=True, use_graph=True)
    st.load(state)
    for _ in range(3):
        st.step()
    torch.cuda.synchronize()
    host = state.coeffs.cpu().pin_memory()
    out_host = torch.empty_like(host).pin_memory()
    norms = torch.empty(5, dtype=torch.float64).pin_memory()
    errh = torch.empty(4, dtype=torch.int32).pin_memory()
    for rep in range(3):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev[0].record()
        dev = host.to("cuda", non_blocking=True)
        ev[1].record()
        st.load(P.DofState(dev))
        ev[2].record()
        for _ in range(a.steps):
            st.step()
            norms.copy_(st.norms, non_blocking=True)
            errh.copy_(disc.err, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        ev[3].record()
        s = st.state().coeffs
        ev[4].record()
        out_host.copy_(s, non_blocking=True)
        ev[5].record()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        names = ["h2d", "load", "steps", "from_ref", "d2h"]
        ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(5)]
        gb = host.numel() * 8 / 1e9
        print(f"rep {rep}: wall {wall:.1f} ms | " + " ".join(f"{n} {m:.2f}" for n, m in zip(names, ms))
              + f" | h2d {gb / ms[0] * 1e3:.1f} GB/s d2h {gb / ms[4] * 1e3:.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
