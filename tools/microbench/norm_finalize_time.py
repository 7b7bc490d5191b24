"""Time hodg_norm_finalize on a C1M-sized partial buffer (31,196 blocks x 5),
warm (the partials were just written, as after the stage-1 element kernel)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2209_01877_b200 import _lib

L = _lib.lib()
nblk = 31196
part = torch.rand(nblk * 5, dtype=torch.float64, device="cuda")
out = torch.empty(5, dtype=torch.float64, device="cuda")
for _ in range(10):
    L.hodg_norm_finalize(_lib.ptr(part), nblk, _lib.ptr(out), _lib.stream_ptr())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 200
e0.record()
for _ in range(n):
    L.hodg_norm_finalize(_lib.ptr(part), nblk, _lib.ptr(out), _lib.stream_ptr())
e1.record()
torch.cuda.synchronize()
print(f"norm_finalize: {e0.elapsed_time(e1) / n * 1000:.1f} us per launch (back to back)")
ref = torch.sqrt(part.view(nblk, 5).sum(0))
print("max rel diff vs torch:", float(((out - ref).abs() / ref).max()))
