"""Summarise an ncu source page (SASS) CSV: instruction mix and stall hot spots.

usage: ncu -i rep --page source --csv --print-source sass -k regex:NAME > x.csv
       python tools/sass_hot.py x.csv [top]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
sect = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # which kernel section
starts = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
hdr_i = starts[sect]
end = starts[sect + 1] - 1 if sect + 1 < len(starts) else len(rows)
print(rows[hdr_i - 1][:2])
hdr = rows[hdr_i]
data = [r for r in rows[hdr_i + 1:end] if len(r) == len(hdr)]
col = {h: i for i, h in enumerate(hdr)}
S = col["Warp Stall Sampling (All Samples)"]
X = col["Instructions Executed"]
stall_cols = [h for h in hdr if h.startswith("stall_") or "Stall" in h and h not in
              ("Warp Stall Sampling (All Samples)", "Warp Stall Sampling (Not-issued Samples)")]
mix = collections.Counter()
samp = collections.Counter()
tot_s = 0
tot_x = 0
for r in data:
    op = r[1].split()[0] if r[1].split() else "?"
    if op.startswith("@"):
        op = r[1].split()[1]
    base = op.split(".")[0]
    x = float(r[X] or 0)
    s = float(r[S] or 0)
    mix[base] += x
    samp[base] += s
    tot_s += s
    tot_x += x
print(f"instructions executed (warp-level): {tot_x:.4g}; stall samples: {tot_s:.4g}")
print("opcode            exec%   samples%")
for op, x in mix.most_common(20):
    print(f"{op:16s} {100 * x / tot_x:6.2f}  {100 * samp[op] / tot_s:6.2f}")
print("\nhottest instructions (samples):")
hot = sorted(data, key=lambda r: -float(r[S] or 0))[:top]
for r in hot:
    print(f"{r[0][-5:]} {float(r[S] or 0):7.0f}  {r[1].strip()[:90]}")
