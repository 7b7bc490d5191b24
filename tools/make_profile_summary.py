"""Write profiles/<tag>_summary.md (+ traffic.json) from a launch-list CSV
and an ncu --set full report brought back in gpurun_out/."""
import collections
import csv
import json
import os
import subprocess
import sys

tag, key = sys.argv[1], sys.argv[2]  # e.g. r1g n55_p2_prec64
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
go = os.path.join(root, "gpurun_out")
out = []
rows = list(csv.reader(open(os.path.join(go, f"{tag}_launches.csv"))))
hdr = None
data = collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            data[d["Kernel Name"].split("(")[0][:70]].append(float(d["Metric Value"].replace(",", "")))
tot = sum(sum(v) for v in data.values())
out.append(f"# ncu summary {tag} ({key})\n")
out.append("## Launch list (gpu__time_duration.sum, cold-cache, serialised; whole bench process incl. setup)\n")
out.append("| share | launches | avg us | kernel |\n|---|---|---|---|")
for k, v in sorted(data.items(), key=lambda kv: -sum(kv[1]))[:16]:
    out.append(f"| {sum(v) / tot * 100:.1f}% | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | `{k}` |")
stage = {k: v for k, v in data.items() if "face_flux" in k or "elem_stage" in k}
st = sum(sum(v) for v in stage.values())
out.append(f"\nWithin the RK stage (face + element kernels): " + ", ".join(
    f"`{k.split('::')[-1]}` {sum(v) / st * 100:.1f}%" for k, v in stage.items()))
rep = os.path.join(go, f"{tag}_full.ncu-rep")
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(txt.splitlines()))
h, u = rr[0], rr[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct", "launch__grid_size",
        "launch__block_size"]
out.append("\n## `ncu --set full` of the two stage kernels\n")
traffic = {}
for r in rr[2:]:
    name = r[h.index("Kernel Name")].split("(")[0]
    out.append(f"### `{name}`\n")
    out.append("| metric | value | unit |\n|---|---|---|")
    for k in keys:
        if k in h:
            i = h.index(k)
            out.append(f"| {k} | {r[i]} | {u[i]} |")
    stalls = [(x, r[i]) for i, x in enumerate(h) if x.startswith("smsp__average_warps_issue_stalled_")
              and x.endswith("_per_issue_active.ratio")]
    stalls = sorted(stalls, key=lambda s: -float(s[1].replace(",", "") or 0))[:6]
    out.append("\nTop stall reasons (warps per issue): " + ", ".join(
        f"{s.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {float(v):.2f}"
        for s, v in stalls) + "\n")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rb = float(r[h.index("dram__bytes_read.sum")].replace(",", "")) * scale[u[h.index("dram__bytes_read.sum")]]
    wb = float(r[h.index("dram__bytes_write.sum")].replace(",", "")) * scale[u[h.index("dram__bytes_write.sum")]]
    traffic["face" if "face" in name else "elem"] = rb + wb
open(os.path.join(root, "profiles", f"{tag}_summary.md"), "w").write("\n".join(out) + "\n")
tj = os.path.join(root, "profiles", "traffic.json")
d = json.load(open(tj)) if os.path.exists(tj) else {}
d[key] = traffic.get("face", 0) + traffic.get("elem", 0)
d[key + "_detail"] = traffic
json.dump(d, open(tj, "w"), indent=1)
print("\n".join(out))
