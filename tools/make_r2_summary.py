"""Write profiles/r2_summary.md from the round-2 captures in gpurun_out/:
launch list (r2p_launches.csv), --set full of the stage kernels (r2p_fp64 /
r2p_mixed: face kernels; r2q_elem64 / r2q_elem32: element kernels) and the
warm-cache DRAM traffic per launch (r2p_warm_traffic.csv); also refresh
profiles/traffic.json (mean DRAM bytes per RK stage, warm cache)."""
import collections
import csv
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GO = os.path.join(ROOT, "gpurun_out")
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "lts__t_sector_hit_rate.pct",
        "launch__grid_size", "launch__block_size"]


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for k in KEYS:
            if k in hdr:
                d[k] = (r[hdr.index(k)], units[hdr.index(k)])
        st = [(h, r[i]) for i, h in enumerate(hdr)
              if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
        st = sorted(st, key=lambda x: -float(x[1].replace(",", "") or 0))[:6]
        d["stalls"] = ", ".join(f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {float(v):.2f}" for h, v in st)
        res.append(d)
    return res


def main():
    out = ["# ncu summary, round 2 (C1M P2, `bench.py --no-cpu --no-sub --steps 5 --warmup 3`)\n",
           "Captured on the B200 after the round-2 kernel changes (flux-moment volume integral, exact face-gather "
           "folding, regrouped Roe dissipation, FP32 state shadow in mixed precision, branch-free face traces, packed "
           "FP32 (FFMA2) contractions in the mixed kernels, cp.async FP32 face records; state rows and FP64 records by "
           "per-row TMA bulk copies -- the gather4 variants are off by default, DESIGN.md section 3). "
           "Commands: `tools/profile_r2.sh`, `tools/profile_elem.sh`.\n",
           "## Launch list (gpu__time_duration.sum, cold-cache, serialised; whole bench process incl. setup)\n"]
    rows = list(csv.reader(open(os.path.join(GO, "r2p_launches.csv"))))
    hdr, data = None, collections.defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                data[d["Kernel Name"].split("(")[0][:80]].append(float(d["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in data.values())
    out.append("| share | launches | avg us | kernel |\n|---|---|---|---|")
    for k, v in sorted(data.items(), key=lambda kv: -sum(kv[1]))[:14]:
        out.append(f"| {sum(v) / tot * 100:.1f}% | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | `{k}` |")
    stage = {k: v for k, v in data.items() if "face_flux" in k or "elem_stage" in k}
    st = sum(sum(v) for v in stage.values())
    out.append("\nWithin the RK stage (FP64): " + ", ".join(
        f"`{k.split('::')[-1]}` {sum(v) / st * 100:.1f}%" for k, v in stage.items()) + "\n")
    for title, rep in (("FP64 face kernels", "r2p_fp64"), ("FP64 element kernel", "r2q_elem64"),
                       ("mixed-precision face kernels (FP32 shadow rows)", "r2p_mixed"),
                       ("mixed-precision element kernel (element-slot records, FP32 shadow out)", "r2q_elem32")):
        path = os.path.join(GO, rep + ".ncu-rep")
        if not os.path.exists(path):
            continue
        out.append(f"## `ncu --set full`: {title} (`{rep}`)\n")
        for d in full(path):
            out.append(f"### `{d['kernel']}`\n\n| metric | value | unit |\n|---|---|---|")
            for k in KEYS:
                if k in d:
                    out.append(f"| {k} | {d[k][0]} | {d[k][1]} |")
            out.append(f"\nTop stall reasons (warps per issue): {d['stalls']}\n")
    # warm traffic
    rows = list(csv.reader(open(os.path.join(GO, "r2p_warm_traffic.csv"))))
    hdr, rec = None, collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            rec.setdefault((int(d["ID"]), d["Kernel Name"].split("(")[0]), {})[d["Metric Name"]] = \
                float(d["Metric Value"].replace(",", ""))
    out.append("## Warm-cache DRAM traffic per launch (`ncu --cache-control none`, FP64, 12 launches = 4 stages)\n")
    out.append("| launch | kernel | DRAM read GB | DRAM write GB | L2 hit % | us |\n|---|---|---|---|---|---|")
    for (i, k), v in rec.items():
        out.append(f"| {i} | `{k.split('::')[-1][:48]}` | {v['dram__bytes_read.sum'] / 1e9:.3f} | "
                   f"{v['dram__bytes_write.sum'] / 1e9:.3f} | {v['lts__t_sector_hit_rate.pct']:.1f} | "
                   f"{v['gpu__time_duration.sum'] / 1e3:.1f} |")
    vals = list(rec.values())
    per = [sum(x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in vals[i:i + 3])
           for i in range(0, len(vals) - 2, 3)]
    mean3 = sum(per[:3]) / 3
    out.append(f"\nDRAM bytes per RK stage (face interior + boundary + element): "
               + ", ".join(f"{p / 1e9:.3f} GB" for p in per)
               + f"; mean over one SSP-RK3 step {mean3 / 1e9:.3f} GB against 1.265 GB algorithmic.\n")
    with open(os.path.join(ROOT, "profiles", "r2_summary.md"), "w") as fh:
        fh.write("\n".join(out) + "\n")
    tj = {"n55_p2_prec64": mean3,
          "_source": {"n55_p2_prec64": "profiles/r2_summary.md (warm-cache ncu, mean DRAM bytes per SSP-RK3 "
                                       "stage, r2p_warm_traffic.csv)"}}
    with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as fh:
        json.dump(tj, fh, indent=1)
    print("wrote profiles/r2_summary.md", mean3)


if __name__ == "__main__":
    main()
