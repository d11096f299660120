"""Summarise ncu evidence into profiles/ (tracked): a launch-list table and
per-kernel full-set metrics, plus profiles/ncu_summary.json (DRAM traffic per
launch, read by bench.py for roofline.traffic).

    python tools/ncu_summary.py <launches.csv> <full.ncu-rep> <config> <out.md> [note] [clouds_per_launch]
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

launch_csv, rep, config, out_md = sys.argv[1:5]
note = sys.argv[5] if len(sys.argv) > 5 else ""
clouds_per_launch = int(sys.argv[6]) if len(sys.argv) > 6 else None  # wave size of the full capture

# ---- launch list ------------------------------------------------------------
rows = list(csv.reader(open(launch_csv)))
hdr, agg = None, collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        if r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue  # launch lists may carry DRAM byte counts too
        k = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
        unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
        v = float(r[hdr.index("Metric Value")].replace(",", "")) * {"ns": 1, "nsecond": 1, "us": 1e3,
                                                                   "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
tot = sum(v[1] for v in agg.values())

# ---- full-set metrics -------------------------------------------------------
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
H, U = rr[0], rr[1]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9,
         "msecond": 1e6, "second": 1e9}
want = {
    "gpu__time_duration.sum": "duration (ns)",
    "dram__bytes_read.sum": "DRAM read (B)",
    "dram__bytes_write.sum": "DRAM write (B)",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "registers/thread",
    "launch__occupancy_limit_registers": "CTA limit (registers)",
    "launch__occupancy_limit_shared_mem": "CTA limit (smem)",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps active %",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue active %",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "SM throughput %",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "memory throughput %",
    "lts__t_sector_hit_rate.pct": "L2 hit %",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "FMA pipe active %",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "ALU pipe active %",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "LSU pipe %",
}
kern = collections.OrderedDict()
for r in rr[2:]:
    if len(r) != len(H):
        continue
    name = r[H.index("Kernel Name")].split("(")[0].replace("void ", "")
    m = {}
    for key in want:
        if key in H:
            i = H.index(key)
            try:
                m[key] = float(r[i].replace(",", "")) * SCALE.get(U[i], 1)
            except ValueError:
                m[key] = r[i]
    kern.setdefault(name.split("<")[0], m)

with open(out_md, "w") as f:
    f.write(f"# ncu evidence — {config}\n\n{note}\n\n")
    f.write("## Launch list (`--metrics gpu__time_duration.sum --clock-control none`; "
            "cold-cache and serialised by ncu — compare shares, not absolutes)\n\n")
    f.write("| kernel | launches | total ms | ms / launch | share |\n|---|---|---|---|---|\n")
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        f.write(f"| {k} | {n} | {v / 1e6:.3f} | {v / 1e6 / n:.3f} | {100 * v / tot:.1f}% |\n")
    f.write("\n## Full-set metrics (`--set full --clock-control none`, one launch each)\n\n")
    names = list(kern)
    f.write("| metric | " + " | ".join(names) + " |\n|---|" + "---|" * len(names) + "\n")
    for key, label in want.items():
        vals = []
        for k in names:
            v = kern[k].get(key, "")
            vals.append(f"{v:,.0f}" if isinstance(v, float) and v >= 100 else
                        (f"{v:.1f}" if isinstance(v, float) else str(v)))
        f.write(f"| {label} | " + " | ".join(vals) + " |\n")
print(open(out_md).read())

js = "profiles/ncu_summary.json"
d = json.load(open(js)) if os.path.exists(js) else {}
d[config] = {k: {"dram_bytes_per_launch": m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0),
                 "duration_ns": m.get("gpu__time_duration.sum"), "clouds_per_launch": clouds_per_launch,
                 "source": os.path.basename(out_md)} for k, m in kern.items()}
# bench.py times the page decode as one event pair around k_page_decode +
# k_page_matches: its traffic is the pair's
if "k_page_decode" in d[config] and "k_page_matches" in d[config]:
    a, b = d[config]["k_page_decode"], d[config]["k_page_matches"]
    d[config]["k_page_decode+k_page_matches"] = {
        "dram_bytes_per_launch": a["dram_bytes_per_launch"] + b["dram_bytes_per_launch"],
        "duration_ns": (a["duration_ns"] or 0) + (b["duration_ns"] or 0),
        "clouds_per_launch": clouds_per_launch, "source": os.path.basename(out_md)}
json.dump(d, open(js, "w"), indent=1)
