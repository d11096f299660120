"""Summarise an ncu launch list (--csv --metrics gpu__time_duration.sum[,dram__bytes_*]):
per kernel name: launches, total / mean duration, DRAM bytes.
Usage: python tools/launch_summary.py launches.csv"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
iid, ik, im, iv = hdr.index("ID"), hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
per = defaultdict(dict)
names = {}
for r in rows[1:]:
    per[r[iid]][r[im]] = float(r[iv].replace(",", "") or 0)
    names[r[iid]] = r[ik].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]
agg = defaultdict(lambda: [0, 0.0, 0.0])
for i, m in per.items():
    a = agg[names[i]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':28s} {'n':>5s} {'total ms':>10s} {'share':>6s} {'mean us':>9s} {'DRAM MB':>10s}")
for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:28s} {n:5d} {t / 1e6:10.3f} {t / tot:6.3f} {t / n / 1e3:9.1f} {b / 1e6:10.1f}")
print(f"{'TOTAL':28s} {sum(a[0] for a in agg.values()):5d} {tot / 1e6:10.3f}")
