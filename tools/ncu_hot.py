"""Summarise an ncu --page source --csv (SASS) dump: top instructions by
warp-stall samples with their leading stall reasons, plus sample share per
4 KiB code block.  Usage: python tools/ncu_hot.py dump.csv [n_top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
S = hdr.index("Warp Stall Sampling (All Samples)")
I = hdr.index("Instructions Executed")
tot = sum(int(r[S] or 0) for r in data)
print("total samples", tot)
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for r in sorted(data, key=lambda r: -int(r[S] or 0))[:n]:
    st = sorted([(int(r[i]), hdr[i][6:]) for i in stall_cols if r[i].isdigit() and int(r[i]) > 0], reverse=True)[:3]
    print(r[0][-5:], r[S].rjust(6), r[I].rjust(10), r[1].strip()[:48].ljust(48), st)
blk = defaultdict(int)
for r in data:
    blk[int(r[0], 16) >> 12] += int(r[S] or 0)
print("by 4K block:", [(hex(a << 12)[-5:], round(100 * v / tot, 1)) for a, v in sorted(blk.items(), key=lambda x: -x[1])[:8]])
