"""Warp-stall samples of an ncu SASS source dump (--page source --csv
--print-source sass) per CUDA source line, using nvdisasm -g line info of the
same build.  Usage:
  python tools/sass_lines.py dump.csv lib.so kernel_substring [n_top]
(the .so must be the build that ran under ncu)."""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

dump, so, kname = sys.argv[1:4]
n_top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
rows = list(csv.reader(open(dump)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
S = hdr.index("Warp Stall Sampling (All Samples)")
if os.environ.get("METRIC"):  # e.g. METRIC="Instructions Executed"
    S = hdr.index(os.environ["METRIC"])
base = int(data[0][0], 16)
samples = {int(r[0], 16) - base: int(r[S] or 0) for r in data}
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
reasons = {int(r[0], 16) - base: [(int(r[i]), hdr[i][6:]) for i in stall_cols if r[i].isdigit() and int(r[i]) > 0]
           for r in data}

tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
text = None
for f in sorted(os.listdir(tmp)):
    if f.endswith(".cubin"):
        out = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, f)], capture_output=True, text=True).stdout
        if kname in out:
            text = out
            break
if text is None:
    sys.exit(f"{kname} not found in {so}")
line = None
infn = False
per_line = defaultdict(int)
per_reason = defaultdict(lambda: defaultdict(int))
for ln in text.splitlines():
    if ln.startswith("//---") or ln.startswith(".text."):
        infn = kname in ln
        continue
    if not infn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m and line:
        off = int(m.group(1), 16)
        per_line[line] += samples.get(off, 0)
        for c, name in reasons.get(off, []):
            per_reason[line][name] += c
tot = sum(samples.values())
print("total samples", tot)
src_cache = {}
for key, v in sorted(per_line.items(), key=lambda x: -x[1])[:n_top]:
    f, no = key.split(":")
    path = next((p for p in (os.path.join("paper_2603_16945_b200/csrc", f),) if os.path.exists(p)), None)
    if path and path not in src_cache:
        src_cache[path] = open(path).read().splitlines()
    src = src_cache[path][int(no) - 1].strip()[:70] if path else ""
    top = sorted(((c, n) for n, c in per_reason[key].items()), reverse=True)[:2]
    print(f"{key:22s} {v:7d} {100 * v / max(1, tot):5.1f}%  {src:70s} {top}")
