"""Attribute ncu per-instruction counts to CUDA source lines.

    python tools/sass_lines.py <cubin> <kernel-substring> <ncu sass csv> <src.cu> [units]

<ncu sass csv> = `ncu -i rep --page source --csv --print-source sass`.  The
cubin must be the one the report was taken with (compile with -lineinfo).
Lines are inlined-callee lines of `src.cu` (other files are grouped by name).
"""
import csv
import re
import subprocess
import sys
from collections import defaultdict

cubin, kern, sass_csv, src = sys.argv[1:5]
units = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
txt = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout.splitlines()
start = next(i for i, l in enumerate(txt) if l.startswith("//---") and kern in l and ".text." in l)
idx2 = []
cur = ("?", 0)
for l in txt[start + 1:]:
    if l.startswith("//---") and ".text." in l:
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if re.match(r"\s*/\*[0-9a-f]{4,6}\*/", l):
        idx2.append(cur)
rows = list(csv.reader(open(sass_csv)))
h = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] in ("Kernel Name", "Address"):
        break  # the next kernel's section
    if len(r) == len(h):
        data.append(dict(zip(h, r)))
agg = defaultdict(float)
stall = defaultdict(float)
for i, d in enumerate(data):
    key = idx2[i] if i < len(idx2) else ("?", 0)
    agg[key] += int(d["Instructions Executed"])
    stall[key] += int(d["Warp Stall Sampling (All Samples)"])
srcl = open(src).read().splitlines()
base = src.split("/")[-1]
tot_st = sum(stall.values()) or 1
print(f"instructions {sum(agg.values())/units:.1f} per unit; {len(idx2)} SASS / {len(data)} rows")
for key, v in sorted(agg.items(), key=lambda kv: -kv[1])[:45]:
    f, ln = key
    s = srcl[ln - 1].strip()[:78] if f == base and 0 < ln <= len(srcl) else f
    print(f"{v/units:8.2f}  stall {stall[key]/tot_st*100:5.1f}%  L{ln:4d} {s}")
