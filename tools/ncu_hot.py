"""Hottest SASS instructions of an ncu report (source page, stall samples).

    python tools/ncu_hot.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
# the first row names the kernel; the header row starts with "Address"
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h, body = rows[hi], rows[hi + 1:]
print("columns:", h)
ci = {k: i for i, k in enumerate(h)}
samp = next(k for k in h if k.startswith("Warp Stall Sampling (All"))
recs = [r for r in body if len(r) == len(h)]
tot = sum(float(r[ci[samp]] or 0) for r in recs)
print("total samples", tot)
for r in sorted(recs, key=lambda r: -float(r[ci[samp]] or 0))[:top]:
    print(f"{r[ci['Address']]:>8s} {float(r[ci[samp]] or 0):8.0f} {r[ci['Source']][:90]}")
