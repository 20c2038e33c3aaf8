"""Full SASS listing of an ncu report with stall samples per instruction and
the top stall reasons, for reading a latency-bound kernel's critical path.

    python tools/ncu_listing.py report.ncu-rep > listing.txt
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h, body = rows[hi], rows[hi + 1:]
ci = {k: i for i, k in enumerate(h)}
samp = next(k for k in h if k.startswith("Warp Stall Sampling (All"))
stall_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
for r in body:
    if len(r) != len(h):
        continue
    s = float(r[ci[samp]] or 0)
    ex = r[ci["Instructions Executed"]]
    st = sorted(((float(r[ci[k]] or 0), k[6:]) for k in stall_cols), reverse=True)[:2]
    why = " ".join(f"{n}:{v:.0f}" for v, n in st if v > 0)
    print(f"{r[ci['Address']][-5:]} {s:6.0f} {ex:>8s}  {r[ci['Source']].strip()[:60]:60s} {why}")
