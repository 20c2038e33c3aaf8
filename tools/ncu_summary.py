"""Summarise an ncu report: key throughput metrics, stall reasons, SASS mix.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [steps_per_launch] [kernel-regex]
"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
steps = float(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
kfilt = ["--kernel-name", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []


def page(*args):
    out = subprocess.run(["ncu", "-i", rep, *kfilt, *args, "--csv"], capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))


raw = page("--page", "raw")
h, u, v = raw[0], raw[1], raw[2]
m = dict(zip(h, v))
keys = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_requests_pipe_lsu_mem_local_op_ld.sum", "smsp__inst_executed.sum"]
for k in keys:
    if k in m:
        print(f"{k:80s} {m[k]}")
stalls = {k: float(v2) for k, v2 in m.items()
          if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")
          and v2 not in ("", "n/a")}
if not stalls:
    stalls = {k: float(v2) for k, v2 in m.items()
              if "warp_issue_stalled" in k and k.endswith("per_warp_active.pct") and v2 not in ("", "n/a")}
print("-- stall reasons (top)")
for k, val in sorted(stalls.items(), key=lambda kv: -kv[1])[:10]:
    print(f"   {k:90s} {val:8.2f}")
src = page("--page", "source", "--print-source", "sass")
# one section per profiled kernel: a name row, then a header row starting "Address"
hi = next(i for i, r in enumerate(src) if r and r[0] == "Address")
hh = src[hi]
rows = []
for r in src[hi + 1:]:
    if r and r[0] == "Address":
        break  # the next kernel's section
    if len(r) == len(hh):
        rows.append(dict(zip(hh, r)))
tot = sum(int(r["Instructions Executed"]) for r in rows)
c = Counter()
for r in rows:
    t = r["Source"].strip().split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    c[op.split(".")[0]] += int(r["Instructions Executed"])
den = steps / 32 if steps else 1.0
print(f"-- SASS warp instructions: {tot}" + (f" = {tot/den:.1f} per warp-step" if steps else ""))
for op, n in c.most_common(22):
    print(f"   {op:10s} {n/den:10.2f}")
