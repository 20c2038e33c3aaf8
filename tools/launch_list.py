"""Per-kernel launch list from `ncu --metrics gpu__time_duration.sum --csv --log-file X.csv`:
launches, total and per-launch time, share of the total (the dfma_peak microbenchmark
excluded from the shares).

    python tools/launch_list.py launches.csv
"""
import csv
import re
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
ci = {k: i for i, k in enumerate(h)}
agg = OrderedDict()
for r in rows[1:]:
    if r[ci["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*$", "", r[ci["Kernel Name"]])
    name = re.sub(r"^(void )?(uwb::)?(<unnamed>::)?", "", name)
    v = float(r[ci["Metric Value"]].replace(",", ""))
    unit = r[ci["Metric Unit"]]
    ms = v * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1e-6)
    n, t = agg.get(name, (0, 0.0))
    agg[name] = (n + 1, t + ms)
tot = sum(t for k, (n, t) in agg.items() if "dfma_peak" not in k)
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    share = "" if "dfma_peak" in k else f"share {100 * t / tot:5.1f} %"
    print(f"{k[:60]:60s} launches {n:4d}  total {t:9.3f} ms  per launch {t / n:8.4f} ms  {share}")
