"""The FP64 roofline denominator, with the clocks it was measured at:
uwb_fp64_peak (independent DFMA chains on every SM, CUDA events, best of 3
after a warm-up) repeated R times while nvidia-smi samples the SM clock.

    python tools/fp64_peak.py [--reps 20] > profiles/r02_fp64_peak.json
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2401_18022_b200 as uwb  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--reps", type=int, default=20)
a = p.parse_args()
eng = uwb.Engine(0)
info = eng.device_info()
lines = []
proc = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,clocks.max.sm,power.draw",
                         "--format=csv,noheader,nounits", "-lms", "50"],
                        stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
t = threading.Thread(target=lambda: [lines.append(x.strip()) for x in proc.stdout], daemon=True)
t.start()
time.sleep(0.3)
vals = [eng.fp64_peak_tflops() for _ in range(a.reps)]
time.sleep(0.2)
proc.terminate()
sm = []
mx = 0.0
for ln in lines:
    f = [x.strip() for x in ln.split(",")]
    try:
        sm.append(float(f[0]))
        mx = max(mx, float(f[1]))
    except (ValueError, IndexError):
        pass
sm_sorted = sorted(sm)
med = sm_sorted[len(sm_sorted) // 2] if sm else None
nominal = info["sm_count"] * 128 * (mx or 1965.0) * 1e6 / 1e12
print(json.dumps({
    "what": "FP64 DFMA peak of this B200 (uwb_fp64_peak: 148 x 8 CTAs x 256 threads, 8 independent "
            "DFMA chains per thread, CUDA events, best of 3 after a warm-up), repeated",
    "tflops": vals, "tflops_max": max(vals), "tflops_median": sorted(vals)[len(vals) // 2],
    "sm_count": info["sm_count"], "sm_mhz_median": med, "sm_max_mhz": mx or None,
    "clock_samples": len(sm),
    "nominal_tflops_at_max_clock": nominal,
    "fraction_of_nominal": max(vals) / nominal}, indent=1))
eng.close()
