"""Throughput of uwb_evaluate_link_many (the optimiser's batched cost calls):
n_eval random launch profiles of the 589-ch plan, wall time per evaluation.

    python tools/time_batch.py [--n-eval 56] [--n-r 150] [--density 1.4]
UWB_BATCH_SERIAL=1 disables the ODE/NLI overlap for comparison.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2401_18022_b200 as uwb  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n-eval", type=int, default=56)
p.add_argument("--n-r", type=int, default=150)
p.add_argument("--density", type=float, default=1.4)
p.add_argument("--interleave", type=int, default=0,
               help="batches of n_eval, each preceded by one single evaluation (the optimiser's "
                    "value + gradient pattern); 0 = one batch")
a = p.parse_args()
eng = uwb.Engine(0)
grid = uwb.make_default_uwb_grid()
uwb.set_uniform_launch(grid, 1e-3)
res = uwb.ResidentLink(uwb.default_fibre(), grid,
                       uwb.LinkConfig(gn=uwb.GnSolverConfig(n_r=a.n_r, mean_step_density=a.density)),
                       engine=eng)
rng = np.random.default_rng(20240131)
base = np.asarray(grid.psd)
psd = np.stack([base * 10 ** (rng.uniform(-0.5, 0.5, base.size) / 10) for _ in range(a.n_eval)])
res.run_many(psd[:2])
if a.interleave:
    t0 = time.perf_counter()
    for _ in range(a.interleave):
        res.run_many(psd[:1])
        loss, reps = res.run_many(psd, reports=True)
    dt = (time.perf_counter() - t0) / a.interleave
else:
    t0 = time.perf_counter()
    loss, reps = res.run_many(psd, reports=True)
    dt = time.perf_counter() - t0
print(json.dumps({"n_eval": a.n_eval, "interleave": a.interleave, "n_r": a.n_r, "density": a.density, "wall_s": dt,
                  "ms_per_eval": dt / a.n_eval * 1e3, "serial": os.environ.get("UWB_BATCH_SERIAL", "0"),
                  "loss_sum": float(np.sum(loss)), "eta_sum": float(np.sum(reps[:, :grid.size()]))}))
