"""A/B timing of the integrand: median device time of nli_rows over R full
evaluations of the bench workload, plus an eta checksum (variants must agree).

    UWB_LIB_PATH=scratch/v/x.so python tools/time_nli.py [--n-r 150] [--density 1.4] [--reps 7]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_18022_b200 as uwb  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n-r", type=int, default=150)
p.add_argument("--density", type=float, default=1.4)
p.add_argument("--reps", type=int, default=7)
p.add_argument("--tag", default=os.environ.get("UWB_LIB_PATH", "main"))
p.add_argument("--grid", default="uwb589", choices=["uwb589", "oband11", "cband11"])
p.add_argument("--precision", default="fp64", choices=["fp64", "mixed"])
a = p.parse_args()
eng = uwb.Engine(0)
eng.set_precision(a.precision)
if a.grid == "uwb589":
    grid = uwb.make_default_uwb_grid()
    uwb.set_uniform_launch(grid, 1e-3)
else:  # BASELINE configs 1/2: 11 x 96 GBd, 100 GHz, at 1550 nm (0 dBm) / 1302.3 nm (2 dBm)
    lam, dbm = (1550e-9, 0.0) if a.grid == "cband11" else (1302.3e-9, 2.0)
    grid = uwb.make_uniform_grid(11, 100e9, 96e9, 299792458.0 / lam)
    uwb.set_uniform_launch(grid, 1e-3 * 10 ** (dbm / 10))
res = uwb.ResidentLink(uwb.default_fibre(), grid,
                       uwb.LinkConfig(gn=uwb.GnSolverConfig(n_r=a.n_r, mean_step_density=a.density)),
                       engine=eng)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
psd = torch.tensor(grid.psd, dtype=torch.float64, device="cuda:0")
rep = torch.zeros(res.report_len, dtype=torch.float64, device="cuda:0")
ks, ts, os_ = [], [], []
for i in range(a.reps + 2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    res.run(psd.data_ptr(), rep.data_ptr(), st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    if i >= 2:
        st_ = eng.last_nli_stats()
        ks.append(st_["kernel_ms"])
        os_.append(eng.last_ode_stats())
        ts.append(e0.elapsed_time(e1))
res.check_status()
n = grid.size()
eta = rep[:n].cpu().numpy()
print(json.dumps({"tag": a.tag, "grid": a.grid, "n_r": a.n_r, "density": a.density,
                  "nli_ms": float(np.median(ks)),
                  "evaluated": st_["evaluated_points"], "active": st_["active_points"],
                  "ode_ms": float(np.median([o["ode_ms"] for o in os_])),
                  "ode_rhs": os_[-1]["rhs_evals"],
                  "ode_us_per_rhs": float(np.median([o["ode_ms"] for o in os_])) * 1e3 / max(1, os_[-1]["rhs_evals"]), "eval_ms": float(np.median(ts)),
                  "eta_sum": float(np.sum(eta)), "eta_max": float(np.max(eta)),
                  "loss": float(rep[4 * n].item())}), flush=True)
