"""BASELINE config 4: integration-grid resolution sweep on the 589-ch plan.

For N_R x N_M-density settings: device time of one full SNR evaluation
(ResidentLink, median of 3, CUDA events) and the NLI accuracy against the
(N_R=500, density 2.0) evaluation of the same engine (max / mean |d eta| in dB
over active channels) -- the accuracy-vs-time trade-off of PAPER.md:126.
Each setting also runs the compensated-FP32 integrand ("mixed",
uwb_set_precision): its time and its max relative eta deviation from the FP64
evaluation at the same setting (the "FP64 vs compensated FP32" column).

    python tools/sweep.py [--out profiles/r01_config4_sweep.json]
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
p.add_argument("--out", default=None)
p.add_argument("--n-r", default="25,50,75,100,150,250,500")
p.add_argument("--density", default="0.5,0.95,1.4,2.0")
a = p.parse_args()
eng = uwb.Engine(0)
grid = uwb.make_default_uwb_grid()
uwb.set_uniform_launch(grid, 1e-3)
fibre = uwb.default_fibre()
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
psd = torch.tensor(grid.psd, dtype=torch.float64, device="cuda:0")
n = grid.size()


def run(nr, dens, precision="fp64"):
    eng.set_precision(precision)
    res = uwb.ResidentLink(fibre, grid, uwb.LinkConfig(gn=uwb.GnSolverConfig(n_r=nr, mean_step_density=dens)),
                           engine=eng)
    rep = torch.zeros(res.report_len, dtype=torch.float64, device="cuda:0")
    ts = []
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        res.run(psd.data_ptr(), rep.data_ptr(), st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res.check_status()
    s = eng.last_nli_stats()
    return float(np.median(ts[1:])), rep[:n].cpu().numpy(), s


t_ref, eta_ref, _ = run(500, 2.0)
act = eta_ref > 0
rows = []
for nr in [int(x) for x in a.n_r.split(",")]:
    for dens in [float(x) for x in a.density.split(",")]:
        t, eta, s = run(nr, dens)
        d = np.abs(10 * np.log10(eta[act] / eta_ref[act]))
        tm, eta_m, sm = run(nr, dens, "mixed")
        rel_m = np.abs(eta_m[act] - eta[act]) / eta[act]
        rows.append({"n_r": nr, "density": dens, "eval_ms": t, "nli_kernel_ms": s["kernel_ms"],
                     "evaluated_points": s["evaluated_points"], "active_points": s["active_points"],
                     "max_abs_deta_db": float(d.max()), "mean_abs_deta_db": float(d.mean()),
                     "mixed_eval_ms": tm, "mixed_nli_kernel_ms": sm["kernel_ms"],
                     "mixed_max_rel_eta_vs_fp64": float(rel_m.max()),
                     "mixed_max_abs_deta_db_vs_fp64": float(np.max(np.abs(10 * np.log10(eta_m[act] / eta[act]))))})
        print(json.dumps(rows[-1]), flush=True)
out = {"reference_setting": {"n_r": 500, "density": 2.0, "eval_ms": t_ref}, "rows": rows,
       "workload": "589ch O-U, 80 km, 0 dBm/ch, ISRS on; accuracy vs this engine at (500, 2.0)"}
if a.out:
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=1)
