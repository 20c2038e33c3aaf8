"""FP64 vs compensated-FP32 ("mixed") integrand: accuracy and time per
workload (BASELINE config 4 column "FP64 vs compensated FP32").

    python tools/mixed_accuracy.py [--out gpurun_out/mixed.json]

For each workload: median integrand ms in both modes, max / median relative
|eta_mixed - eta_fp64| / eta_fp64 over active channels, and the max SNR
difference in dB of the full link report.
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
p.add_argument("--reps", type=int, default=5)
p.add_argument("--quick", action="store_true")
a = p.parse_args()

eng = uwb.Engine(0)


def grid_for(name):
    if name == "uwb589":
        g = uwb.make_default_uwb_grid()
        uwb.set_uniform_launch(g, 1e-3)
        return g
    lam, dbm = (1550e-9, 0.0) if name == "cband11" else (1302.3e-9, 2.0)
    n = 101 if name == "oband101" else 11
    g = uwb.make_uniform_grid(n, 100e9, 96e9, 299792458.0 / lam)
    uwb.set_uniform_launch(g, 1e-3 * 10 ** (dbm / 10))
    return g


def run(name, n_r, dens, mode):
    eng.set_precision(mode)
    grid = grid_for(name)
    res = uwb.ResidentLink(uwb.default_fibre(), grid,
                           uwb.LinkConfig(gn=uwb.GnSolverConfig(n_r=n_r, mean_step_density=dens)),
                           engine=eng)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    psd = torch.tensor(grid.psd, dtype=torch.float64, device="cuda:0")
    rep = torch.zeros(res.report_len, dtype=torch.float64, device="cuda:0")
    ks = []
    for i in range(a.reps + 1):
        res.run(psd.data_ptr(), rep.data_ptr(), st.cuda_stream)
        torch.cuda.synchronize()
        if i:
            ks.append(eng.last_nli_stats()["kernel_ms"])
    res.check_status()
    n = grid.size()
    r = rep.cpu().numpy()
    return {"nli_ms": float(np.median(ks)), "eta": r[:n], "snr_db": r[2 * n:3 * n]}


cases = [("uwb589", 150, 1.4), ("uwb589", 75, 0.95), ("cband11", 150, 1.4), ("oband11", 150, 1.4),
         ("oband101", 150, 1.4), ("uwb589", 500, 2.0)]
if a.quick:
    cases = cases[:2]
rows = []
for name, n_r, dens in cases:
    f = run(name, n_r, dens, "fp64")
    m = run(name, n_r, dens, "mixed")
    act = f["eta"] > 0
    rel = np.abs(m["eta"][act] - f["eta"][act]) / f["eta"][act]
    row = {"workload": name, "n_r": n_r, "density": dens,
           "fp64_nli_ms": f["nli_ms"], "mixed_nli_ms": m["nli_ms"],
           "speedup": f["nli_ms"] / m["nli_ms"],
           "max_rel_eta": float(rel.max()), "median_rel_eta": float(np.median(rel)),
           "max_abs_dsnr_db": float(np.max(np.abs(m["snr_db"][act] - f["snr_db"][act])))}
    rows.append(row)
    print(json.dumps(row), flush=True)
eng.set_precision("fp64")
if a.out:
    with open(a.out, "w") as fh:
        json.dump({"tolerance": {"rel_eta": 1e-6, "snr_db": 0.01}, "rows": rows}, fh, indent=1)
