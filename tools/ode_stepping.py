"""Raman ODE step-size policy: reference restart vs continuous stepping.

For the bench workload (and 75/0.95): ODE device ms and RHS count in both
modes, and the deviation of the continuous mode from the restart mode (max
|d log rho| via eta/SNR of the full evaluation) plus, for the golden cases,
from the reference's own outputs (tests/golden/golden.json).

    python tools/ode_stepping.py [--out gpurun_out/ode_stepping.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_18022_b200 as uwb  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--out", default=None)
a = p.parse_args()
eng = uwb.Engine(0)


def run(grid, n_r, dens, mode, reps=5):
    eng.set_ode_stepping(mode)
    res = uwb.ResidentLink(uwb.default_fibre(), grid,
                           uwb.LinkConfig(gn=uwb.GnSolverConfig(n_r=n_r, mean_step_density=dens)),
                           engine=eng)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    psd = torch.tensor(grid.psd, dtype=torch.float64, device="cuda:0")
    rep = torch.zeros(res.report_len, dtype=torch.float64, device="cuda:0")
    ts, os_ = [], []
    for i in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        res.run(psd.data_ptr(), rep.data_ptr(), st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        if i:
            ts.append(e0.elapsed_time(e1))
            os_.append(eng.last_ode_stats())
    res.check_status()
    n = grid.size()
    r = rep.cpu().numpy()
    eng.set_ode_stepping("restart")
    return {"eval_ms": float(np.median(ts)), "ode_ms": float(np.median([o["ode_ms"] for o in os_])),
            "rhs": os_[-1]["rhs_evals"], "eta": r[:n], "snr": r[2 * n:3 * n]}


rows = []
g589 = uwb.make_default_uwb_grid()
uwb.set_uniform_launch(g589, 1e-3)
for n_r, dens in ((150, 1.4), (75, 0.95)):
    rs = run(g589, n_r, dens, "restart")
    cs = run(g589, n_r, dens, "continuous")
    act = rs["eta"] > 0
    row = {"workload": f"uwb589 {n_r}/{dens}", "restart_ode_ms": rs["ode_ms"], "restart_rhs": rs["rhs"],
           "continuous_ode_ms": cs["ode_ms"], "continuous_rhs": cs["rhs"],
           "restart_eval_ms": rs["eval_ms"], "continuous_eval_ms": cs["eval_ms"],
           "max_rel_eta_vs_restart": float(np.max(np.abs(cs["eta"][act] / rs["eta"][act] - 1))),
           "max_abs_dsnr_db_vs_restart": float(np.max(np.abs(cs["snr"][act] - rs["snr"][act])))}
    rows.append(row)
    print(json.dumps(row), flush=True)

# against the reference's own evaluate_link outputs
from pyoracle import Case  # noqa: E402
from helpers import cfg_of, product_scenario  # noqa: E402

with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as fh:
    golden = json.load(fh)
for name, rec in golden["evaluate_link"].items():
    case = Case.from_json(rec["case"])
    grid, fibre = product_scenario(case)
    lc = uwb.LinkConfig(gn=cfg_of(case), raman=uwb.RamanSolveOptions(bool(case.raman)))
    out = {}
    for mode in ("restart", "continuous"):
        eng.set_ode_stepping(mode)
        rep = uwb.evaluate_link(fibre, grid, lc, engine=eng)
        eta_ref = np.array(rec["eta"])
        act = eta_ref > 0
        out[mode] = {"max_rel_eta_vs_reference": float(np.max(np.abs(rep.eta[act] / eta_ref[act] - 1))),
                     "max_abs_dsnr_db_vs_reference": float(np.max(np.abs(rep.snr_db[act] - np.array(rec["snr_db"])[act])))}
    eng.set_ode_stepping("restart")
    row = {"golden": name, **{f"{m}_{k}": v for m, d in out.items() for k, v in d.items()}}
    rows.append(row)
    print(json.dumps(row), flush=True)
if a.out:
    with open(a.out, "w") as fh:
        json.dump({"rows": rows}, fh, indent=1)
