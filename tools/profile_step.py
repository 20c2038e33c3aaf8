"""Short driver for ncu: a few full SNR evaluations of the bench workload.

    python tools/profile_step.py [--n-r 150] [--density 1.4] [--iters 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_18022_b200 as uwb  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n-r", type=int, default=150)
p.add_argument("--density", type=float, default=1.4)
p.add_argument("--iters", type=int, default=3)
p.add_argument("--precision", default="fp64", choices=["fp64", "mixed"])
a = p.parse_args()
eng = uwb.Engine(0)
eng.set_precision(a.precision)
grid = uwb.make_default_uwb_grid()
uwb.set_uniform_launch(grid, 1e-3)
res = uwb.ResidentLink(uwb.default_fibre(), grid,
                       uwb.LinkConfig(gn=uwb.GnSolverConfig(n_r=a.n_r, mean_step_density=a.density)),
                       engine=eng)
torch.cuda.set_stream(torch.cuda.Stream())
psd = torch.tensor(grid.psd, dtype=torch.float64, device="cuda:0")
rep = torch.zeros(res.report_len, dtype=torch.float64, device="cuda:0")
for _ in range(a.iters):
    res.run(psd.data_ptr(), rep.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
res.check_status()
print("loss", rep[4 * grid.size()].item(), "stats", eng.last_nli_stats())
