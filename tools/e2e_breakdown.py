"""Where the host-side part of the e2e evaluation goes (uwb.evaluate_link on
the bench workload): Python-side input marshalling vs the C-ABI call, and
the C-ABI call's device time.

    python tools/e2e_breakdown.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2401_18022_b200 as uwb  # noqa: E402
from paper_2401_18022_b200 import _native as N  # noqa: E402
from paper_2401_18022_b200.gn_integral import _fibre_c, _link_c  # noqa: E402

eng = uwb.Engine(0)
grid = uwb.make_default_uwb_grid()
uwb.set_uniform_launch(grid, 1e-3)
fibre = uwb.default_fibre()
lc = uwb.LinkConfig(gn=uwb.GnSolverConfig(n_r=150, mean_step_density=1.4))
for _ in range(3):
    uwb.evaluate_link(fibre, grid, lc, engine=eng)
T = {"fibre_sample": [], "link_cfg": [], "grid_view": [], "c_call": [], "total": [], "device": []}
for _ in range(10):
    t0 = time.perf_counter()
    fc, keep, _ = _fibre_c(fibre, grid)
    t1 = time.perf_counter()
    lk, keep2 = _link_c(grid, lc, lc.gn)
    t2 = time.perf_counter()
    g, c = grid._c(), lc.gn._c()
    n = grid.size()
    out = {k: np.zeros(n) for k in ("eta", "p_ase", "snr_db", "capacity", "rho_end")}
    bp, bc = np.zeros(6), np.zeros(6)
    rep = N.LinkReportC(*(N.dptr(out[k]) for k in ("eta", "p_ase", "snr_db", "capacity", "rho_end")),
                        N.dptr(bp), N.dptr(bc))
    t3 = time.perf_counter()
    N.check(eng.lib.uwb_evaluate_link(eng.h, N.C.byref(g), N.C.byref(fc), N.C.byref(lk),
                                      N.C.byref(c), N.C.byref(rep)))
    t4 = time.perf_counter()
    T["fibre_sample"].append(t1 - t0)
    T["link_cfg"].append(t2 - t1)
    T["grid_view"].append(t3 - t2)
    T["c_call"].append(t4 - t3)
    T["total"].append(t4 - t0)
    T["device"].append(rep.elapsed_seconds)
print({k: round(float(np.median(v)) * 1e3, 4) for k, v in T.items()}, "ms (medians)")
