"""Small workloads that exercise every device kernel, for compute-sanitizer
(memcheck / racecheck / synccheck), one tool per run:

    compute-sanitizer --tool racecheck python tools/sanitize_case.py

Covers: the integrand (one- and multi-span, Simpson, symmetric and direct
quadrants), the probe / finalize kernels, the Raman ODE on a one-warp comb
(11 ch) and a four-warp comb (589 ch), the link report kernels, the
overlapped batch (second ODE stream) and a multi-context split evaluation."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2401_18022_b200 as uwb  # noqa: E402

C0 = 299792458.0
eng = uwb.Engine(0)
fibre = uwb.default_fibre()

# 11-ch C-band, N_R 24 (the verdict's case), full evaluation + Simpson NLI
g = uwb.make_uniform_grid(11, 100e9, 96e9, C0 / 1550e-9)
uwb.set_uniform_launch(g, 1e-3)
lc = uwb.LinkConfig(gn=uwb.GnSolverConfig(n_r=24, mean_step_density=0.95))
r = uwb.evaluate_link(fibre, g, lc, engine=eng)
zg = uwb.build_distance_grid(fibre.length_m, 0.95)
evo = uwb.solve_power_evolution(fibre, g, zg, engine=eng)
betas = uwb.beta_from_dispersion(fibre, C0 / g.centre)
cfg = uwb.GnSolverConfig(n_r=24, mean_step_density=0.95, simpson_channel_average=True)
s = uwb.all_channels_nli(g, [evo, evo], betas, fibre, cfg, engine=eng)
cfg2 = uwb.GnSolverConfig(n_r=17, mean_step_density=0.95, mirror_q4=False)
s2 = uwb.all_channels_nli(g, [evo], betas, fibre, cfg2, engine=eng)

# 589 ch: the four-warp ODE and the resident / batch paths on a coarse grid
G = uwb.make_default_uwb_grid()
uwb.set_uniform_launch(G, 1e-3)
lc2 = uwb.LinkConfig(gn=uwb.GnSolverConfig(n_r=6, mean_step_density=0.1))
res = uwb.ResidentLink(fibre, G, lc2, engine=eng)
prof = np.stack([np.array(G.psd), np.array(G.psd) * 1.1])
loss = res.run_many(prof)

# multi-context split (two contexts on this GPU)
m = uwb.Engine(devices=[0, 0])
rm = uwb.evaluate_link(fibre, g, lc, engine=m)
assert np.array_equal(rm.eta, r.eta)
m.close()
eng.close()
print("sanitize case OK", float(r.loss_value), float(s.eta[5]), float(s2.eta[5]), loss.tolist())
nl, ol = uwb._native.C.c_int(), uwb._native.C.c_int()
uwb._native.load().uwb_debug_bounds(uwb._native.C.byref(nl), uwb._native.C.byref(ol))
print("bounds check: integrand first failing line", nl.value, "| ODE", ol.value,
      "(0 = clean, -1 = not a bounds-checked build)")
