"""Short driver for ncu on the device Raman ODE alone: a few
solve_power_evolution calls on one comb.

    python tools/profile_ode.py [--grid uwb589|cband11] [--density 1.4] [--iters 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2401_18022_b200 as uwb  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--grid", default="uwb589", choices=["uwb589", "cband11"])
p.add_argument("--density", type=float, default=1.4)
p.add_argument("--iters", type=int, default=2)
a = p.parse_args()
eng = uwb.Engine(0)
if a.grid == "uwb589":
    grid = uwb.make_default_uwb_grid()
else:
    grid = uwb.make_uniform_grid(11, 100e9, 96e9, 299792458.0 / 1550e-9)
uwb.set_uniform_launch(grid, 1e-3)
fibre = uwb.default_fibre()
zg = uwb.build_distance_grid(fibre.length_m, a.density)
for _ in range(a.iters):
    evo = uwb.solve_power_evolution(fibre, grid, zg, engine=eng)
print("rho_end[0]", evo.rho_end[0])
