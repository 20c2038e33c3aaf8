"""Shared test helpers: turn a golden/oracle case into engine inputs."""
from __future__ import annotations

import numpy as np

import paper_2401_18022_b200 as uwb
from pyoracle import KC0, Case


def to_db(x):
    return 10.0 * np.log10(x)


def engine_inputs_from_oracle(prep, density):
    """Engine-side objects built from the ORACLE's inputs (grid, log_rho,
    betas, gamma), so NLI parity is isolated from the input builders."""
    ga = prep["grid_arrays"]
    grid = uwb.ChannelGrid(ga["freq"].copy(), ga["psd"].copy(), ga["guard"].copy(), ga["spacing"],
                           ga["bch"], ga["centre"], ga["half_band"])
    spans = []
    for s in prep["spans"]:
        zg = uwb.DistanceGrid(s["edge"], s["mid"], s["width"], s["length"], density)
        spans.append(uwb.PowerEvolution(zg, ga["freq"], ga["psd"] * ga["bch"], s["log_rho"],
                                        prep["rho_end"], ga["spacing"]))
    return grid, spans, uwb.BetaCoefficients(*prep["betas"]), np.asarray(prep["gamma"])


def cfg_of(case: Case):
    return uwb.GnSolverConfig(n_r=case.n_r, mean_step_density=case.density,
                              u1_sampling=uwb.U1Sampling.kUniform if case.u1_uniform else uwb.U1Sampling.kLog,
                              u1_min_ratio=case.u1_min_ratio,
                              simpson_channel_average=bool(case.simpson),
                              mirror_q4=bool(case.mirror_q4))


def product_scenario(case: Case):
    """The same case assembled ONLY from the product's own builders."""
    if case.uwb_default:
        grid = uwb.make_default_uwb_grid()
    else:
        grid = uwb.make_uniform_grid(case.n_ch, case.spacing, case.bch, case.centre)
    if case.guard is not None:
        grid.guard = np.asarray(case.guard, np.uint8).copy()
    if case.launch_w is not None:
        uwb.set_launch(grid, case.launch_w)
    else:
        uwb.set_uniform_launch(grid, case.uniform_w)
    fibre = (uwb.flat_fibre(case.flat_alpha_db_km, case.length_m, case.span_count)
             if case.fibre_kind == 1 else uwb.FibreSpec(case.length_m, case.span_count))
    return grid, fibre
