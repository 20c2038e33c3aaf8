"""Parity pinned on EXACTLY the benchmarked configuration: the 589-ch O->U plan
at N_R = 150, N_M density 1.4 /km (bench.py's workload), at 0 dBm/ch and at
the config-5 random launch profile.

Fixtures: tests/golden/golden_headline.{npz,json}, written by
tests/golden/make_golden_headline.py from the UNMODIFIED reference
(oracle/_ref/libuwbref.so): full evaluate_link reports and the full 65,968-entry
log_rho table of solve_power_evolution.

Tolerances: eta 1e-9 relative, SNR 1e-8 dB, loss / capacity 1e-9 relative,
log rho 1e-9 absolute (BASELINE north star: 1e-6 eta, 0.01 dB).
"""
import json
import os

import numpy as np
import pytest

from pyoracle import Case

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = ["uwb589_150_1.4", "uwb589_150_1.4_random"]


@pytest.fixture(scope="module")
def headline():
    arr = np.load(os.path.join(HERE, "golden", "golden_headline.npz"))
    with open(os.path.join(HERE, "golden", "golden_headline.json")) as fh:
        meta = json.load(fh)
    return arr, meta


def _rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    den = np.where(b == 0, 1.0, np.abs(b))
    return float(np.max(np.abs(a - b) / den)) if a.size else 0.0


# ------------------------------------------------------------------ CPU
def test_headline_fixture_is_consistent(headline, golden):
    """The two independently written fixtures agree bit for bit where they
    overlap: evaluate_link's eta at 150/1.4, 0 dBm == all_channels_nli's eta
    of golden.json (same reference, same inputs)."""
    arr, meta = headline
    np.testing.assert_array_equal(arr["uwb589_150_1.4/eta"],
                                  np.array(golden["all_channels_nli"]["uwb589_150_1.4"]["eta"]))
    assert arr["uwb589_150_1.4/log_rho"].size == 589 * 112
    for c in CASES:
        assert meta["power_evolution"][c]["steps"] == 112
        assert meta["evaluate_link"][c]["case"]["n_r"] == 150


@pytest.mark.parametrize("name", CASES)
def test_oracle_power_evolution_full_table(name, headline, oracle):
    """The C restatement's ODE reproduces the reference's FULL log_rho table of
    the benchmarked plan bit for bit (the previous fixture kept 64 samples)."""
    arr, meta = headline
    case = Case.from_json(meta["power_evolution"][name]["case"])
    r = oracle.power_evolution(case)
    np.testing.assert_array_equal(r["log_rho"], arr[f"{name}/log_rho"])
    np.testing.assert_array_equal(r["rho_end"], arr[f"{name}/rho_end"])


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_evaluate_link_headline_config(name, headline, engine):
    """Device ODE + NLI + SNR assembly in ONE public call (uwb_evaluate_link)
    against the reference's evaluate_link at the bench configuration."""
    import paper_2401_18022_b200 as uwb
    from helpers import cfg_of, product_scenario

    arr, meta = headline
    m = meta["evaluate_link"][name]
    case = Case.from_json(m["case"])
    grid, fibre = product_scenario(case)
    lc = uwb.LinkConfig(gn=cfg_of(case), raman=uwb.RamanSolveOptions(True))
    rep = uwb.evaluate_link(fibre, grid, lc, engine=engine)
    eta = arr[f"{name}/eta"]
    act = eta > 0
    assert np.array_equal(rep.eta > 0, act)
    assert _rel(rep.eta[act], eta[act]) < 1e-9
    assert np.max(np.abs(rep.snr_db[act] - arr[f"{name}/snr_db"][act])) < 1e-8
    assert _rel(rep.p_ase[act], arr[f"{name}/p_ase"][act]) < 1e-9
    assert _rel(rep.capacity[act], arr[f"{name}/capacity"][act]) < 1e-9
    assert rep.loss_value == pytest.approx(m["loss"], rel=1e-9)
    assert rep.total_capacity == pytest.approx(m["total_capacity"], rel=1e-9)
    assert rep.total_power_dbm == pytest.approx(m["total_power_dbm"], abs=1e-9)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_power_evolution_headline_full_table(name, headline, engine):
    """Device Raman ODE: every one of the 65,968 log_rho entries within 1e-9."""
    import paper_2401_18022_b200 as uwb
    from helpers import product_scenario

    arr, meta = headline
    case = Case.from_json(meta["power_evolution"][name]["case"])
    grid, fibre = product_scenario(case)
    zg = uwb.build_distance_grid(case.length_m, case.density)
    evo = uwb.solve_power_evolution(fibre, grid, zg, uwb.RamanSolveOptions(True), engine=engine)
    np.testing.assert_allclose(evo.log_rho, arr[f"{name}/log_rho"], rtol=0, atol=1e-9)
    np.testing.assert_allclose(evo.rho_end, arr[f"{name}/rho_end"], rtol=1e-9)


@pytest.mark.gpu
def test_resident_batch_at_headline_config(headline, engine):
    """The optimiser's batched path (uwb_evaluate_link_many, ODE overlapped with
    the integrand) at the bench configuration: both golden launch profiles in
    one batch reproduce the reference reports."""
    import paper_2401_18022_b200 as uwb
    from helpers import cfg_of, product_scenario

    arr, meta = headline
    case = Case.from_json(meta["evaluate_link"][CASES[1]]["case"])
    grid, fibre = product_scenario(case)
    lc = uwb.LinkConfig(gn=cfg_of(case))
    res = uwb.ResidentLink(fibre, grid, lc, engine=engine)
    g0, _ = product_scenario(Case.from_json(meta["evaluate_link"][CASES[0]]["case"]))
    psd = np.stack([g0.psd, grid.psd])
    loss, reps = res.run_many(psd, reports=True)
    n = grid.size()
    for k, name in enumerate(CASES):
        eta = arr[f"{name}/eta"]
        act = eta > 0
        assert _rel(reps[k][:n][act], eta[act]) < 1e-9
        assert np.max(np.abs(reps[k][2 * n:3 * n][act] - arr[f"{name}/snr_db"][act])) < 1e-8
        assert loss[k] == pytest.approx(meta["evaluate_link"][name]["loss"], rel=1e-9)
