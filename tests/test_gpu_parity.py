"""GPU parity: the CUDA path (libuwbnli.so through the C-ABI) against the
reference's own outputs (tests/golden, generated from the unmodified
reference headers) and the C oracle on the same inputs.

Tolerances (BASELINE.json north_star: <= 1e-6 relative eta, <= 0.01 dB SNR):
  NLI on identical inputs ............ 1e-9 relative (FP64; observed ~1e-13)
  full path (device ODE + NLI + SNR) . 1e-6 relative eta, 0.01 dB SNR
"""
import os

import numpy as np
import pytest

import paper_2401_18022_b200 as uwb
from helpers import cfg_of, engine_inputs_from_oracle, product_scenario, to_db
from pyoracle import Case, oband11, toy_case

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu

NLI_TOL = 1e-9

SMALL_CASES = ["cband11", "oband11", "oband11_simpson", "cband11_nr40", "cband11_uniform",
               "cband11_direct_q4", "toy5_nr64", "toy5_guard", "toy5_simpson", "toy5_2mw",
               "toy3_3span", "cband11_uniform_z", "uwb589_random_launch"]


def _rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    den = np.where(b == 0, 1.0, np.abs(b))
    return float(np.max(np.abs(a - b) / den)) if a.size else 0.0


@pytest.mark.parametrize("name", SMALL_CASES + ["uwb589_75_0.95", "uwb589_150_1.4"])
def test_all_channels_nli_matches_reference(name, golden, oracle, engine):
    rec = golden["all_channels_nli"][name]
    case = Case.from_json(rec["case"])
    prep = oracle.prepare(case)
    grid, spans, betas, gamma = engine_inputs_from_oracle(prep, case.density)
    r = uwb.all_channels_nli(grid, spans, betas, None, cfg_of(case), engine=engine, gamma=gamma)
    assert np.array_equal(r.skipped, np.array(rec["skipped"], np.uint8))
    assert _rel(r.eta, rec["eta"]) < NLI_TOL
    assert _rel(r.nli_psd, rec["nli_psd"]) < NLI_TOL
    assert _rel(r.nli_power, rec["nli_power"]) < NLI_TOL
    q = np.array(rec["quadrant"])
    assert _rel(r.quadrant, q) < NLI_TOL
    assert r.elapsed_seconds > 0.0


def test_nli_psd_at_and_cartesian(golden, oracle, engine):
    for rec in golden["nli_psd_at"]:
        case = Case.from_json(rec["case"])
        prep = oracle.prepare(case)
        grid, spans, betas, _ = engine_inputs_from_oracle(prep, case.density)
        q = np.zeros(4)
        v = uwb.nli_psd_at(grid, spans, betas, rec["gamma"], cfg_of(case), rec["nu"],
                           quadrant_diag=q, engine=engine)
        assert abs(v / rec["value"] - 1.0) < NLI_TOL
        assert _rel(q, rec["quad"]) < NLI_TOL
        if "cartesian600" in rec:  # test_gn_integral.cpp:226-235
            assert abs(to_db(v / rec["cartesian600"])) < 0.1


def test_mirror_q4_equals_direct_q4(oracle, engine):
    """test_gn_integral.cpp:250-263 on the device."""
    case = toy_case(3, n_r=80)
    prep = oracle.prepare(case)
    grid, spans, betas, _ = engine_inputs_from_oracle(prep, case.density)
    qa, qb = np.zeros(4), np.zeros(4)
    nu = grid.freq[0]
    a = uwb.nli_psd_at(grid, spans, betas, 1.3e-3, cfg_of(case), nu, quadrant_diag=qa, engine=engine)
    direct = cfg_of(case)
    direct.mirror_q4 = False
    b = uwb.nli_psd_at(grid, spans, betas, 1.3e-3, direct, nu, quadrant_diag=qb, engine=engine)
    assert a == pytest.approx(b, rel=1e-12)
    assert qa[3] == pytest.approx(qb[3], rel=1e-12)
    assert qb[1] == pytest.approx(qb[3], rel=1e-12)


def test_batched_probes_equal_single_probes(oracle, engine):
    case = toy_case(5, n_r=40)
    prep = oracle.prepare(case)
    grid, spans, betas, _ = engine_inputs_from_oracle(prep, case.density)
    nus = grid.freq.copy()
    batch = uwb.nli_psd_at(grid, spans, betas, np.full(5, 1.3e-3), cfg_of(case), nus, engine=engine)
    for k, nu in enumerate(nus):
        single = uwb.nli_psd_at(grid, spans, betas, 1.3e-3, cfg_of(case), float(nu), engine=engine)
        assert single == batch[k]  # bit-identical: per-probe reductions are order-fixed


def test_channel_nli_simpson(oracle, engine):
    case = toy_case(5, n_r=64, simpson=1)
    prep = oracle.prepare(case)
    grid, spans, betas, gamma = engine_inputs_from_oracle(prep, case.density)
    ref = oracle.all_channels_nli(case, prep)
    for ch in range(5):
        v = uwb.channel_nli(grid, spans, betas, gamma[ch], cfg_of(case), ch, engine=engine)
        assert v == pytest.approx(ref["nli_psd"][ch], rel=NLI_TOL)


def test_deterministic_and_partition_independent(golden, oracle, engine):
    """Bit-identity across worker counts (test_gn_integral.cpp:291-300) becomes
    bit-identity across runs and across channel partitions (multi-GPU)."""
    case = Case.from_json(golden["all_channels_nli"]["cband11_nr40"]["case"])
    prep = oracle.prepare(case)
    grid, spans, betas, gamma = engine_inputs_from_oracle(prep, case.density)
    cfg = cfg_of(case)
    a = uwb.all_channels_nli(grid, spans, betas, None, cfg, engine=engine, gamma=gamma)
    b = uwb.all_channels_nli(grid, spans, betas, None, cfg, engine=engine, gamma=gamma)
    assert np.array_equal(a.eta, b.eta) and np.array_equal(a.quadrant, b.quadrant)
    merged = np.zeros_like(a.eta)
    for part in (np.arange(0, 11, 2), np.arange(1, 11, 2)):
        engine.set_channel_subset(part)
        r = uwb.all_channels_nli(grid, spans, betas, None, cfg, engine=engine, gamma=gamma)
        merged[part] = r.eta[part]
        others = np.setdiff1d(np.arange(11), part)
        assert np.all(r.skipped[others] == 1) and np.all(r.eta[others] == 0.0)
    engine.set_channel_subset(None)
    assert np.array_equal(merged, a.eta)


def test_cubic_power_scaling(oracle, engine):
    """test_gn_integral.cpp:277-289 / acceptance C4: Raman off, +3 dB -> +9 dB."""
    base = toy_case(5, n_r=64)
    loud = toy_case(5, n_r=64, uniform_w=2e-3)
    out = []
    for case in (base, loud):
        prep = oracle.prepare(case)
        grid, spans, betas, gamma = engine_inputs_from_oracle(prep, case.density)
        out.append(uwb.all_channels_nli(grid, spans, betas, None, cfg_of(case), engine=engine,
                                        gamma=gamma))
    assert np.all(out[0].eta > 0)
    np.testing.assert_allclose(out[1].nli_power, 8.0 * out[0].nli_power, rtol=1e-9)
    np.testing.assert_allclose(out[1].eta, out[0].eta, rtol=1e-9)


def test_config_errors(oracle, engine):
    """test_gn_integral.cpp:339-346: ConfigError contract."""
    case = toy_case(5, n_r=64)
    prep = oracle.prepare(case)
    grid, spans, betas, _ = engine_inputs_from_oracle(prep, case.density)
    bad = cfg_of(case)
    bad.n_r = 1
    with pytest.raises(uwb.ConfigError):
        uwb.nli_psd_at(grid, spans, betas, 1e-3, bad, grid.centre, engine=engine)
    with pytest.raises(uwb.ConfigError):
        uwb.nli_psd_at(grid, [], betas, 1e-3, cfg_of(case), grid.centre, engine=engine)
    other = uwb.make_uniform_grid(4, 12e9, 10e9, 193.5e12)
    with pytest.raises(uwb.ConfigError):
        uwb.nli_psd_at(other, spans, betas, 1e-3, cfg_of(case), other.centre, engine=engine)
    with pytest.raises(uwb.ConfigError):  # quadrant_limits: probe outside the half band
        uwb.nli_psd_at(grid, spans, betas, 1e-3, cfg_of(case), grid.centre + 2 * grid.half_band,
                       engine=engine)


def test_dark_grid_reports_zeros(oracle, engine):
    case = toy_case(5, n_r=64)
    prep = oracle.prepare(case)
    grid, spans, betas, gamma = engine_inputs_from_oracle(prep, case.density)
    grid.psd[:] = 0.0
    grid.guard[:] = 1
    r = uwb.all_channels_nli(grid, spans, betas, None, cfg_of(case), engine=engine, gamma=gamma)
    assert np.all(r.skipped == 1) and np.all(r.eta == 0.0)


# ---------------------------------------------------------------- device ODE
@pytest.mark.parametrize("name", ["cband11", "oband11", "toy3", "toy3_lossless", "uwb589",
                                  "uwb589_2dbm", "uwb589_random_launch"])
def test_power_evolution_matches_reference(name, golden, engine):
    rec = golden["power_evolution"][name]
    case = Case.from_json(rec["case"])
    grid, fibre = product_scenario(case)
    zg = uwb.build_distance_grid(case.length_m, case.density)
    evo = uwb.solve_power_evolution(fibre, grid, zg, uwb.RamanSolveOptions(bool(case.raman)),
                                    engine=engine)
    assert evo.steps() == rec["steps"]
    np.testing.assert_allclose(evo.rho_end, rec["rho_end"], rtol=1e-9)
    if "log_rho" in rec:
        np.testing.assert_allclose(evo.log_rho, rec["log_rho"], rtol=0, atol=1e-9)
    for i, v in rec["log_rho_samples"]:
        assert abs(evo.log_rho[i] - v) < 1e-9
    assert abs(np.sum(evo.log_rho) - rec["log_rho_sum"]) < 1e-6


# ---------------------------------------------------------------- full SNR evaluation
@pytest.mark.parametrize("name", ["uwb589_75_0.95", "uwb589_random_launch"])
def test_evaluate_link_matches_reference(name, golden, engine):
    rec = golden["evaluate_link"][name]
    case = Case.from_json(rec["case"])
    grid, fibre = product_scenario(case)
    lc = uwb.LinkConfig(gn=cfg_of(case), raman=uwb.RamanSolveOptions(bool(case.raman)))
    rep = uwb.evaluate_link(fibre, grid, lc, engine=engine)
    eta_ref = np.array(rec["eta"])
    act = eta_ref > 0
    assert _rel(rep.eta[act], eta_ref[act]) < 1e-6
    assert np.max(np.abs(rep.snr_db[act] - np.array(rec["snr_db"])[act])) < 0.01
    np.testing.assert_allclose(rep.p_ase[act], np.array(rec["p_ase"])[act], rtol=1e-6)
    assert rep.loss_value == pytest.approx(rec["loss"], rel=1e-9)
    assert rep.total_capacity == pytest.approx(rec["total_capacity"], rel=1e-9)
    assert rep.total_power_dbm == pytest.approx(rec["total_power_dbm"], abs=1e-9)


def test_resident_link_equals_host_call(golden, engine):
    import torch

    rec = golden["evaluate_link"]["uwb589_random_launch"]
    case = Case.from_json(rec["case"])
    grid, fibre = product_scenario(case)
    lc = uwb.LinkConfig(gn=cfg_of(case))
    host = uwb.evaluate_link(fibre, grid, lc, engine=engine)
    res = uwb.ResidentLink(fibre, grid, lc, engine=engine)
    psd = torch.tensor(grid.psd, dtype=torch.float64, device="cuda:0")
    out = torch.zeros(res.report_len, dtype=torch.float64, device="cuda:0")
    res.run(psd.data_ptr(), out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    n = grid.size()
    assert np.array_equal(o[:n], host.eta)
    assert np.array_equal(o[2 * n:3 * n], host.snr_db)
    assert o[4 * n] == host.loss_value


def test_evaluate_link_many_equals_single_evaluations(golden, engine):
    """uwb_evaluate_link_many (the optimiser's batched cost calls) reproduces
    one-at-a-time evaluations, in order, bit for bit: the batch runs the same
    ODE kernel and split (on a second stream, overlapped with the previous
    evaluation's integrand) and the integrand's reductions do not depend on
    its grid size."""
    rec = golden["evaluate_link"]["uwb589_random_launch"]
    case = Case.from_json(rec["case"])
    grid, fibre = product_scenario(case)
    lc = uwb.LinkConfig(gn=uwb.GnSolverConfig(n_r=24, mean_step_density=0.95))
    res = uwb.ResidentLink(fibre, grid, lc, engine=engine)
    rng = np.random.default_rng(7)
    base = np.array(grid.psd)
    psd = np.stack([base * (1.0 + 0.2 * rng.random(base.size)) * (base > 0) for _ in range(4)])
    loss, reps = res.run_many(psd, reports=True)
    for k in range(4):
        g = grid.copy()
        g.psd = psd[k].copy()
        one = uwb.evaluate_link(fibre, g, lc, engine=engine)
        assert loss[k] == one.loss_value
        assert np.array_equal(reps[k][:grid.size()], one.eta)


def test_u2_symmetry_sharing_matches_full_evaluation():
    """Quadrants 1 and 3 share |K|^2 between u2 and -u2; the
    quadrant sums with sharing off (UWB_NLI_NO_MIRROR=1, every column
    evaluated) must agree to rounding, on a case with a centre probe (Q2 at
    f = 0 is NOT a symmetry) and Simpson probes."""
    import json
    import subprocess
    import sys

    code = r'''
import json, sys
sys.path.insert(0, "oracle"); sys.path.insert(0, "tests")
import numpy as np
import paper_2401_18022_b200 as uwb
from pyoracle import Oracle, oband11
from helpers import engine_inputs_from_oracle, cfg_of
case = oband11(n_r=60, density=0.95)
case.simpson = 1
O = Oracle(); prep = O.prepare(case)
grid, spans, betas, gamma = engine_inputs_from_oracle(prep, case.density)
eng = uwb.Engine(0)
r = uwb.all_channels_nli(grid, spans, betas, None, cfg_of(case), engine=eng, gamma=gamma)
st = eng.last_nli_stats()
print(json.dumps({"q": np.asarray(r.quadrant).ravel().tolist(), "eta": np.asarray(r.eta).tolist(),
                  "evaluated": st["evaluated_points"], "active": st["active_points"]}))
'''
    out = {}
    for flag in ("0", "1"):
        env = dict(os.environ, UWB_NLI_NO_MIRROR=flag)
        p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                           timeout=600, cwd=ROOT)
        assert p.returncode == 0, p.stderr
        out[flag] = json.loads(p.stdout.strip().splitlines()[-1])
    on, off = out["0"], out["1"]
    assert on["active"] == off["active"] == off["evaluated"]
    assert on["evaluated"] < 0.75 * off["evaluated"]
    assert _rel(on["q"], off["q"]) < 1e-13
    assert _rel(on["eta"], off["eta"]) < 1e-13


def test_split_evaluation_bit_identical_to_fused():
    """evaluate_link's split integrand (nli_setup_kernel beside the Raman ODE,
    then nli_list_kernel over the listed points) keeps the fused kernel's
    point order and group sums, so the report is bit-identical to the fused
    nli_rows_kernel's (UWB_NLI_NO_SPLIT=1), on a profile with dark channels
    and an odd n_r (a self-mirrored middle column)."""
    import json
    import subprocess
    import sys

    code = r'''
import json
import numpy as np
import paper_2401_18022_b200 as uwb
eng = uwb.Engine(0)
grid = uwb.make_default_uwb_grid()
uwb.set_uniform_launch(grid, 1e-3)
rng = np.random.default_rng(3)
psd = np.array(grid.psd) * (1.0 + 0.3 * rng.random(grid.size()))
psd[rng.random(grid.size()) < 0.05] = 0.0
grid.psd = psd
out = {}
for n_r, dens in ((41, 0.95), (150, 1.4)):
    lc = uwb.LinkConfig(gn=uwb.GnSolverConfig(n_r=n_r, mean_step_density=dens))
    r = uwb.evaluate_link(uwb.default_fibre(), grid, lc, engine=eng)
    st = eng.last_nli_stats()
    out[str(n_r)] = {"eta": [float(x).hex() for x in np.asarray(r.eta)],
                     "loss": float(r.loss_value).hex(), "evaluated": st["evaluated_points"],
                     "active": st["active_points"]}
print(json.dumps(out))
'''
    out = {}
    for flag in ("0", "1"):
        env = dict(os.environ, UWB_NLI_NO_SPLIT=flag)
        p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                           timeout=600, cwd=ROOT)
        assert p.returncode == 0, p.stderr
        out[flag] = json.loads(p.stdout.strip().splitlines()[-1])
    assert out["0"] == out["1"]
    assert out["0"]["41"]["active"] > 0


@pytest.mark.parametrize("kw", [
    dict(n_r=41),                                   # odd n_r: the middle column is its own mirror
    dict(n_r=33, u1_uniform=1),                     # uniform u1 edges
    dict(n_r=41, mirror_q4=0),                      # direct Q4 (not symmetric) alongside Q1/Q3
    dict(n_r=27, span_count=2),                     # two spans: per-point z / half-log loads
    dict(n_r=3),                                    # tiny rows
], ids=["odd", "uniform", "direct_q4", "two_spans", "tiny"])
def test_all_channels_nli_edge_cases_vs_oracle(kw, oracle, engine):
    """Small edge cases against the C oracle (pinned bit-exact to the
    reference) on identical inputs; exercises the u2-symmetric row path with
    odd/tiny n_r, uniform u1, direct Q4 and multi-span tables."""
    case = oband11(**kw)
    prep = oracle.prepare(case)
    ref = oracle.all_channels_nli(case, prep)
    grid, spans, betas, gamma = engine_inputs_from_oracle(prep, case.density)
    r = uwb.all_channels_nli(grid, spans, betas, None, cfg_of(case), engine=engine, gamma=gamma)
    assert np.array_equal(r.skipped, ref["skipped"])
    assert _rel(r.eta, ref["eta"]) < NLI_TOL
    assert _rel(np.asarray(r.quadrant).ravel(), np.asarray(ref["quadrant"]).ravel()) < NLI_TOL


# ---------------------------------------------------------------- compensated FP32 ("mixed")
MIXED_TOL = 1e-6  # north_star: <= 1e-6 relative eta (the FP64 path meets 1e-9)


@pytest.fixture
def mixed_engine(engine):
    engine.set_precision("mixed")
    yield engine
    engine.set_precision("fp64")


@pytest.mark.parametrize("name", ["cband11", "oband11", "oband11_simpson", "toy3_3span",
                                  "cband11_nr40", "uwb589_75_0.95", "uwb589_150_1.4"])
def test_mixed_precision_nli_within_tolerance(name, golden, oracle, mixed_engine):
    """BASELINE config 4's compensated-FP32 column: the mixed integrand stays
    within the north-star tolerance of the reference on the golden cases
    (observed <= 5e-8)."""
    rec = golden["all_channels_nli"][name]
    case = Case.from_json(rec["case"])
    prep = oracle.prepare(case)
    grid, spans, betas, gamma = engine_inputs_from_oracle(prep, case.density)
    r = uwb.all_channels_nli(grid, spans, betas, None, cfg_of(case), engine=mixed_engine,
                             gamma=gamma)
    assert np.array_equal(r.skipped, np.array(rec["skipped"], np.uint8))
    eta = np.array(rec["eta"])
    act = eta > 0
    assert _rel(r.eta[act], eta[act]) < MIXED_TOL
    assert np.max(np.abs(to_db(r.eta[act]) - to_db(eta[act]))) < 0.01


def test_mixed_precision_evaluate_link(golden, mixed_engine):
    rec = golden["evaluate_link"]["uwb589_random_launch"]
    case = Case.from_json(rec["case"])
    grid, fibre = product_scenario(case)
    lc = uwb.LinkConfig(gn=cfg_of(case), raman=uwb.RamanSolveOptions(bool(case.raman)))
    rep = uwb.evaluate_link(fibre, grid, lc, engine=mixed_engine)
    eta_ref = np.array(rec["eta"])
    act = eta_ref > 0
    assert _rel(rep.eta[act], eta_ref[act]) < MIXED_TOL
    assert np.max(np.abs(rep.snr_db[act] - np.array(rec["snr_db"])[act])) < 0.01


def test_precision_mode_errors(engine):
    with pytest.raises(uwb.ConfigError):
        engine.set_precision("fp16")


# ---------------------------------------------------------------- closed-form model (§8 f4)
@pytest.mark.parametrize("name", ["cband11", "oband11", "toy5_guard", "toy3_3span", "uwb589_0.95",
                                  "uwb589_random_launch"])
def test_cfm_all_channels_nli_matches_reference(name, golden_cfm, oracle, engine):
    """cfm_all_channels_nli (gn_closed_form.hpp:70-144) on the device vs the
    reference's own outputs, on the oracle's (bit-exact) ODE tables."""
    rec = golden_cfm["cfm_all_channels_nli"][name]
    case = Case.from_json(rec["case"])
    prep = oracle.prepare(case)
    grid, spans, betas, gamma = engine_inputs_from_oracle(prep, case.density)
    r = uwb.cfm_all_channels_nli(grid, spans, betas, None, engine=engine, gamma=gamma)
    assert np.array_equal(r.skipped, np.array(rec["skipped"], np.uint8))
    assert _rel(r.eta, rec["eta"]) < NLI_TOL
    assert _rel(r.nli_psd, rec["nli_psd"]) < NLI_TOL
    assert _rel(r.nli_power, rec["nli_power"]) < NLI_TOL
    assert np.all(np.asarray(r.quadrant) == 0.0)
    assert r.elapsed_seconds > 0.0


def test_cfm_config_errors(oracle, engine):
    case = oband11()
    prep = oracle.prepare(case)
    grid, spans, betas, gamma = engine_inputs_from_oracle(prep, case.density)
    with pytest.raises(uwb.ConfigError):
        uwb.cfm_all_channels_nli(grid, [], betas, None, engine=engine, gamma=gamma)


# ---------------------------------------------------------------- acceptance checks on the device
C0 = 299792458.0


def _device_nli(engine, n_ch, lam, dbm, n_r, density, raman=True):
    fibre = uwb.default_fibre()
    grid = uwb.make_uniform_grid(n_ch, 100e9, 96e9, C0 / lam)
    uwb.set_uniform_launch(grid, 1e-3 * 10 ** (dbm / 10))
    zg = uwb.build_distance_grid(fibre.length_m, density)
    evo = uwb.solve_power_evolution(fibre, grid, zg, uwb.RamanSolveOptions(raman), engine=engine)
    betas = uwb.beta_from_dispersion(fibre, C0 / grid.centre)
    cfg = uwb.GnSolverConfig(n_r=n_r, mean_step_density=density)
    return uwb.all_channels_nli(grid, [evo], betas, fibre, cfg, engine=engine)


def test_acceptance_c2_resolution_tradeoff(engine):
    """acceptance_main.cpp:88-137 (C2) on the device: 64-ch C-band, (75, 0.95)
    within 0.6 dB and (150, 1.4) within 0.15 dB of (500, 2.0).  The C2 worker
    check (1 vs 4 identical) is test_deterministic_and_partition_independent;
    its CPU-thread timing ratios have no device counterpart."""
    ref = _device_nli(engine, 64, 1550e-9, 0.0, 500, 2.0)
    coarse = _device_nli(engine, 64, 1550e-9, 0.0, 75, 0.95)
    mid = _device_nli(engine, 64, 1550e-9, 0.0, 150, 1.4)
    dev_c = np.max(np.abs(to_db(coarse.eta / ref.eta)))
    dev_m = np.max(np.abs(to_db(mid.eta / ref.eta)))
    assert dev_c <= 0.6 and dev_m <= 0.15, (dev_c, dev_m)


def test_acceptance_c4_cubic_scaling_raman_off(engine):
    """acceptance_main.cpp:183-217 (C4): +3 dB launch -> +9 dB NLI power within
    0.01 dB and eta drift <= 1e-6 (16-ch C-band, Raman off, N_R 64, 0.8/km)."""
    base = _device_nli(engine, 16, 1550e-9, 0.0, 64, 0.8, raman=False)
    boost = _device_nli(engine, 16, 1550e-9, 3.0, 64, 0.8, raman=False)
    gain = 10 * np.log10(boost.nli_power / base.nli_power)
    assert np.max(np.abs(gain - 9.0)) <= 0.01
    assert np.max(np.abs(boost.eta / base.eta - 1.0)) <= 1e-6


# ---------------------------------------------------------------- ODE step-size policy extension
@pytest.fixture
def continuous_engine(engine):
    engine.set_ode_stepping("continuous")
    yield engine
    engine.set_ode_stepping("restart")


@pytest.mark.parametrize("name", ["uwb589_75_0.95", "uwb589_random_launch"])
def test_continuous_ode_stepping_within_tolerance(name, golden, continuous_engine):
    """uwb_set_ode_stepping(CONTINUOUS): the reference's Dormand-Prince
    controller without the restart at every midpoint (~3x fewer RHS).  Full
    evaluation within the north-star tolerance of the reference (observed
    2.5e-10 eta, 5e-9 dB)."""
    rec = golden["evaluate_link"][name]
    case = Case.from_json(rec["case"])
    grid, fibre = product_scenario(case)
    lc = uwb.LinkConfig(gn=cfg_of(case), raman=uwb.RamanSolveOptions(bool(case.raman)))
    rep = uwb.evaluate_link(fibre, grid, lc, engine=continuous_engine)
    eta_ref = np.array(rec["eta"])
    act = eta_ref > 0
    assert _rel(rep.eta[act], eta_ref[act]) < 1e-8
    assert np.max(np.abs(rep.snr_db[act] - np.array(rec["snr_db"])[act])) < 1e-6


@pytest.mark.parametrize("name", ["uwb589", "cband11", "toy3"])
def test_continuous_ode_power_evolution(name, golden, continuous_engine):
    rec = golden["power_evolution"][name]
    case = Case.from_json(rec["case"])
    grid, fibre = product_scenario(case)
    zg = uwb.build_distance_grid(case.length_m, case.density)
    evo = uwb.solve_power_evolution(fibre, grid, zg, uwb.RamanSolveOptions(bool(case.raman)),
                                    engine=continuous_engine)
    np.testing.assert_allclose(evo.rho_end, rec["rho_end"], rtol=1e-8)
    for i, v in rec["log_rho_samples"]:
        assert abs(evo.log_rho[i] - v) < 1e-8


def test_ode_stepping_mode_errors(engine):
    with pytest.raises(uwb.ConfigError):
        engine.set_ode_stepping("adaptive")


def test_power_evolution_gain_table_with_gap(oracle, engine):
    """A Raman gain table with a zero stretch between two gain lobes: the
    device's contiguous window-edge pieces (raman_segments fills the gap with
    a zero piece) against the C oracle's dense mat-vec on the same table."""
    import ctypes as C
    rx = np.array([0.0, 10e12, 20e12, 25e12, 100e12])
    ry = np.array([0.2e-3, 0.0, 0.0, 0.2e-3, 0.0])
    case = Case(uwb_default=1, n_r=8, density=0.95, raman=1, name="gap")
    # oracle: default fibre with the table replaced
    f, g = oracle.fibre(case), oracle.grid(case)
    f.raman_gain.n = rx.size
    for k in range(rx.size):
        f.raman_gain.x[k], f.raman_gain.y[k] = rx[k], ry[k]
    zg = oracle.distance_grid(case.length_m, case.density)
    n, s = g.n, zg["steps"]
    lr, re, ev = np.zeros(n * s), np.zeros(n), C.c_long()
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    rc = oracle.lib.or_power_evolution(C.byref(f), C.byref(g), dp(zg["mid"]), s,
                                       C.c_double(case.length_m), 1, dp(lr), dp(re), C.byref(ev))
    assert rc == 0
    grid, fibre = product_scenario(case)
    fibre.raman_x, fibre.raman_y = rx, ry
    evo = uwb.solve_power_evolution(fibre, grid, uwb.build_distance_grid(case.length_m, case.density),
                                    uwb.RamanSolveOptions(True), engine=engine)
    np.testing.assert_allclose(evo.log_rho, lr, rtol=0, atol=1e-9)
    np.testing.assert_allclose(evo.rho_end, re, rtol=1e-9)
    # the table really couples channels: differs from the default triangle
    base = uwb.solve_power_evolution(uwb.default_fibre(), grid,
                                     uwb.build_distance_grid(case.length_m, case.density),
                                     uwb.RamanSolveOptions(True), engine=engine)
    assert np.max(np.abs(base.log_rho - evo.log_rho)) > 1e-3


@pytest.mark.parametrize("name", ["oband101", "oband101_simpson_nr80"])
def test_stress_oband101_matches_reference(name, golden_stress, oracle, engine):
    """BASELINE config 2 stress variant: 101 channels straddling the
    zero-dispersion wavelength (MCI-dominated, 63 % sinc-branch points)."""
    rec = golden_stress["all_channels_nli"][name]
    case = Case.from_json(rec["case"])
    prep = oracle.prepare(case)
    grid, spans, betas, gamma = engine_inputs_from_oracle(prep, case.density)
    r = uwb.all_channels_nli(grid, spans, betas, None, cfg_of(case), engine=engine, gamma=gamma)
    assert np.array_equal(r.skipped, np.array(rec["skipped"], np.uint8))
    assert _rel(r.eta, rec["eta"]) < NLI_TOL
    assert _rel(np.asarray(r.quadrant).ravel(), np.asarray(rec["quadrant"]).ravel()) < NLI_TOL


@pytest.mark.parametrize("seed", range(int(os.environ.get("UWB_RANDOM_CASES", "24"))))
def test_randomised_configs_vs_oracle(seed, oracle, engine):
    """Seeded random small configurations against the C oracle (pinned
    bit-exact to the reference; UWB_RANDOM_CASES=300 widens the sweep, run
    clean on the v14 build): channel count, spacing, width, centre
    wavelength, per-channel launch power, n_r, step density (1-13 steps per
    lane, i.e. hoisted and non-hoisted kernels, FULL and ragged step counts),
    span count, u1 sampling, Simpson and direct Q4."""
    rng = np.random.default_rng(1000 + seed)
    n_ch = int(rng.integers(3, 41))
    spacing = float(rng.choice([50e9, 75e9, 100e9, 150e9]))
    lam = float(rng.uniform(1280e-9, 1620e-9))
    case = Case(n_ch=n_ch, spacing=spacing, bch=spacing * float(rng.uniform(0.6, 0.96)),
                centre=299792458.0 / lam,
                launch_w=1e-3 * 10 ** (rng.uniform(-3, 3, n_ch) / 10),
                n_r=int(rng.integers(6, 48)), density=float(rng.choice([0.25, 0.8, 1.4, 2.5])),
                span_count=int(rng.integers(1, 4)), length_m=float(rng.choice([50e3, 80e3])),
                u1_uniform=int(rng.random() < 0.25), simpson=int(rng.random() < 0.25),
                mirror_q4=int(rng.random() < 0.75), name=f"rand{seed}")
    from pyoracle import OracleError
    prep = oracle.prepare(case)
    grid, spans, betas, gamma = engine_inputs_from_oracle(prep, case.density)
    try:
        ref = oracle.all_channels_nli(case, prep)
    except OracleError as exc:  # the reference rejects it: so must the engine, alike
        assert exc.code == 2
        with pytest.raises(uwb.ConfigError):
            uwb.all_channels_nli(grid, spans, betas, None, cfg_of(case), engine=engine, gamma=gamma)
        return
    r = uwb.all_channels_nli(grid, spans, betas, None, cfg_of(case), engine=engine, gamma=gamma)
    assert np.array_equal(r.skipped, ref["skipped"])
    assert _rel(r.eta, ref["eta"]) < NLI_TOL, case
    assert _rel(np.asarray(r.quadrant).ravel(), np.asarray(ref["quadrant"]).ravel()) < NLI_TOL


@pytest.mark.parametrize("seed", range(12))
def test_randomised_power_evolution_vs_oracle(seed, oracle, engine):
    """Seeded random combs (3-700 channels: the one-warp and multi-warp
    channel splits, 1-3 pieces of gain table in range), random launch powers
    and step densities: the device Raman ODE against the C oracle's
    restatement of the reference solve (dense mat-vec RK45), 1e-9 in log rho."""
    rng = np.random.default_rng(2000 + seed)
    n_ch = int(rng.choice([int(rng.integers(3, 33)), int(rng.integers(33, 97)),
                           int(rng.integers(97, 701))]))
    spacing = float(rng.choice([50e9, 75e9, 100e9]))
    lam = float(rng.uniform(1300e-9, 1600e-9))
    case = Case(n_ch=n_ch, spacing=spacing, bch=0.9 * spacing, centre=299792458.0 / lam,
                launch_w=1e-3 * 10 ** (rng.uniform(-4, 4, n_ch) / 10),
                density=float(rng.choice([0.3, 0.95, 1.4, 2.0])), raman=1, name=f"ode{seed}")
    ref = oracle.power_evolution(case)
    grid, fibre = product_scenario(case)
    zg = uwb.build_distance_grid(case.length_m, case.density)
    evo = uwb.solve_power_evolution(fibre, grid, zg, uwb.RamanSolveOptions(True), engine=engine)
    assert evo.steps() == ref["steps"]
    np.testing.assert_allclose(evo.log_rho, ref["log_rho"], rtol=0, atol=1e-9)
    np.testing.assert_allclose(evo.rho_end, ref["rho_end"], rtol=1e-9)


@pytest.mark.parametrize("n_ch", [800, 1500])
def test_wide_comb_power_evolution_vs_oracle(n_ch, oracle, engine):
    """Combs beyond 256 ODE threads (the 512-thread CTA: 9 and 16 warps of 3
    channels, the rolled cross-warp offsets) against the oracle, 1e-9 in
    log rho."""
    rng = np.random.default_rng(4000 + n_ch)
    case = Case(n_ch=n_ch, spacing=25e9, bch=22e9, centre=299792458.0 / 1450e-9,
                launch_w=1e-4 * 10 ** (rng.uniform(-3, 3, n_ch) / 10),
                density=0.3, raman=1, name=f"wide{n_ch}")
    ref = oracle.power_evolution(case)
    grid, fibre = product_scenario(case)
    zg = uwb.build_distance_grid(case.length_m, case.density)
    evo = uwb.solve_power_evolution(fibre, grid, zg, uwb.RamanSolveOptions(True), engine=engine)
    assert evo.steps() == ref["steps"]
    np.testing.assert_allclose(evo.log_rho, ref["log_rho"], rtol=0, atol=1e-9)
    np.testing.assert_allclose(evo.rho_end, ref["rho_end"], rtol=1e-9)


@pytest.mark.parametrize("seed", range(6))
def test_randomised_evaluate_link_vs_reference(seed, engine):
    """Full evaluate_link (device ODE + NLI + SNR assembly) on seeded random
    small combs against the UNMODIFIED reference run here through its harness
    (oracle/_ref/libuwbref.so; skipped where it was not built)."""
    from pyoracle import RefLib
    if not RefLib.available():
        pytest.skip("oracle/_ref/libuwbref.so not built")
    R = RefLib()
    rng = np.random.default_rng(3000 + seed)
    n_ch = int(rng.integers(5, 41))
    lam = float(rng.uniform(1290e-9, 1610e-9))
    case = Case(n_ch=n_ch, spacing=100e9, bch=96e9, centre=299792458.0 / lam,
                launch_w=1e-3 * 10 ** (rng.uniform(-3, 3, n_ch) / 10),
                n_r=int(rng.integers(8, 31)), density=float(rng.choice([0.95, 1.4])),
                span_count=int(rng.integers(1, 3)), name=f"link{seed}")
    ref = R.evaluate_link(case)
    grid, fibre = product_scenario(case)
    lc = uwb.LinkConfig(gn=cfg_of(case), raman=uwb.RamanSolveOptions(True))
    rep = uwb.evaluate_link(fibre, grid, lc, engine=engine)
    act = ref["eta"] > 0
    assert _rel(rep.eta[act], ref["eta"][act]) < 1e-9
    assert np.max(np.abs(rep.snr_db[act] - ref["snr_db"][act])) < 1e-8
    np.testing.assert_allclose(rep.p_ase[act], ref["p_ase"][act], rtol=1e-9)
    assert rep.loss_value == pytest.approx(ref["loss"], rel=1e-9)
    assert rep.total_capacity == pytest.approx(ref["total_capacity"], rel=1e-9)


@pytest.mark.parametrize("density", [3.5, 6.0])
def test_long_spans_vs_oracle(density, oracle, engine):
    """More than 256 distance steps per span (the K = 17..32 kernels): 80 km at
    3.5 and 6.0 steps/km (281 / 481 steps), against the oracle at 1e-9."""
    case = oband11(n_r=24, density=density, name=f"long{density}")
    prep = oracle.prepare(case)
    assert prep["spans"][0]["steps"] > 256
    ref = oracle.all_channels_nli(case, prep)
    grid, spans, betas, gamma = engine_inputs_from_oracle(prep, case.density)
    r = uwb.all_channels_nli(grid, spans, betas, None, cfg_of(case), engine=engine, gamma=gamma)
    assert _rel(r.eta, ref["eta"]) < NLI_TOL
    # and the full device path (ODE writes the K > 16 lane layout)
    g2, fibre = product_scenario(case)
    rep = uwb.evaluate_link(fibre, g2, uwb.LinkConfig(gn=cfg_of(case)), engine=engine)
    assert _rel(rep.eta, ref["eta"]) < 1e-8


# ---------------------------------------------------------------- spans of their own
def _span_of(oracle, case):
    """One span's evolution (its own distance grid) for `case`'s grid."""
    prep = oracle.prepare(case)
    return prep, prep["spans"][0]


def test_spans_with_different_lengths_and_densities_vs_oracle(oracle, engine):
    """The reference builds one SpanView per span and walks each span's own
    step count (gn_integral.hpp:95-99, 141-145, 231-251): an 80 km span at
    1.4 steps/km (112 steps) followed by a 50 km span at 0.95 steps/km
    (48 steps) -- previously a ConfigError here -- against the oracle."""
    a = oband11(n_r=30, density=1.4, length_m=80e3)
    b = oband11(n_r=30, density=0.95, length_m=50e3)
    prep, sa = _span_of(oracle, a)
    _, sb = _span_of(oracle, b)
    assert sa["steps"] != sb["steps"]
    prep = dict(prep)
    prep["spans"] = [sa, sb]
    ref = oracle.all_channels_nli(a, prep)
    grid, _, betas, gamma = engine_inputs_from_oracle(dict(prep, spans=[sa]), a.density)
    spans = []
    for s in (sa, sb):
        zg = uwb.DistanceGrid(s["edge"], s["mid"], s["width"], s["length"], 1.0)
        spans.append(uwb.PowerEvolution(zg, grid.freq, grid.psd * grid.bch, s["log_rho"],
                                        prep["rho_end"], grid.spacing))
    r = uwb.all_channels_nli(grid, spans, betas, None, cfg_of(a), engine=engine, gamma=gamma)
    assert np.array_equal(r.skipped, ref["skipped"])
    assert _rel(r.eta, ref["eta"]) < NLI_TOL
    assert _rel(np.asarray(r.quadrant).ravel(), np.asarray(ref["quadrant"]).ravel()) < NLI_TOL
    # the span order matters (z offsets): swapped spans are a different link
    ref2 = oracle.all_channels_nli(a, dict(prep, spans=[sb, sa]))
    r2 = uwb.all_channels_nli(grid, spans[::-1], betas, None, cfg_of(a), engine=engine, gamma=gamma)
    assert _rel(r2.eta, ref2["eta"]) < NLI_TOL


@pytest.mark.parametrize("density", [8.0])
def test_spans_beyond_512_steps_vs_oracle(density, oracle, engine):
    """More than 512 distance steps per span (80 km at 8 steps/km = 640
    steps): the rolled K = 0 integrand, previously a ConfigError, against the
    oracle; and the full device path (ODE table in the same layout)."""
    case = oband11(n_r=12, density=density, name=f"long{density}")
    prep = oracle.prepare(case)
    assert prep["spans"][0]["steps"] > 512
    ref = oracle.all_channels_nli(case, prep)
    grid, spans, betas, gamma = engine_inputs_from_oracle(prep, case.density)
    r = uwb.all_channels_nli(grid, spans, betas, None, cfg_of(case), engine=engine, gamma=gamma)
    assert _rel(r.eta, ref["eta"]) < NLI_TOL
    g2, fibre = product_scenario(case)
    rep = uwb.evaluate_link(fibre, g2, uwb.LinkConfig(gn=cfg_of(case)), engine=engine)
    assert _rel(rep.eta, ref["eta"]) < 1e-8
