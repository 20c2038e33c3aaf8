"""CPU: the reference's hot-path unit tests (tests/test_gn_integral.cpp,
test_raman_power.cpp, test_optimizer.cpp), re-expressed against the oracle.
Catch2 is not installed, so these restate the assertions in pytest; they
check the oracle behaves like the reference on the reference's own cases.
"""
import numpy as np
import pytest

from pyoracle import Case, OracleError, toy_case


def test_phase_mismatch_vanishes_on_axes(oracle):  # :38-41
    b = (-1.9474701795517992e-26, 9.84268860900867e-41, -3.036944725627878e-55)
    assert oracle.phase_mismatch(0.0, 5e11, 1e12, b) == 0.0
    assert oracle.phase_mismatch(5e11, 0.0, -1e12, b) == 0.0


def test_phase_mismatch_term_isolation(oracle):  # :60-72
    f1, f2, fi = 2e11, -1.5e11, 7e11
    pi = np.pi
    expect = -4.0 * pi * pi * f1 * f2 * pi * 1e-40 * (f1 + f2 + 2.0 * fi)
    assert oracle.phase_mismatch(f1, f2, fi, (0.0, 1e-40, 0.0)) == pytest.approx(expect, rel=1e-12)
    f = 3e11
    expect4 = -4.0 * pi * pi * f * f * (2.0 * pi * pi / 3.0) * (-2e-55) * 3.5 * f * f
    assert oracle.phase_mismatch(f, f, 0.0, (0.0, 0.0, -2e-55)) == pytest.approx(expect4, rel=1e-12)


def test_quadrant_map_back_and_jacobian(oracle):  # :119-162
    rng = np.random.default_rng(11)
    b = 1e12
    for q in (1, 2, 3, 4):
        b1, b2, s1, s2, u1m = oracle.quadrant_limits(q, b, 0.2e12)
        for _ in range(16):
            u1 = rng.uniform(0.05, 0.95) * u1m
            su = np.sqrt(u1)
            hi, lo = np.log(b1 / su), -np.log(b2 / su)
            u2 = lo + rng.uniform(0.05, 0.95) * (hi - lo)
            g1 = su * np.exp(u2)
            g2 = u1 / g1
            assert g1 * g2 == pytest.approx(u1, rel=1e-12)
            assert g1 <= b1 * (1 + 1e-12) and g2 <= b2 * (1 + 1e-12)


def test_constant_power_kernel_is_analytic(oracle):  # :166-182
    case = toy_case(3, fibre_kind=1, flat_alpha_db_km=0.0, density=1.0)
    prep = oracle.prepare(case)
    nu = prep["grid_arrays"]["centre"]
    for phi in (1e-7, 1e-5, 1e-3, 0.05, 0.4):
        got = oracle.kernel_abs2_reference(prep, nu + 2e9, nu - 3e9, nu, phi)
        want = (2.0 - 2.0 * np.cos(phi * 80e3)) / (phi * phi)
        assert got == pytest.approx(want, rel=1e-9)
    assert oracle.kernel_abs2_reference(prep, nu, nu, nu, 0.0) == pytest.approx(80e3 ** 2, rel=1e-9)


def test_hyperbolic_vs_cartesian_toy(oracle):  # :226-235 (N_R=150 vs 600 cells)
    case = toy_case(3, n_r=150)
    prep = oracle.prepare(case)
    nu = prep["grid_arrays"]["centre"]
    hyp, _ = oracle.nli_psd_at(case, 1.3e-3, nu, prep)
    cart = oracle.cartesian_nli_psd(case, 1.3e-3, nu, 600, prep)
    assert abs(10 * np.log10(hyp / cart)) < 0.1


def test_uniform_u1_sampling(oracle):  # :237-248
    a, _ = oracle.nli_psd_at(toy_case(3, n_r=150), 1.3e-3, 193.5e12)
    b, _ = oracle.nli_psd_at(toy_case(3, n_r=300, u1_uniform=1), 1.3e-3, 193.5e12)
    assert abs(10 * np.log10(a / b)) < 0.3


def test_q4_mirror(oracle):  # :250-263
    nu = 193.5e12 - 12e9
    a, qa = oracle.nli_psd_at(toy_case(3, n_r=80), 1.3e-3, nu)
    b, qb = oracle.nli_psd_at(toy_case(3, n_r=80, mirror_q4=0), 1.3e-3, nu)
    assert a == pytest.approx(b, rel=1e-12)
    assert qa[3] == pytest.approx(qb[3], rel=1e-12)
    assert qb[1] == pytest.approx(qb[3], rel=1e-12)


def test_cubic_scaling_and_workers(oracle):  # :277-300
    base = oracle.all_channels_nli(toy_case(5, n_r=64, workers=1))
    loud = oracle.all_channels_nli(toy_case(5, n_r=64, workers=1, uniform_w=2e-3))
    assert np.all(base["eta"] > 0)
    np.testing.assert_allclose(loud["nli_power"], 8 * base["nli_power"], rtol=1e-9)
    np.testing.assert_allclose(loud["eta"], base["eta"], rtol=1e-9)
    par = oracle.all_channels_nli(toy_case(5, n_r=64, workers=4))
    assert np.array_equal(par["eta"], base["eta"])  # bit-identical across workers


def test_guard_and_dark_grid(oracle):  # :302-324
    r = oracle.all_channels_nli(toy_case(5, n_r=64, guard=np.array([0, 0, 1, 0, 0], np.uint8)))
    assert r["skipped"][2] == 1 and r["eta"][2] == 0.0 and r["eta"][1] > 0 and r["eta"][3] > 0
    dark = oracle.all_channels_nli(toy_case(5, n_r=64, guard=np.ones(5, np.uint8)))
    assert np.all(dark["skipped"] == 1) and np.all(dark["eta"] == 0.0)


def test_simpson_close_to_centre(oracle):  # :326-337
    c = oracle.all_channels_nli(toy_case(5, n_r=64))
    s = oracle.all_channels_nli(toy_case(5, n_r=64, simpson=1))
    assert np.all(np.abs(10 * np.log10(s["eta"] / c["eta"])) < 0.6)


def test_config_errors(oracle):  # :339-346
    with pytest.raises(OracleError):
        oracle.nli_psd_at(toy_case(5, n_r=1), 1e-3, 193.5e12)


def test_refinement_converges(oracle):  # :349-361
    e = {nr: oracle.nli_psd_at(toy_case(3, n_r=nr), 1.3e-3, 193.5e12)[0] for nr in (75, 150, 300)}
    d150 = abs(10 * np.log10(e[150] / e[300]))
    d75 = abs(10 * np.log10(e[75] / e[300]))
    assert d150 < d75 + 1e-9 and d150 < 0.1


def test_rho_without_raman_is_attenuation(oracle):  # test_raman_power.cpp:49-83
    case = toy_case(3, density=1.0, raman=0)
    e = oracle.power_evolution(case)
    alpha = 0.2 * np.log(10) / 10 / 1000
    mid = e["zgrid"]["mid"]
    rho = np.exp(e["log_rho"].reshape(3, -1))
    np.testing.assert_allclose(rho, np.exp(-alpha * mid)[None, :].repeat(3, 0), rtol=1e-6)
    np.testing.assert_allclose(e["rho_end"], np.exp(-alpha * 80e3), rtol=1e-6)


def test_photon_flux_conserved_lossless(oracle):  # test_raman_power.cpp:85-108
    case = Case(fibre_kind=1, flat_alpha_db_km=0.0, n_ch=2, spacing=13.2e12, bch=96e9,
                centre=193.4e12, uniform_w=10e-3, density=1.0)
    e = oracle.power_evolution(case)
    g = oracle.grid_arrays(oracle.grid(case))
    p = g["psd"] * g["bch"]
    rho = np.exp(e["log_rho"].reshape(2, -1))
    flux = (p[:, None] * rho / g["freq"][:, None]).sum(0)
    flux0 = (p / g["freq"]).sum()
    np.testing.assert_allclose(flux, flux0, rtol=1e-6)
    assert e["rho_end"][1] < 1.0


def test_ase_frozen_value(oracle):  # test_optimizer.cpp:16-20
    assert oracle.lib.or_ase_power(5.0, 10 ** 1.6, 193.4e12, 96e9) == pytest.approx(
        1.5098555472604998e-06, rel=1e-10)
