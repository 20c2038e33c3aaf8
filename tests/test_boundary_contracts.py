"""Boundary contracts where a wrong answer could otherwise come back with
status OK:

(a) ChannelGrid::validate (channel_grid.hpp:44-61) runs wherever the reference
    runs it -- solve_power_evolution calls it first (raman_power.hpp:56), so the
    device ODE, evaluate_link and the prepared link reject a grid that is not
    equally spaced or whose half band does not cover the occupied hull;
(b) the prepared / batched path re-derives the skip set (guard or psd <= 0,
    gn_integral.hpp:349-352) from EVERY call's launch profile: channels that
    are dark when the link is prepared and lit later (and the reverse) give
    exactly what single evaluate_link calls give.
"""
import numpy as np
import pytest

import paper_2401_18022_b200 as uwb

pytestmark = pytest.mark.gpu

C0 = 299792458.0


def _cband(n=11):
    g = uwb.make_uniform_grid(n, 100e9, 96e9, C0 / 1550e-9)
    uwb.set_uniform_launch(g, 1e-3)
    return g


def _lc(n_r=16, density=0.5):
    return uwb.LinkConfig(gn=uwb.GnSolverConfig(n_r=n_r, mean_step_density=density))


def test_non_uniform_grid_raises_where_the_reference_validates(engine):
    fibre = uwb.default_fibre()
    g = _cband()
    g.freq = g.freq.copy()
    g.freq[5] += 1e9  # still ascending, no longer equally spaced
    zg = uwb.build_distance_grid(fibre.length_m, 0.5)
    with pytest.raises(uwb.ConfigError, match="equally spaced"):
        uwb.solve_power_evolution(fibre, g, zg, engine=engine)
    with pytest.raises(uwb.ConfigError, match="equally spaced"):
        uwb.evaluate_link(fibre, g, _lc(), engine=engine)
    with pytest.raises(uwb.ConfigError, match="equally spaced"):
        uwb.ResidentLink(fibre, g, _lc(), engine=engine)


def test_half_band_smaller_than_hull_raises(engine):
    fibre = uwb.default_fibre()
    g = _cband()
    g.half_band = g.half_band - 10e9
    with pytest.raises(uwb.ConfigError, match="half_band"):
        uwb.evaluate_link(fibre, g, _lc(), engine=engine)
    zg = uwb.build_distance_grid(fibre.length_m, 0.5)
    with pytest.raises(uwb.ConfigError, match="half_band"):
        uwb.solve_power_evolution(fibre, g, zg, engine=engine)


def test_valid_grid_still_evaluates(engine):
    rep = uwb.evaluate_link(uwb.default_fibre(), _cband(), _lc(), engine=engine)
    assert np.all(rep.eta > 0)


def _profiles(base, rng):
    """Four launch profiles over the same grid: channels 2 and 7 dark in the
    first (the prepared one), lit in the second, 4 dark in the third, all lit
    in the fourth."""
    p = []
    for dark in ([2, 7], [], [4], []):
        x = base * (1.0 + 0.3 * rng.random(base.size))
        x[dark] = 0.0
        p.append(x)
    return np.stack(p)


@pytest.mark.parametrize("simpson", [False, True])
def test_batch_where_dark_channels_light_up_equals_single_calls(engine, simpson):
    fibre = uwb.default_fibre()
    g = _cband()
    rng = np.random.default_rng(11)
    prof = _profiles(np.array(g.psd), rng)
    lc = _lc()
    lc.gn.simpson_channel_average = simpson
    g.psd = prof[0].copy()  # prepare with channels 2 and 7 dark
    res = uwb.ResidentLink(fibre, g, lc, engine=engine)
    loss, reps = res.run_many(prof, reports=True)
    n = g.size()
    for k in range(len(prof)):
        gk = g.copy()
        gk.psd = prof[k].copy()
        one = uwb.evaluate_link(fibre, gk, lc, engine=engine)
        eta = reps[k][:n]
        assert np.array_equal(eta > 0, prof[k] > 0), k
        np.testing.assert_allclose(eta, one.eta, rtol=1e-12, atol=0)
        np.testing.assert_allclose(reps[k][2 * n:3 * n], one.snr_db, rtol=0, atol=1e-10)
        assert loss[k] == pytest.approx(one.loss_value, rel=1e-12)


def test_resident_call_where_dark_channel_lights_up(engine):
    """Same contract through uwb_evaluate_link_resident (device buffers)."""
    import torch

    fibre = uwb.default_fibre()
    g = _cband()
    lit = np.array(g.psd)
    dark = lit.copy()
    dark[[0, 5]] = 0.0
    g.psd = dark.copy()
    res = uwb.ResidentLink(fibre, g, _lc(), engine=engine)
    n = g.size()
    psd = torch.tensor(lit, dtype=torch.float64, device="cuda:0")
    out = torch.zeros(res.report_len, dtype=torch.float64, device="cuda:0")
    res.run(psd.data_ptr(), out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    g2 = g.copy()
    g2.psd = lit.copy()
    one = uwb.evaluate_link(fibre, g2, _lc(), engine=engine)
    o = out.cpu().numpy()
    assert np.all(o[:n] > 0)
    np.testing.assert_allclose(o[:n], one.eta, rtol=1e-12)
    assert res.report_len == 4 * n + 3 + 2 * uwb.gn_integral.N_BANDS
