"""Multi-GPU contexts at the C-ABI (uwb_ctx_create_multi): the reference's
worker pool (GnSolverConfig::workers -> parallel_for_batches, parallel.hpp:
21-47) with GPUs as the workers.

The reference's contract is bit-identity for any worker count
(test_gn_integral.cpp:291-300, acceptance C2/C10).  On the one-GPU test box
several sub-contexts on device 0 stand in for several GPUs: the channel
split, the per-device ODE, the cudaMemcpyPeerAsync eta gather and the
lead's report all run exactly as on an 8-GPU node (a peer copy between two
contexts of one device is a device-to-device copy).
"""
import numpy as np
import pytest

import paper_2401_18022_b200 as uwb
from helpers import cfg_of, engine_inputs_from_oracle, product_scenario
from pyoracle import Case, cband11, oband11

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def multi():
    eng = uwb.Engine(devices=[0, 0, 0])
    yield eng
    eng.close()


def test_width(multi, engine):
    assert multi.width() == 3 and engine.width() == 1


@pytest.mark.parametrize("simpson", [0, 1])
def test_all_channels_nli_split_is_bit_identical(multi, engine, oracle, simpson):
    case = oband11(n_r=40, density=0.95, simpson=simpson)
    prep = oracle.prepare(case)
    grid, spans, betas, gamma = engine_inputs_from_oracle(prep, case.density)
    one = uwb.all_channels_nli(grid, spans, betas, None, cfg_of(case), engine=engine, gamma=gamma)
    for _ in range(2):  # the second call is balanced by the first call's measured work
        r = uwb.all_channels_nli(grid, spans, betas, None, cfg_of(case), engine=multi, gamma=gamma)
        assert np.array_equal(r.eta, one.eta)
        assert np.array_equal(r.quadrant, one.quadrant)
        assert np.array_equal(r.skipped, one.skipped)
    st = multi.last_partition_stats()
    assert st["first_channel"][0] == 0 and st["first_channel"] == sorted(st["first_channel"])


def test_channel_work_cost_model(multi, engine, oracle):
    """The per-channel |K|^2 counts the split balances on are the device's own
    (summed over the devices they equal the single-device counts)."""
    case = cband11(n_r=30, density=0.95)
    prep = oracle.prepare(case)
    grid, spans, betas, gamma = engine_inputs_from_oracle(prep, case.density)
    uwb.all_channels_nli(grid, spans, betas, None, cfg_of(case), engine=engine, gamma=gamma)
    w1 = engine.last_channel_work(grid.size())
    uwb.all_channels_nli(grid, spans, betas, None, cfg_of(case), engine=multi, gamma=gamma)
    wm = multi.last_channel_work(grid.size())
    assert np.all(w1 > 0)
    assert np.array_equal(w1, wm)
    assert w1.sum() == engine.last_nli_stats()["evaluated_points"]


def test_evaluate_link_split_is_bit_identical(multi, engine, golden):
    rec = golden["evaluate_link"]["uwb589_random_launch"]
    case = Case.from_json(rec["case"])
    grid, fibre = product_scenario(case)
    lc = uwb.LinkConfig(gn=cfg_of(case))
    one = uwb.evaluate_link(fibre, grid, lc, engine=engine)
    rep = uwb.evaluate_link(fibre, grid, lc, engine=multi)
    assert np.array_equal(rep.eta, one.eta)
    assert np.array_equal(rep.snr_db, one.snr_db)
    assert rep.loss_value == one.loss_value
    assert rep.total_capacity == one.total_capacity
    assert np.array_equal(rep.band_capacity, one.band_capacity)
    st = multi.last_partition_stats()
    assert all(ms > 0 for ms in st["nli_ms"]) and all(ms > 0 for ms in st["ode_ms"])


def test_resident_and_batch_on_multi(multi, engine, golden):
    import torch

    rec = golden["evaluate_link"]["uwb589_random_launch"]
    case = Case.from_json(rec["case"])
    grid, fibre = product_scenario(case)
    lc = uwb.LinkConfig(gn=uwb.GnSolverConfig(n_r=20, mean_step_density=0.95))
    r1 = uwb.ResidentLink(fibre, grid, lc, engine=engine)
    rm = uwb.ResidentLink(fibre, grid, lc, engine=multi)
    assert rm.report_len == r1.report_len
    psd = torch.tensor(grid.psd, dtype=torch.float64, device="cuda:0")
    o1 = torch.zeros(r1.report_len, dtype=torch.float64, device="cuda:0")
    om = torch.zeros(rm.report_len, dtype=torch.float64, device="cuda:0")
    st = torch.cuda.current_stream().cuda_stream
    r1.run(psd.data_ptr(), o1.data_ptr(), st)
    rm.run(psd.data_ptr(), om.data_ptr(), st)
    torch.cuda.synchronize()
    rm.check_status()
    assert torch.equal(o1, om)
    # batches deal whole evaluations over the devices
    rng = np.random.default_rng(5)
    base = np.array(grid.psd)
    prof = np.stack([base * (1.0 + 0.3 * rng.random(base.size)) for _ in range(7)])
    l1, p1 = r1.run_many(prof, reports=True)
    lm, pm = rm.run_many(prof, reports=True)
    assert np.array_equal(l1, lm) and np.array_equal(p1, pm)


def test_single_device_stages_are_rejected(multi):
    with pytest.raises(uwb.ConfigError):
        multi.set_channel_subset([1, 2])
