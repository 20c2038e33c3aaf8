"""CPU, world_size 2 over gloo: the multi-GPU data path's host logic.

Each rank evaluates only its partition of the channels (here with the oracle
standing in for the GPU kernel -- test-only), the per-rank eta vectors are
combined by the same allreduce_eta the bench uses, and the result must be
bit-identical to a single-process run (the reference's bit-identity across
worker counts, test_gn_integral.cpp:291-300)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2401_18022_b200.multigpu import (EtaGather, active_channels, allreduce_eta,
                                            partition_channels)


def test_partition_covers_and_balances():
    ch = np.arange(557)
    for world in (1, 2, 3, 4, 8):
        parts = partition_channels(ch, world)
        allc = np.sort(np.concatenate(parts))
        assert np.array_equal(allc, ch)
        sizes = [len(p) for p in parts]
        assert max(sizes) - min(sizes) <= 1
    cost = np.linspace(1.0, 1.32, 557)  # O-band edge COIs are heavier
    parts = partition_channels(ch, 8, cost)
    loads = [cost[np.isin(ch, p)].sum() for p in parts]
    assert max(loads) / min(loads) < 1.02  # one item of granularity
    assert np.array_equal(np.sort(np.concatenate(parts)), ch)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.join(os.path.dirname(here), "oracle"))
    from pyoracle import Oracle, cband11

    O = Oracle()
    case = cband11(n_r=24, density=0.95, workers=1)
    prep = O.prepare(case)
    ga = prep["grid_arrays"]

    class G:
        guard = ga["guard"]
        psd = ga["psd"]

    parts = partition_channels(active_channels(G), world)
    mine = parts[rank]
    full = O.all_channels_nli(case, prep)
    eta = torch.zeros(len(ga["freq"]), dtype=torch.float64)
    # rank-local evaluation: only this rank's channels are non-zero
    eta[mine] = torch.from_numpy(full["eta"][mine])
    eta2 = eta.clone()
    allreduce_eta(eta)
    # the bench's exchange: one all-gather of the packed per-rank slices (an
    # uneven LPT deal, so the padding path is exercised too)
    cost = np.arange(len(ga["freq"]), dtype=np.float64)[active_channels(G)] ** 2
    parts2 = partition_channels(active_channels(G), world, cost)
    eta3 = torch.zeros_like(eta2)
    eta3[parts2[rank]] = torch.from_numpy(full["eta"][parts2[rank]])
    EtaGather(parts2, rank, torch.device("cpu")).gather(eta3)
    if rank == 0:
        q.put((eta.numpy().copy(), full["eta"], eta3.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_allreduce_is_bit_identical():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, want, gathered = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(got, want)
    assert np.array_equal(gathered, want)


def _gpu_worker(rank, world, port, q):
    """One rank of the real sharded evaluation: the engine's kernels on cuda:0
    (both ranks share the one GPU of the test box -- their kernels never wait
    on each other; the exchange is a host-side gloo all-reduce), then the
    same all-reduce + SNR report as bench.py's NCCL path."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2401_18022_b200 as uwb
    from paper_2401_18022_b200.multigpu import ShardedLink

    torch.cuda.set_device(0)
    eng = uwb.Engine(0)
    grid = uwb.make_default_uwb_grid()
    uwb.set_uniform_launch(grid, 1e-3)
    lc = uwb.LinkConfig(gn=uwb.GnSolverConfig(n_r=24, mean_step_density=0.95))
    sh = ShardedLink(uwb.default_fibre(), grid, lc, rank, world, engine=eng)
    st = torch.cuda.Stream()
    psd = torch.tensor(grid.psd, dtype=torch.float64, device="cuda:0")
    rep = torch.zeros(sh.report_len, dtype=torch.float64, device="cuda:0")
    with torch.cuda.stream(st):
        sh.run(psd.data_ptr(), rep.data_ptr(), st.cuda_stream)
    torch.cuda.synchronize()
    sh.check_status()
    first = rep.cpu().numpy().copy()
    # re-deal by LPT on the per-channel work both ranks measured, run again
    cost = sh.rebalance()
    with torch.cuda.stream(st):
        sh.run(psd.data_ptr(), rep.data_ptr(), st.cuda_stream)
    torch.cuda.synchronize()
    sh.check_status()
    if rank == 0:
        q.put((first, rep.cpu().numpy().copy(), float(np.sum(cost)), sh.balance()))
    dist.barrier()
    dist.destroy_process_group()
    eng.close()


@pytest.mark.gpu
def test_two_rank_sharded_link_matches_single_gpu():
    import paper_2401_18022_b200 as uwb

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, again, total_work, balance = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    eng = uwb.Engine(0)
    grid = uwb.make_default_uwb_grid()
    uwb.set_uniform_launch(grid, 1e-3)
    lc = uwb.LinkConfig(gn=uwb.GnSolverConfig(n_r=24, mean_step_density=0.95))
    one = uwb.evaluate_link(uwb.default_fibre(), grid, lc, engine=eng)
    eng.close()
    n = grid.size()
    assert np.array_equal(got[:n], one.eta)          # bit-identical eta
    assert np.array_equal(got[2 * n:3 * n], one.snr_db)
    assert got[4 * n] == one.loss_value
    # the cost-balanced (LPT on measured per-channel work) re-deal changes
    # nothing but the balance
    assert np.array_equal(again, got)
    assert total_work > 0 and balance is not None and balance < 1.01
