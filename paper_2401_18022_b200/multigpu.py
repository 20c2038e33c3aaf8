"""Multi-GPU channel partition (one process per GPU, torch.distributed).

The reference's only parallelism is channel-level data parallelism over host
threads (parallel_for_batches, parallel.hpp:21-47): every channel writes only
its own output slot, so results are bit-identical for any worker count
(test_gn_integral.cpp:291-300).  The B200 version keeps that contract across
GPUs:

* each rank runs the (tiny, replicated) Raman ODE and the NLI of its own
  channels -- no collective inside the data path;
* the per-channel eta vectors (zeros outside each rank's channels) are
  combined by ONE all-reduce(sum) -- x + 0 == x exactly, so the result is
  bit-identical to a single-GPU run whatever the partition;
* the SNR report is then assembled on every rank from the full vector.

Partitioning: channels are dealt by longest-processing-time (LPT) on a cost
model (default: uniform -- adjacent channels have near-equal cost, so a
round-robin deal balances to ~1 %).
"""
from __future__ import annotations

import heapq

import numpy as np


def partition_channels(channels, world: int, cost=None) -> list[np.ndarray]:
    """Split `channels` into `world` sorted index arrays, LPT on `cost`.

    Deterministic: ties are broken by channel order, then rank.
    """
    channels = np.asarray(channels, dtype=np.int64)
    if world < 1:
        raise ValueError("world must be >= 1")
    if cost is None:
        # uniform cost: round-robin deal (the LPT schedule for equal weights)
        return [np.sort(channels[r::world]) for r in range(world)]
    cost = np.asarray(cost, dtype=np.float64)
    if cost.shape != channels.shape:
        raise ValueError("cost must match channels")
    order = sorted(range(len(channels)), key=lambda i: (-cost[i], channels[i]))
    heap = [(0.0, r) for r in range(world)]
    parts = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        parts[r].append(channels[i])
        heapq.heappush(heap, (load + cost[i], r))
    return [np.sort(np.asarray(p, dtype=np.int64)) for p in parts]


def active_channels(grid) -> np.ndarray:
    """Channels all_channels_nli evaluates (gn_integral.hpp:349-352)."""
    return np.flatnonzero((np.asarray(grid.guard) == 0) & (np.asarray(grid.psd) > 0.0))


def allreduce_eta(eta, group=None):
    """Sum the per-rank eta vectors in place (zeros outside each rank's
    channels).  Works for CUDA tensors (NCCL) and CPU tensors (gloo)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(eta, op=dist.ReduceOp.SUM, group=group)
    return eta


class ShardedLink:
    """Full SNR evaluation on N GPUs: this rank's share of the channels.

    Wraps gn_integral.ResidentLink: run(psd_dev) = noise (ODE + this rank's
    NLI) -> NCCL all-reduce of eta -> SNR report (device-resident throughout).
    """

    def __init__(self, fibre, grid, cfg, rank: int, world: int, engine=None, cost=None):
        import torch

        from .gn_integral import ResidentLink, get_engine

        self.rank, self.world = rank, world
        self.eng = engine or get_engine()
        self.parts = partition_channels(active_channels(grid), world, cost)
        self.mine = self.parts[rank]
        self.eng.set_channel_subset(self.mine if world > 1 else None)
        self.res = ResidentLink(fibre, grid, cfg, engine=self.eng)
        ptr, n = self.res.eta_buffer()
        dev = torch.device("cuda", torch.cuda.current_device())

        class _Cai:  # zero-copy torch view of the engine's eta buffer
            __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                        "version": 3}

        self.eta = torch.as_tensor(_Cai(), device=dev)
        self.report_len = self.res.report_len

    def run(self, psd_ptr: int, report_ptr: int, stream_ptr: int) -> int:
        """One evaluation; returns the number of engine kernel launches."""
        if self.world == 1:
            self.res.run(psd_ptr, report_ptr, stream_ptr)
            return self.eng.last_launches()
        self.res.run_noise(psd_ptr, stream_ptr)
        n = self.eng.last_launches()
        allreduce_eta(self.eta)
        self.res.run_report(report_ptr, stream_ptr)
        return n + self.eng.last_launches()

    def check_status(self):
        self.res.check_status()
