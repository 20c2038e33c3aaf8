"""Multi-GPU channel partition (one process per GPU, torch.distributed).

The reference's only parallelism is channel-level data parallelism over host
threads (parallel_for_batches, parallel.hpp:21-47): every channel writes only
its own output slot, so results are bit-identical for any worker count
(test_gn_integral.cpp:291-300).  The B200 version keeps that contract across
GPUs:

* each rank runs the (tiny, replicated) Raman ODE and the NLI of its own
  channels -- no collective inside the data path;
* the per-channel eta values are exchanged by ONE all-gather: every rank
  packs its own channels' eta (in its partition order, padded to the largest
  share) and scatters the gathered slices into the full vector by the
  partition every rank knows -- pure copies, so the result is bit-identical to
  a single-GPU run whatever the partition;
* the SNR report is then assembled on every rank from the full vector.

Partitioning: channels are dealt by longest-processing-time (LPT) on a cost
model.  The first evaluation deals round-robin; ShardedLink.rebalance() then
takes the per-channel work every rank measured on its device (|K|^2
evaluations per channel, uwb_last_channel_work: the active points and the
heavier MCI-region channels near lambda_0), sums it over the
ranks with one all-reduce, and re-deals by LPT.  The C-ABI's own multi-GPU
context (uwb_ctx_create_multi, one process driving several GPUs) uses the same
measured cost with contiguous ranges.
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


class EtaGather:
    """The per-COI eta exchange as one all-gather (north star item 4).

    Rank r owns the channels parts[r]; pack() copies its values into a slot
    of width m = max |parts| and gather() all-gathers the [world, m] slots and
    scatters them back into the full eta vector by the (shared) partition.
    Works for CUDA tensors (NCCL) and CPU tensors (gloo)."""

    def __init__(self, parts, rank: int, device):
        import torch

        self.world, self.rank = len(parts), rank
        self.m = max(1, max(len(p) for p in parts))
        idx = np.zeros((self.world, self.m), dtype=np.int64)
        valid = np.zeros((self.world, self.m), dtype=bool)
        for r, p in enumerate(parts):
            idx[r, :len(p)] = p
            valid[r, :len(p)] = True
        self.mine = torch.as_tensor(np.asarray(parts[rank], dtype=np.int64), device=device)
        self.dst = torch.as_tensor(idx[valid], device=device)
        self.valid = torch.as_tensor(valid.reshape(-1), device=device)

    def gather(self, eta, group=None):
        import torch
        import torch.distributed as dist

        if not (dist.is_available() and dist.is_initialized()) or self.world == 1:
            return eta
        send = torch.zeros(self.m, dtype=eta.dtype, device=eta.device)
        send[:len(self.mine)] = eta[self.mine]
        recv = torch.empty(self.world * self.m, dtype=eta.dtype, device=eta.device)
        dist.all_gather_into_tensor(recv, send, group=group)
        eta[self.dst] = recv[self.valid]
        return eta


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
    NLI) -> NCCL all-gather of eta -> SNR report (device-resident throughout).
    """

    def __init__(self, fibre, grid, cfg, rank: int, world: int, engine=None, cost=None):
        self.rank, self.world = rank, world
        self.fibre, self.grid, self.cfg = fibre, grid, cfg
        from .gn_integral import get_engine

        self.eng = engine or get_engine()
        self._setup(cost)

    def _setup(self, cost):
        import torch

        from .gn_integral import ResidentLink

        grid, world, rank = self.grid, self.world, self.rank
        act = active_channels(grid)
        self.parts = partition_channels(act, world, None if cost is None else np.asarray(cost)[act])
        self.mine = self.parts[rank]
        self.eng.set_channel_subset(self.mine if world > 1 else None)
        self.res = ResidentLink(self.fibre, grid, self.cfg, engine=self.eng)
        ptr, n = self.res.eta_buffer()
        dev = torch.device("cuda", torch.cuda.current_device())

        class _Cai:  # zero-copy torch view of the engine's eta buffer
            __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                        "version": 3}

        self.eta = torch.as_tensor(_Cai(), device=dev)
        self.report_len = self.res.report_len
        self.exchange = EtaGather(self.parts, rank, dev)

    def rebalance(self):
        """Re-deal the channels by LPT on the per-channel work the last
        evaluation measured on every rank (one all-reduce of the cost
        vector).  Results do not change -- only the balance."""
        import torch
        import torch.distributed as dist

        n = self.grid.size()
        w = torch.tensor(self.eng.last_channel_work(n), dtype=torch.float64,
                         device=self.eta.device)
        if self.world > 1 and dist.is_available() and dist.is_initialized():
            dist.all_reduce(w, op=dist.ReduceOp.SUM)
        self.cost = w.cpu().numpy()
        self._setup(self.cost)
        return self.cost

    def balance(self):
        """max / mean of the measured cost over the ranks' shares (1.0 = even)."""
        c = getattr(self, "cost", None)
        if c is None:
            return None
        loads = [float(np.sum(c[p])) for p in self.parts]
        return max(loads) / (sum(loads) / len(loads)) if sum(loads) > 0 else None

    def run(self, psd_ptr: int, report_ptr: int, stream_ptr: int) -> int:
        """One evaluation; returns the number of engine kernel launches."""
        if self.world == 1:
            self.res.run(psd_ptr, report_ptr, stream_ptr)
            return self.eng.last_launches()
        self.res.run_noise(psd_ptr, stream_ptr)
        n = self.eng.last_launches()
        self.exchange.gather(self.eta)
        self.res.run_report(report_ptr, stream_ptr)
        return n + self.eng.last_launches()

    def check_status(self):
        self.res.check_status()
