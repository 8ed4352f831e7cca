"""Multi-GPU sharding of batched evaluation (one process per GPU).

Candidates are independent — ``simulate`` is pure (reference SPEC.md:241) —
so a batch shards by contiguous global index ranges with no data-path
communication. Only two small exchanges cross ranks:

* the elite: every rank reduces its shard to a top-k on device
  (``Evaluator.evaluate_topk``); the per-rank blocks (k records + count, one
  message) go through ONE NCCL all-gather over NVLink/NVSwitch and are merged
  on device with ``ls_topk_merge``; contiguous ranges keep "earliest global
  index wins" consistent, and the merge rule is exact for any arrival order.
  With ``overlap=True`` the all-gather and the merge run on a side stream
  while the next batch is evaluated (the evaluate kernels leave one SM free
  for them, ``ls_reserve_sms``), so the exchange is off the critical path;
* reward shaping across ranks (``SearchEnv.step`` semantics, env.py:159-164):
  each rank needs the best valid raw of all EARLIER ranks as its starting
  baseline — one all-gather of one float per rank.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch
import torch.distributed as dist

__all__ = ["shard_range", "exclusive_prefix_best", "ShardedSweep", "SweepResult"]


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) slice of n global candidates owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    return n * rank // world, n * (rank + 1) // world


def exclusive_prefix_best(local_best: float, b0: float, group=None) -> tuple[float, float]:
    """(baseline for this rank, best over all ranks) for the exclusive running max.

    ``local_best`` is this rank's best valid raw (or -inf when none). Works on
    any backend (gloo for the CPU tests, NCCL on GPUs).
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = torch.device("cpu") if dist.get_backend(group) == "gloo" else torch.device("cuda", torch.cuda.current_device())
    mine = torch.tensor([local_best], dtype=torch.float64, device=dev)
    allv = torch.empty(world, dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(allv, mine, group=group)
    vals = allv.cpu().tolist()
    base = max([b0] + vals[:rank])
    return base, max([b0] + vals)


@dataclass
class SweepResult:
    elites: list  # list[Elite], best first
    local_count: int


class ShardedSweep:
    """Evaluate a globally indexed batch split across ranks and merge the elite."""

    launches_per_merge = 2  # the NCCL all-gather kernel + ls_topk_merge

    def __init__(self, evaluator, k: int = 8, group=None, overlap: bool = False):
        """``overlap``: run each step's exchange on a side stream so the caller's
        stream goes straight on to the next batch; ``wait()`` joins it."""
        self.ev = evaluator
        self.k = int(k)
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        dev = evaluator.device
        self.transport = "local" if self.world == 1 else "nccl"
        self.overlap = bool(overlap) and self.world > 1
        nbuf = 4 if self.overlap else 1
        # one message per rank: k records + a 32-byte row holding the count
        self._sends = [torch.zeros((self.k + 1, 32), dtype=torch.uint8, device=dev) for _ in range(nbuf)]
        self._gathered = [torch.empty((self.world * (self.k + 1), 32), dtype=torch.uint8, device=dev)
                          for _ in range(nbuf)]
        self._merged = [(torch.empty((self.k, 32), dtype=torch.uint8, device=dev),
                         torch.zeros(1, dtype=torch.int32, device=dev)) for _ in range(nbuf)]
        self._free = [None] * nbuf  # side-stream event: slot's buffers no longer read
        self._slot = 0
        self._seq = 0
        self._signal = torch.zeros(1, dtype=torch.int32, device=dev)  # last fused launch whose elite is written
        self._side = torch.cuda.Stream(dev) if self.overlap else None
        if self.overlap:
            evaluator.reserve_sms(1)

    @property
    def _send(self) -> torch.Tensor:
        """The send block the next evaluation writes into (k records + count row)."""
        return self._sends[self._slot]

    def run(self, candidates: torch.Tensor, index_base: int, out=None, verdicts: bool = True):
        """Score this rank's candidates (global indices index_base..) and return the global elite.

        ``candidates``: [A, n] uint8 planes, or n packed 64-bit words.
        Returns (out, recs, count) with recs/count the merged global top-k on device
        (with ``overlap``, valid on the caller's stream only after ``wait()``).

        With ``overlap`` and packed words, nothing but the fused launch is put on the
        caller's stream: the side stream waits for the launch's completion signal
        (ls_stream_wait_signal), so consecutive launches keep overlapping (PDL).
        """
        cur = torch.cuda.current_stream(self.ev.device)
        free = self._free[self._slot]
        if self.world > 1 and free is not None and not free.query():
            cur.wait_event(free)  # the slot's previous exchange is still reading it (rare)
        into = self._send if self.world > 1 else None
        if candidates.dim() == 1:
            sig = None
            if self.overlap:
                self._seq += 1
                sig = self._signal
            out, recs, count = self.ev.evaluate_packed_topk(candidates, k=self.k, index_base=index_base, out=out,
                                                            verdicts=verdicts, into=into, signal=sig, seq=self._seq)
        else:
            out, recs, count = self.ev.evaluate_topk(candidates, k=self.k, index_base=index_base, out=out,
                                                     verdicts=verdicts, into=into)
        recs, count = self.merge(recs, count, signalled=candidates.dim() == 1)
        return out, recs, count

    def merge(self, recs: torch.Tensor, count: torch.Tensor, signalled: bool = False):
        """All-gather every rank's device top-k (k x 32 B + count) in ONE collective and merge on device."""
        if self.world == 1:
            return recs, count
        slot = self._slot
        send = self._sends[slot]
        if recs.data_ptr() != send.data_ptr():  # not produced in place by run()
            send[: self.k].copy_(recs)
            send[self.k, :4].view(torch.int32).copy_(count)
            signalled = False
        gathered = self._gathered[slot]
        cur = torch.cuda.current_stream(self.ev.device)
        if self._side is None:
            dist.all_gather_into_tensor(gathered, send, group=self.group)
            return self._merge_gathered(gathered, self._merged[slot])
        if signalled and self.overlap:
            self.ev.wait_signal(self._signal, self._seq, stream=self._side)
        else:
            ready = torch.cuda.Event()
            ready.record(cur)
            self._side.wait_event(ready)
        with torch.cuda.stream(self._side):
            dist.all_gather_into_tensor(gathered, send, group=self.group)
            res = self._merge_gathered(gathered, self._merged[slot])
            done = torch.cuda.Event()
            done.record(self._side)
        self._free[slot] = done
        self._slot = (slot + 1) % len(self._sends)
        return res

    def _merge_gathered(self, gathered: torch.Tensor, into):
        g = gathered.view(self.world, self.k + 1, 32)
        counts = g[:, self.k, :4].contiguous().view(torch.int32).reshape(self.world)
        # each rank's list is k_in = k + 1 slots; the count row is never read (count <= k)
        return self.ev.merge_records(gathered, counts, self.k + 1, self.k, into=into)

    def last_local(self):
        """(records, count) this rank contributed to the most recent exchange."""
        send = self._sends[(self._slot - 1) % len(self._sends)] if self.overlap else self._sends[0]
        return send[: self.k], send[self.k, :4].view(torch.int32)

    def wait(self) -> None:
        """Make the caller's stream wait for every exchange issued so far."""
        if self._side is not None:
            torch.cuda.current_stream(self.ev.device).wait_stream(self._side)
