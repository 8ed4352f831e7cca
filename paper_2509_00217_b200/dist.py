"""Multi-GPU sharding of batched evaluation (one process per GPU).

Candidates are independent — ``simulate`` is pure (reference SPEC.md:241) —
so a batch shards by contiguous global index ranges with no data-path
communication. Only two small exchanges cross ranks:

* the elite: every rank reduces its shard to a top-k on device
  (``Evaluator.evaluate_topk``); the per-rank blocks (k records + count, one
  message) go through ONE NCCL all-gather and are merged on device with
  ``ls_topk_merge`` — or, opt-in, are exchanged over peer memory and merged
  in one kernel (``ls_elite_exchange``: LL-tagged P2P stores into every
  rank's symmetric buffer over NVLink/NVSwitch, then the merge); contiguous
  ranges keep "earliest global index wins" consistent, and the merge rule is
  exact for any arrival order;
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

    def __init__(self, evaluator, k: int = 8, group=None, transport: str = "auto"):
        """``transport``: "nccl" (one all-gather + the merge kernel; the
        default, "auto") or "p2p" (peer-memory exchange fused with the merge,
        ``ls_elite_exchange``). The p2p kernel is exact (same tests) but, as
        measured on the B200 boxes of round 1, its peer stores/polls over the
        torch symmetric-memory mapping take ~1.3 ms per exchange against
        ~70 µs for NCCL, so it is opt-in until that is understood."""
        self.ev = evaluator
        self.k = int(k)
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        dev = evaluator.device
        # one message per rank: k records + a 32-byte row holding the count
        self._send = torch.empty((self.k + 1, 32), dtype=torch.uint8, device=dev)
        self._gathered = torch.empty((self.world * (self.k + 1), 32), dtype=torch.uint8, device=dev)
        self.transport = "local" if self.world == 1 else "nccl"
        if self.world > 1 and transport == "p2p":
            try:
                self._init_p2p(dev)
                self.transport = "p2p"
            except Exception:
                if transport == "p2p":
                    raise

    def _init_p2p(self, dev):
        import torch.distributed._symmetric_memory as symm

        lib = self.ev._lib
        nbytes = int(lib.ls_elite_exchange_bytes(self.world, self.k))
        if nbytes == 0 or self.world > 8 or self.k > 32:
            raise ValueError("p2p elite exchange supports world <= 8 and k <= 32")
        self._buf = symm.empty(nbytes, dtype=torch.uint8, device=dev)
        self._buf.zero_()
        torch.cuda.synchronize(dev)
        self._hdl = symm.rendezvous(self._buf, self.group if self.group is not None else dist.group.WORLD)
        self._peer_bases = torch.tensor([int(p) for p in self._hdl.buffer_ptrs], dtype=torch.int64, device=dev)
        self._seq = 0
        self._out = torch.empty((self.k, 32), dtype=torch.uint8, device=dev)
        self._count = torch.empty(1, dtype=torch.int32, device=dev)
        dist.barrier(self.group)  # every buffer is zeroed before any rank pushes

    def run(self, candidates: torch.Tensor, index_base: int, out=None, verdicts: bool = True):
        """Score this rank's candidates (global indices index_base..) and return the global elite.

        ``candidates``: [A, n] uint8 planes, or n packed 64-bit words.
        Returns (out, recs, count) with recs/count the merged global top-k on device.
        """
        into = self._send if self.world > 1 else None
        if candidates.dim() == 1:
            out, recs, count = self.ev.evaluate_packed_topk(candidates, k=self.k, index_base=index_base, out=out,
                                                            verdicts=verdicts, into=into)
        else:
            out, recs, count = self.ev.evaluate_topk(candidates, k=self.k, index_base=index_base, out=out,
                                                     verdicts=verdicts, into=into)
        recs, count = self.merge(recs, count)
        return out, recs, count

    def merge(self, recs: torch.Tensor, count: torch.Tensor):
        """All-gather every rank's device top-k (k x 32 B + count) in ONE collective and merge on device."""
        if self.world == 1:
            return recs, count
        if recs.data_ptr() != self._send.data_ptr():  # not produced in place by run()
            self._send[: self.k].copy_(recs)
            self._send[self.k, :4].view(torch.int32).copy_(count)
        if self.transport == "p2p":
            from ._native import check

            self._seq += 1
            check(self.ev._lib.ls_elite_exchange(
                ctypes.c_void_p(self._send.data_ptr()), ctypes.c_void_p(self._peer_bases.data_ptr()),
                ctypes.c_void_p(self._buf.data_ptr()), self.rank, self.world, self.k, self._seq,
                ctypes.c_void_p(self._out.data_ptr()), ctypes.c_void_p(self._count.data_ptr()),
                self.ev._stream()))
            return self._out, self._count
        dist.all_gather_into_tensor(self._gathered, self._send, group=self.group)
        g = self._gathered.view(self.world, self.k + 1, 32)
        counts = g[:, self.k, :4].contiguous().view(torch.int32).reshape(self.world)
        # each rank's list is k_in = k + 1 slots; the count row is never read (count <= k)
        return self.ev.merge_records(self._gathered, counts, self.k + 1, self.k)
