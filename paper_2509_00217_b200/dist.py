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
  while the next batch is evaluated, so the exchange is off the critical
  path;
* reward shaping across ranks (``SearchEnv.step`` semantics, env.py:159-164):
  each rank needs the best valid raw of all EARLIER ranks as its starting
  baseline — one all-gather of one float per rank.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch
import torch.distributed as dist

from ._native import check

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

    launches_per_merge = 2  # without grouping: the NCCL all-gather kernel + ls_topk_merge (per step)

    def __init__(self, evaluator, k: int = 8, group=None, overlap: bool = False, group_steps: int = 4,
                 reserve_sms: int = 0, transport: str = "nccl", lap_steps: int = 16):
        """``overlap``: run the exchanges on a side stream so the caller's stream goes
        straight on to the next batch; ``wait()`` joins it. With packed words the
        exchange is batched: every ``group_steps`` steps the side stream waits ONCE
        for the last launch's completion signal (ls_stream_wait_signal), all-gathers
        the group's per-rank lists in one collective and merges each step's — a wait
        on the side stream costs ~15 us of the next fused launch's overlap, so it is
        paid once per group. The global elite of a step is ready at ``wait()``.
        ``reserve_sms``: SMs the fused launches leave free for the side stream's
        kernels (ls_reserve_sms); 0 measured fastest (NCCL's kernel starts as the
        fused CTAs exit at a step boundary; one reserved SM cost 0.3 %).
        ``transport="p2p"`` (packed words, ``overlap``, one node; every rank falls back
        to the NCCL exchange when any rank cannot map its peers' memory): no collective at
        all — each fused launch's last CTA writes its elite block straight into
        every rank's exchange ring (peer HBM mapped with CUDA IPC, NVLink), and
        each rank merges a lap of ``lap_steps`` steps in one launch that first
        waits on the device for the blocks' sequence words (``_merge_pending``,
        at lap boundaries and in ``wait()``). The ring holds two laps, so a rank
        can never overwrite blocks its peer has not merged yet."""
        self.ev = evaluator
        self.k = int(k)
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        dev = evaluator.device
        self.transport = "local" if self.world == 1 else "nccl"
        self.overlap = bool(overlap) and self.world > 1
        G = max(1, int(group_steps)) if self.overlap else 1
        self.group_steps = G
        nbuf = 2 * G if self.overlap else 1  # two groups in flight
        rows = self.k + 1  # one message per rank and step: k records + a row holding the count
        self._sendbuf = torch.zeros((nbuf, rows, 32), dtype=torch.uint8, device=dev)
        self._sends = [self._sendbuf[i] for i in range(nbuf)]
        self._gathered = [torch.empty((self.world * G * rows, 32), dtype=torch.uint8, device=dev)
                          for _ in range(2 if self.overlap else 1)]
        self._mrecs = torch.zeros((nbuf, self.k, 32), dtype=torch.uint8, device=dev)
        self._mcount = torch.zeros(nbuf, dtype=torch.int32, device=dev)
        self._merged = [(self._mrecs[i], self._mcount[i:i + 1]) for i in range(nbuf)]
        self._free = [None, None]  # side-stream event per group: its buffers no longer read
        self._grp = 0       # group being filled
        self._in_grp = 0    # steps launched into it
        self._last = 0      # slot of the last launched step
        self._seq = 0
        self._signal = torch.zeros(1, dtype=torch.int32, device=dev)  # last fused launch whose elite is written
        self._side = torch.cuda.Stream(dev) if self.overlap else None
        if self.overlap and reserve_sms:
            evaluator.reserve_sms(int(reserve_sms))
        if transport not in ("nccl", "p2p"):
            raise ValueError(f"unknown transport {transport!r}")
        self._opened: list[int] = []
        if transport == "p2p" and self.overlap:
            self._setup_p2p(max(1, int(lap_steps)))

    def _setup_p2p(self, S: int) -> None:
        """The exchange ring [world][2S][k + 1][32 B] in this rank's HBM, every peer's
        ring mapped through CUDA IPC, and per slot the device array of the sinks a
        step's fused launch writes to (slot t % 2S of every rank's ring, row block
        ``rank``)."""
        lib, dev, rows = self.ev._lib, self.ev.device, self.k + 1
        slots = 2 * S
        self._lap, self._slots = S, slots
        # the ring is its own cudaMalloc (ls_ipc_alloc): an IPC handle maps an allocation's base,
        # and a tensor from torch's caching allocator may sit inside a larger segment
        ring = ctypes.c_void_p()
        check(lib.ls_ipc_alloc(self.world * slots * rows * 32, ctypes.byref(ring)))
        self._ring_ptr = ring.value
        h = (ctypes.c_char * 64)()
        check(lib.ls_ipc_handle(ring, h))
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(h), group=self.group)
        bases, ok = [], 1
        for r, hr in enumerate(handles):
            if r == self.rank:
                bases.append(self._ring_ptr)
                continue
            p = ctypes.c_void_p()
            if lib.ls_ipc_open(ctypes.create_string_buffer(hr, 64), ctypes.byref(p)) != 0:
                ok = 0  # e.g. ranks on different nodes, or IPC not permitted
                break
            self._opened.append(p.value)
            bases.append(p.value)
        flag = torch.tensor([ok], dtype=torch.int32, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)  # every rank takes the same transport
        if not int(flag.item()):
            for q in self._opened:
                lib.ls_ipc_close(ctypes.c_void_p(q))
            self._opened = []
            dist.barrier(group=self.group)
            lib.ls_ipc_free(ctypes.c_void_p(self._ring_ptr))
            self._ring_ptr = None
            return  # the grouped NCCL exchange stays in place
        blk = rows * 32
        table = [[b + ((self.rank * slots) + j) * blk for b in bases] for j in range(slots)]
        self._sinks = torch.tensor(table, dtype=torch.int64, device=dev)
        self._p_send = torch.zeros((slots, rows, 32), dtype=torch.uint8, device=dev)  # this rank's own block per step
        self._p_recs = torch.zeros((slots, self.k, 32), dtype=torch.uint8, device=dev)
        self._p_count = torch.zeros(slots, dtype=torch.int32, device=dev)
        self._err = torch.zeros(1, dtype=torch.int32, device=dev)
        self._t = 0        # steps launched
        self._merged_upto = 0
        self.transport = "p2p"
        dist.barrier(group=self.group)  # every ring is mapped before any rank writes into one

    def _run_p2p(self, words: torch.Tensor, index_base: int, out, verdicts: bool):
        if out is None or not verdicts:
            raise ValueError("the p2p exchange runs prepared launches: pass out= and verdicts=True")
        if self._t % self._lap == 0:
            self._merge_pending()  # the previous lap, before this lap's blocks reach any ring
        slot = self._t % self._slots
        self._last = slot
        plan = self._plan_for(words, index_base, out, self._p_send[slot], None, self._sinks[slot])
        self._t += 1
        plan(self._t)  # seq = step number + 1 (never 0: fresh rings hold zeros)
        return out, self._p_recs[slot], self._p_count[slot:slot + 1]

    def _merge_pending(self) -> None:
        """Merge the steps launched since the last merge, each after every rank's block arrived."""
        lo, hi = self._merged_upto, self._t
        rows, st = self.k + 1, torch.cuda.current_stream(self.ev.device).cuda_stream
        while lo < hi:  # contiguous slot ranges of the ring
            j0 = lo % self._slots
            n = min(hi - lo, self._slots - j0)
            check(self.ev._lib.ls_topk_merge_steps_wait(
                ctypes.c_void_p(self._ring_ptr + j0 * rows * 32), self.world, n, self._slots, self.k, lo + 1,
                ctypes.c_void_p(self._p_recs[j0].data_ptr()), ctypes.c_void_p(self._p_count[j0:].data_ptr()),
                ctypes.c_void_p(self._err.data_ptr()), ctypes.c_void_p(st)))
            lo += n
        self._merged_upto = hi

    def check(self) -> None:
        """Raise if a p2p merge timed out waiting for a peer's block (synchronises)."""
        if self.transport == "p2p" and int(self._err.item()):
            raise RuntimeError("p2p elite exchange: a peer's block did not arrive within ~10 s")

    def close(self) -> None:
        """Unmap the peers' exchange rings and free this rank's (p2p; collective: every rank calls it)."""
        if self.transport != "p2p" or not getattr(self, "_ring_ptr", None):
            return
        torch.cuda.synchronize(self.ev.device)
        for p in self._opened:
            self.ev._lib.ls_ipc_close(ctypes.c_void_p(p))
        self._opened = []
        dist.barrier(group=self.group)  # no peer maps this ring any more
        self.ev._lib.ls_ipc_free(ctypes.c_void_p(self._ring_ptr))
        self._ring_ptr = None

    @property
    def _send(self) -> torch.Tensor:
        """The send block the next evaluation writes into (k records + count row)."""
        return self._sends[self._grp * self.group_steps + self._in_grp]

    def run(self, candidates: torch.Tensor, index_base: int, out=None, verdicts: bool = True):
        """Score this rank's candidates (global indices index_base..) and return the global elite.

        ``candidates``: [A, n] uint8 planes, or n packed 64-bit words.
        Returns (out, recs, count) with recs/count the merged global top-k on device
        (with ``overlap``, valid on the caller's stream only after ``wait()``).
        """
        if self.world == 1:
            if candidates.dim() == 1:
                if out is not None and verdicts:  # repeated steps over the same buffers: a prepared launch
                    recs, count = self._plan_for(candidates, index_base, out, None, None)()
                    return out, recs, count
                return self.ev.evaluate_packed_topk(candidates, k=self.k, index_base=index_base, out=out,
                                                    verdicts=verdicts)
            return self.ev.evaluate_topk(candidates, k=self.k, index_base=index_base, out=out, verdicts=verdicts)
        if self.transport == "p2p" and candidates.dim() == 1:
            return self._run_p2p(candidates, index_base, out, verdicts)
        cur = torch.cuda.current_stream(self.ev.device)
        if self._in_grp == 0 and self._free[self._grp] is not None and not self._free[self._grp].query():
            cur.wait_event(self._free[self._grp])  # the group's previous exchange still reads it (rare)
        slot = self._grp * self.group_steps + self._in_grp
        into = self._sends[slot]
        self._last = slot
        if candidates.dim() == 1 and self.overlap:
            self._seq += 1
            if out is not None and verdicts:
                self._plan_for(candidates, index_base, out, into, self._signal)(self._seq)
            else:
                out, _, _ = self.ev.evaluate_packed_topk(candidates, k=self.k, index_base=index_base, out=out,
                                                         verdicts=verdicts, into=into, signal=self._signal,
                                                         seq=self._seq)
            self._in_grp += 1
            if self._in_grp == self.group_steps:
                self._flush()
            return out, self._merged[slot][0], self._merged[slot][1]
        if candidates.dim() == 1:
            out, recs, count = self.ev.evaluate_packed_topk(candidates, k=self.k, index_base=index_base, out=out,
                                                            verdicts=verdicts, into=into)
        else:
            out, recs, count = self.ev.evaluate_topk(candidates, k=self.k, index_base=index_base, out=out,
                                                     verdicts=verdicts, into=into)
        recs, count = self.merge(recs, count)
        return out, recs, count

    def _plan_for(self, words, index_base, out, into, signal, sinks=None):
        """The prepared fused launch for these buffers (one per send slot), rebuilt when they change."""
        plans = self.__dict__.setdefault("_plans", {})
        slot_key = None if into is None else into.data_ptr()
        p = plans.get(slot_key)
        st = torch.cuda.current_stream(self.ev.device).cuda_stream
        recs_ptr = into.data_ptr() if into is not None else (p.recs.data_ptr() if p is not None else None)
        key = (words.data_ptr(), words.shape[0], self.k, index_base, recs_ptr,
               (out.reason.data_ptr(), out.throughput.data_ptr() if out.throughput is not None else 0), st,
               None if signal is None else signal.data_ptr(), None if sinks is None else sinks.data_ptr())
        if p is None or p.key != key:
            p = self.ev.fused_plan(words, k=self.k, out=out, into=into, index_base=index_base, signal=signal,
                                   sinks=sinks)
            p.key = key
            plans[slot_key] = p
        return p

    def _flush(self):
        """Exchange the steps launched into the current group (side stream)."""
        n, g, G, rows = self._in_grp, self._grp, self.group_steps, self.k + 1
        if n == 0:
            return
        self.ev.wait_signal(self._signal, self._seq, stream=self._side)
        gathered = self._gathered[g][: self.world * n * rows]
        with torch.cuda.stream(self._side):
            dist.all_gather_into_tensor(gathered, self._sendbuf[g * G: g * G + n].reshape(n * rows, 32),
                                        group=self.group)
            # rank r's block of step j starts at row (r * n + j) * rows: one merge launch for the group
            check(self.ev._lib.ls_topk_merge_steps(ctypes.c_void_p(gathered.data_ptr()), self.world, n, self.k,
                                                   ctypes.c_void_p(self._mrecs[g * G].data_ptr()),
                                                   ctypes.c_void_p(self._mcount[g * G:].data_ptr()),
                                                   ctypes.c_void_p(self._side.cuda_stream)))
            done = torch.cuda.Event()
            done.record(self._side)
        self._free[g] = done
        self._grp ^= 1
        self._in_grp = 0

    def merge(self, recs: torch.Tensor, count: torch.Tensor):
        """All-gather every rank's device top-k (k x 32 B + count) in ONE collective and merge on device."""
        if self.world == 1:
            return recs, count
        slot = self._last
        send = self._sends[slot]
        if recs.data_ptr() != send.data_ptr():  # not produced in place by run()
            send[: self.k].copy_(recs)
            send[self.k, :4].view(torch.int32).copy_(count)
        gathered = self._gathered[0][: self.world * (self.k + 1)]
        if self._side is None:
            dist.all_gather_into_tensor(gathered, send, group=self.group)
            return self._merge_gathered(gathered, self._merged[slot])
        ready = torch.cuda.Event()
        ready.record(torch.cuda.current_stream(self.ev.device))
        self._side.wait_event(ready)
        with torch.cuda.stream(self._side):
            dist.all_gather_into_tensor(gathered, send, group=self.group)
            res = self._merge_gathered(gathered, self._merged[slot])
        torch.cuda.current_stream(self.ev.device).wait_stream(self._side)  # planes: no pipelining
        return res

    def _merge_gathered(self, gathered: torch.Tensor, into):
        g = gathered.view(self.world, self.k + 1, 32)
        counts = g[:, self.k, :4].contiguous().view(torch.int32).reshape(self.world)
        # each rank's list is k_in = k + 1 slots; the count row is never read (count <= k)
        return self.ev.merge_records(gathered, counts, self.k + 1, self.k, into=into)

    def last_local(self):
        """(records, count) this rank contributed to the most recent exchange."""
        send = self._p_send[self._last] if self.transport == "p2p" else self._sends[self._last]
        return send[: self.k], send[self.k, :4].view(torch.int32)

    def wait(self) -> None:
        """Exchange what is still pending and make the caller's stream wait for every exchange."""
        if self.transport == "p2p":
            self._merge_pending()
            return
        if self._side is not None:
            self._flush()
            torch.cuda.current_stream(self.ev.device).wait_stream(self._side)
