"""Two-GPU sharded sweep over NCCL: per-rank fused evaluate + elite, all-gather
of the per-rank records, device merge — must equal the single-GPU elite of the
whole batch. Skipped on boxes with fewer than 2 GPUs."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_two(target, args, attempts=3):
    """Run target(rank, 2, port, *args, q) on two spawned ranks and return rank 0's
    result; a rank that dies early (e.g. the rendezvous port was taken between
    _free_port and the bind) restarts the pair on a fresh port."""
    import queue
    import time

    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    for attempt in range(attempts):
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=target, args=(r, 2, port, *args[:-1], q, *args[-1])) for r in range(2)]
        for p in procs:
            p.start()
        t0, res = time.time(), None
        while res is None and time.time() - t0 < 300:
            try:
                res = q.get(timeout=1)
            except queue.Empty:
                if any(p.exitcode not in (None, 0) for p in procs):
                    break
        if res is None:
            for p in procs:
                p.terminate()
                p.join(timeout=30)
            if attempt + 1 < attempts:
                continue
            raise AssertionError("the two-rank run failed")
        for p in procs:
            p.join(timeout=120)
            assert p.exitcode == 0
        return res


def _worker(rank, world, port, n, k, q, packed=False, overlap=False):
    import torch.distributed as dist

    from paper_2509_00217_b200.config import load_workload
    from paper_2509_00217_b200.dist import ShardedSweep, shard_range
    from paper_2509_00217_b200.evaluator import Evaluator

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        wl = load_workload("moe_1p6t_h100x2048")
        ev = Evaluator(wl, device=rank)
        rng = np.random.default_rng(11)
        planes = np.stack([rng.integers(0, s, size=n, dtype=np.uint8) for s in ev.head_sizes])
        lo, hi = shard_range(n, rank, world)
        mine = torch.from_numpy(np.ascontiguousarray(planes[:, lo:hi])).cuda(rank)
        if packed:  # 8-byte candidate words (the bench's resident format)
            mine = ev.pack(mine)
        sweep = ShardedSweep(ev, k=k, overlap=overlap)
        for _ in range(3):  # repeated steps exercise both slots of the overlapped exchange
            _, recs, count = sweep.run(mine, index_base=lo)
        sweep.wait()
        elites = ev.decode_records(recs, count)
        local = ev.decode_records(*sweep.last_local())
        topk = ev.evaluate_packed_topk if packed else ev.evaluate_topk
        _, r0, c0 = topk(mine, k=k, index_base=lo)
        assert local == ev.decode_records(r0, c0)
        if rank == 0:
            whole = torch.from_numpy(planes).cuda(rank)
            _, r1, c1 = ev.evaluate_topk(whole, k=k)
            q.put(([(e.vector, e.raw, e.index) for e in elites],
                   [(e.vector, e.raw, e.index) for e in ev.decode_records(r1, c1)]))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("overlap", [False, True])
@pytest.mark.parametrize("packed", [False, True])
@pytest.mark.parametrize("k", [3, 8])
def test_two_gpu_elite_equals_single_gpu(k, packed, overlap):
    merged, single = _run_two(_worker, (5_000_003, k, (packed, overlap)))
    assert merged == single and len(merged) == k


def _worker_p2p(rank, world, port, n, k, q, steps, lap):
    import torch.distributed as dist

    from paper_2509_00217_b200.config import load_workload
    from paper_2509_00217_b200.dist import ShardedSweep, shard_range
    from paper_2509_00217_b200.evaluator import BatchResult, Evaluator

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        wl = load_workload("moe_1p6t_h100x2048")
        ev = Evaluator(wl, device=rank)
        rng = np.random.default_rng(12)
        planes = np.stack([rng.integers(0, s, size=n, dtype=np.uint8) for s in ev.head_sizes])
        lo, hi = shard_range(n, rank, world)
        mine = ev.pack(torch.from_numpy(np.ascontiguousarray(planes[:, lo:hi])).cuda(rank))
        out = BatchResult(reason=torch.empty(hi - lo, dtype=torch.uint8, device=rank),
                          throughput=torch.empty(hi - lo, dtype=torch.float64, device=rank))
        sweep = ShardedSweep(ev, k=k, overlap=True, transport="p2p", lap_steps=lap)
        assert sweep.transport == "p2p"
        results = []
        for _ in range(steps):  # several laps: the ring wraps and every lap merges after its peers' blocks
            _, recs, count = sweep.run(mine, index_base=lo, out=out)
            results.append((recs, count))
        sweep.wait()
        torch.cuda.synchronize()
        sweep.check()
        last = [ev.decode_records(r, c) for r, c in results[-min(steps, 2 * lap):]]  # slots not yet reused
        _, r0, c0 = ev.evaluate_packed_topk(mine, k=k, index_base=lo)
        assert ev.decode_records(*sweep.last_local()) == ev.decode_records(r0, c0)
        if rank == 0:
            whole = torch.from_numpy(planes).cuda(rank)
            _, r1, c1 = ev.evaluate_topk(whole, k=k)
            single = [(e.vector, e.raw, e.index) for e in ev.decode_records(r1, c1)]
            q.put(([[(e.vector, e.raw, e.index) for e in el] for el in last], single))
        dist.barrier()
        sweep.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("steps,lap", [(3, 16), (11, 2)])
@pytest.mark.parametrize("k", [3, 8])
def test_two_gpu_p2p_exchange_equals_single_gpu(k, steps, lap):
    """The peer-memory exchange (the fused launch writes its elite into every rank's
    ring over NVLink, laps merged after a device-side wait on the blocks' sequence
    words): every step's merged elite equals the single-GPU elite of the batch."""
    merged, single = _run_two(_worker_p2p, (3_000_017, k, (steps, lap)))
    assert len(single) == k
    for m in merged:
        assert m == single
