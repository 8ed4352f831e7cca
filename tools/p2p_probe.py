"""Time the cross-rank elite exchange alone (torchrun, 2+ GPUs): p2p kernel vs NCCL all-gather + merge.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/p2p_probe.py
"""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2509_00217_b200.config import load_workload  # noqa: E402
from paper_2509_00217_b200.dist import ShardedSweep  # noqa: E402
from paper_2509_00217_b200.evaluator import Evaluator  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
ev = Evaluator(load_workload("moe_1p6t_h100x2048"), device=rank)
n = 1 << 20
g = torch.Generator(device="cuda")
g.manual_seed(rank)
planes = torch.empty((len(ev.head_sizes), n), dtype=torch.uint8, device="cuda")
for h, k in enumerate(ev.head_sizes):
    planes[h] = torch.randint(0, k, (n,), generator=g, device="cuda", dtype=torch.uint8)
words = ev.pack(planes)
for transport in ("nccl", "p2p"):
    sw = ShardedSweep(ev, k=8, transport=transport)
    _, recs, count = sw.run(words, index_base=rank * n)
    for reps in (1, 200):
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record()
        for _ in range(reps):
            r2, c2 = sw.merge(recs, count)
        b.record()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / reps * 1e6
        if rank == 0:
            print(f"{transport:5s} reps {reps:4d}: {a.elapsed_time(b) / reps * 1e3:8.1f} us/exchange (device), "
                  f"{wall:8.1f} us (wall)  count {int(c2.item())}", flush=True)
dist.destroy_process_group()
