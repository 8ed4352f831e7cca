"""In-stream timing of the elite merge and of evaluate with / without the fused top-k.

    python tools/time_merge.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_00217_b200.config import load_workload  # noqa: E402
from paper_2509_00217_b200.evaluator import BatchResult, Evaluator  # noqa: E402


def timed(fn, reps=50):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


ev = Evaluator(load_workload("moe_1p6t_h100x2048"), device=0)
for m in (() if "--no-merge" in sys.argv else (8, 296, 2960)):
    rng = np.random.default_rng(0)
    rec = np.zeros(m * 8, dtype=[("key", "f8"), ("raw", "f8"), ("index", "i8"), ("code", "u8")])
    rec["key"] = np.sort(rng.random(m * 8).reshape(m, 8), axis=1)[:, ::-1].ravel()
    rec["raw"] = rec["key"]
    rec["index"] = np.arange(m * 8)
    rec["code"] = rng.integers(0, 1 << 40, m * 8)
    recs = torch.from_numpy(rec.view(np.uint8).reshape(m * 8, 32).copy()).cuda()
    counts = torch.full((m,), 8, dtype=torch.int32, device="cuda")
    print(f"merge m={m:5d} lists x 8: {timed(lambda: ev.merge_records(recs, counts, 8, 8)):7.1f} us")

n = 1 << 27
g = torch.Generator(device="cuda")
g.manual_seed(0)
planes = torch.empty((len(ev.head_sizes), n), dtype=torch.uint8, device="cuda")
for h, k in enumerate(ev.head_sizes):
    planes[h] = torch.randint(0, k, (n,), generator=g, device="cuda", dtype=torch.uint8)
words = ev.pack(planes)
del planes
out = BatchResult(reason=torch.empty(n, dtype=torch.uint8, device="cuda"),
                  throughput=torch.empty(n, dtype=torch.float64, device="cuda"))
print(f"evaluate_packed          : {timed(lambda: ev.evaluate_packed(words, out=out), 20):7.1f} us")
print(f"evaluate_packed_topk k=8 : {timed(lambda: ev.evaluate_packed_topk(words, k=8, out=out), 20):7.1f} us")
print(f"sweep (no verdicts) k=8  : {timed(lambda: ev.evaluate_packed_topk(words, k=8, out=out, verdicts=False), 20):7.1f} us")
