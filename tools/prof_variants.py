"""Plain vs fused-top-k evaluation of the same packed batch, for an ncu launch list:

    ncu --metrics gpu__time_duration.sum --csv python tools/prof_variants.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2509_00217_b200.config import load_workload  # noqa: E402
from paper_2509_00217_b200.evaluator import BatchResult, Evaluator  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 27
ev = Evaluator(load_workload("moe_1p6t_h100x2048"), device=0)
g = torch.Generator(device="cuda")
g.manual_seed(0)
planes = torch.empty((len(ev.head_sizes), n), dtype=torch.uint8, device="cuda")
for h, k in enumerate(ev.head_sizes):
    planes[h] = torch.randint(0, k, (n,), generator=g, device="cuda", dtype=torch.uint8)
words = ev.pack(planes)
del planes
out = BatchResult(reason=torch.empty(n, dtype=torch.uint8, device="cuda"),
                  throughput=torch.empty(n, dtype=torch.float64, device="cuda"))
for _ in range(3):
    ev.evaluate_packed(words, out=out)
for _ in range(3):
    ev.evaluate_packed_topk(words, k=8, out=out)
torch.cuda.synchronize()
print("done")
