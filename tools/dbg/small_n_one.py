"""One fused step at n (default 1e4) after a warm-up: for an ncu capture of the fixed per-launch cost."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch
from paper_2509_00217_b200.config import load_workload
from paper_2509_00217_b200.evaluator import Evaluator

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**4
ev = Evaluator(load_workload("moe_1p6t_h100x2048"), device=0)
planes = torch.stack([torch.randint(0, k, (n,), device="cuda", dtype=torch.uint8) for k in ev.head_sizes])
words = ev.pack(planes)
out = ev._alloc(n, ("throughput",))
for _ in range(3):
    ev.evaluate_packed_topk(words, k=8, out=out)
torch.cuda.synchronize()
print("ok")
