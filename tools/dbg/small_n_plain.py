"""Plain packed evaluate vs fused evaluate+elite at small n (kernel time via CUDA events over many calls)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch
from paper_2509_00217_b200.config import load_workload
from paper_2509_00217_b200.evaluator import Evaluator

ev = Evaluator(load_workload("moe_1p6t_h100x2048"), device=0)
for n in (10**4, 10**5, 10**6, 10**7):
    planes = torch.stack([torch.randint(0, k, (n,), device="cuda", dtype=torch.uint8) for k in ev.head_sizes])
    words = ev.pack(planes)
    out = ev._alloc(n, ("throughput",))
    into = torch.zeros((9, 32), dtype=torch.uint8, device="cuda")
    res = {}
    for name, fn in (("plain", lambda: ev.evaluate_packed(words, out=out)),
                     ("fused", lambda: ev.evaluate_packed_topk(words, k=8, out=out, into=into)),
                     ("fused_k1", lambda: ev.evaluate_packed_topk(words, k=1, out=out))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(100):
            fn()
        b.record()
        torch.cuda.synchronize()
        res[name] = a.elapsed_time(b) * 10
    print(f"n={n:>9}: " + "  ".join(f"{k} {v:7.2f} us" for k, v in res.items()), flush=True)
