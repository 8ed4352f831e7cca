import sys; sys.path.insert(0, '.')
import torch
from paper_2509_00217_b200.config import load_workload
from paper_2509_00217_b200.evaluator import Evaluator
ev = Evaluator(load_workload("moe_1p6t_h100x2048"), device=0)
n = 1 << 27
planes = torch.randint(0, 3, (len(ev.head_sizes), n), dtype=torch.uint8, device="cuda")
for _ in range(2): ev.pack(planes)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); a.record()
for _ in range(5): w = ev.pack(planes)
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 5
print(f"pack 2^27: {ms:.3f} ms  {24 * n / ms / 1e6:.0f} GB/s (16 B in + 8 B out per candidate)")
