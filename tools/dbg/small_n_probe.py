"""Per-call cost of the fused step at small n: eager Python calls vs one CUDA graph."""
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
    for _ in range(3):
        ev.evaluate_packed_topk(words, k=8, out=out, into=into)
    torch.cuda.synchronize()
    reps = 200
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        ev.evaluate_packed_topk(words, k=8, out=out, into=into)
    b.record(); torch.cuda.synchronize()
    eager = a.elapsed_time(b) / reps * 1e3
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(20):
                ev.evaluate_packed_topk(words, k=8, out=out, into=into)
    torch.cuda.synchronize()
    g.replay(); torch.cuda.synchronize()
    a.record()
    for _ in range(reps // 20):
        g.replay()
    b.record(); torch.cuda.synchronize()
    graph = a.elapsed_time(b) / reps * 1e3
    print(f"n={n:>9}: eager {eager:7.2f} us/call  graph {graph:7.2f} us/call", flush=True)
