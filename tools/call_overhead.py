"""Host cost of one fused call at small n (back-to-back calls, wall clock per call)
and of the other small-batch entry points.

    python tools/call_overhead.py [--n 10000] [--calls 2000]
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_00217_b200.config import load_workload  # noqa: E402
from paper_2509_00217_b200.evaluator import Evaluator  # noqa: E402
from paper_2509_00217_b200.generator import GEN_UNIFORM  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10000)
ap.add_argument("--calls", type=int, default=2000)
args = ap.parse_args()
ev = Evaluator(load_workload("moe_1p6t_h100x2048"), device=0)
planes = ev.generate(GEN_UNIFORM, args.n, seed=0)
words = ev.pack(planes)
out = ev._alloc(args.n, ("throughput",))
recs = torch.empty((9, 32), dtype=torch.uint8, device="cuda")


def timeit(name, fn):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.calls):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name:34s} host {1e6 * (t1 - t0) / args.calls:7.2f} us/call, wall {1e6 * (t2 - t0) / args.calls:7.2f} us/call",
          flush=True)


timeit("evaluate_packed_topk(out, into)", lambda: ev.evaluate_packed_topk(words, k=8, out=out, into=recs))
timeit("evaluate_packed_topk(out)", lambda: ev.evaluate_packed_topk(words, k=8, out=out))
timeit("evaluate_packed(out)", lambda: ev.evaluate_packed(words, out=out))
timeit("evaluate(planes)", lambda: ev.evaluate(planes, out=out))
if hasattr(ev, "fused_plan"):
    p = ev.fused_plan(words, k=8, out=out, into=recs)
    timeit("fused_plan()", p)
