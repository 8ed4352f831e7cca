"""On-device stream sweeps (0 B of candidate input) for timing and ncu.

    python tools/prof_sweep.py [--config moe_1p2t_h100] [--mode 3] [--n 0 (= whole stream)] [--reps 3]
mode 1 = uniform, 2 = full enumeration, 3 = admissible-axis enumeration.
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2509_00217_b200.config import load_workload  # noqa: E402
from paper_2509_00217_b200.evaluator import Evaluator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="moe_1p2t_h100")
ap.add_argument("--mode", type=int, default=3)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--k", type=int, default=8)
ap.add_argument("--fp32", action="store_true", help="the fp32 fast mode (ls_set_precision)")
args = ap.parse_args()
ev = Evaluator(load_workload(args.config), device=0)
if args.fp32:
    ev.set_precision("fp32")
n = args.n or (ev.stream_size(args.mode) if args.mode != 1 else 1 << 30)
recs, count = ev.sweep(args.mode, n, k=args.k)  # warm (stream tables, scratch)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(args.reps):  # back to back: device time per sweep, not host launch latency
    recs, count = ev.sweep(args.mode, n, k=args.k)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / args.reps
print(f"sweep mode {args.mode} {args.config} n={n}: {ms:.3f} ms  {n / ms / 1e6:.2f} G evals/s (device time, "
      f"{args.reps} back-to-back)", flush=True)
best = ev.decode_records(recs, count)[0]
print("best", best.vector, best.raw, best.index)
