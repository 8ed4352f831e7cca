"""Minimal driver for ncu: evaluate one uniform batch a few times.

    python tools/prof_eval.py [--config moe_1p6t_h100x2048] [--n 33554432] [--reps 3] [--dist uniform|adm]
"""

import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2509_00217_b200.config import load_workload  # noqa: E402
from paper_2509_00217_b200.evaluator import BatchResult, Evaluator  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="moe_1p6t_h100x2048")
    ap.add_argument("--n", type=int, default=1 << 25)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--dist", default="uniform")
    ap.add_argument("--fields", default="raw")
    ap.add_argument("--topk", type=int, default=0, help="fused evaluate + elite of this size")
    ap.add_argument("--no-verdicts", action="store_true")
    ap.add_argument("--packed", action="store_true", help="8-byte candidate words instead of planes")
    args = ap.parse_args()
    wl = load_workload(args.config)
    ev = Evaluator(wl, device=0)
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    planes = torch.empty((len(ev.head_sizes), args.n), dtype=torch.uint8, device="cuda")
    for h, k in enumerate(ev.head_sizes):
        if args.dist == "adm" and h >= 4:
            k = 2  # UNSHARDED / DIM0 only: biased toward admissible layouts
        planes[h] = torch.randint(0, k, (args.n,), generator=g, device="cuda", dtype=torch.uint8)
    fields = ("throughput",) if args.fields == "raw" else "all"
    words = ev.pack(planes) if args.packed else None
    if words is not None:  # the first eval_ws_kernel launch is the packed one (ncu -c 1)
        del planes
        out = BatchResult(reason=torch.empty(args.n, dtype=torch.uint8, device="cuda"),
                          throughput=torch.empty(args.n, dtype=torch.float64, device="cuda"))
    else:
        out = ev.evaluate(planes, fields=fields)
    torch.cuda.synchronize()
    for _ in range(args.reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        if words is not None and args.topk:
            ev.evaluate_packed_topk(words, k=args.topk, out=out, verdicts=not args.no_verdicts)
        elif words is not None:
            ev.evaluate_packed(words, fields=fields, out=out)
        elif args.topk:
            ev.evaluate_topk(planes, k=args.topk, out=out, verdicts=not args.no_verdicts)
        else:
            ev.evaluate(planes, fields=fields, out=out)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        print(f"evaluate n={args.n} {ms:.3f} ms  {args.n / ms / 1e6:.3f} Gevals/s", flush=True)
    r = out.reason.bincount(minlength=5).cpu().tolist()
    print("reasons", r[:5])


if __name__ == "__main__":
    main()
