"""Small standalone checks of the top-k paths (debug helper)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2509_00217_b200.config import load_workload
from paper_2509_00217_b200.evaluator import Evaluator

which = sys.argv[1]
wl = load_workload("moe_1p2t_h100")
ev = Evaluator(wl, device=0)
rng = np.random.default_rng(0)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
planes = torch.from_numpy(np.stack([rng.integers(0, k, size=n, dtype=np.uint8) for k in ev.head_sizes])).cuda()
res = ev.evaluate(planes)
torch.cuda.synchronize()
print("evaluate ok", int((res.reason == 0).sum()))
if which == "topk":
    e = ev.topk(planes, res.reason, res.throughput, k=int(sys.argv[3]))
    torch.cuda.synchronize()
    print("topk ok", e[:2])
elif which == "fused":
    out, recs, count = ev.evaluate_topk(planes, k=int(sys.argv[3]))
    torch.cuda.synchronize()
    print("fused ok", ev.decode_records(recs, count)[:2])
