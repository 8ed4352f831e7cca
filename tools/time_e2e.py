"""e2e host-buffer throughput of Evaluator.evaluate_host_packed (pinned in/out).

    LS_HOST_CHUNK_LOG2=22 LS_HOST_PIPE=3 python tools/time_e2e.py
"""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_00217_b200.config import load_workload  # noqa: E402
from paper_2509_00217_b200.evaluator import Evaluator, pinned_results  # noqa: E402

n = 1 << 26
ev = Evaluator(load_workload("moe_1p6t_h100x2048"), device=0)
rng = np.random.default_rng(0)
planes = np.stack([rng.integers(0, k, size=n, dtype=np.uint8) for k in ev.head_sizes])
words = ev.pack(torch.from_numpy(planes).cuda())
host = torch.empty(n, dtype=torch.int64).pin_memory()
host.copy_(words.cpu())
hp = host.numpy()
out = pinned_results(n)
ev.evaluate_host_packed(hp, out=out)
t0 = time.perf_counter()
for _ in range(5):
    ev.evaluate_host_packed(hp, out=out)
dt = (time.perf_counter() - t0) / 5
print(f"chunk 2^{os.environ.get('LS_HOST_CHUNK_LOG2', 'def')} pipe {os.environ.get('LS_HOST_PIPE', 'def')}: "
      f"{n / dt / 1e9:.2f} G evals/s  ({17 * n / dt / 1e9:.1f} GB/s over PCIe)")
