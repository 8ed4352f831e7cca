"""Timeline of four back-to-back fused evaluate + elite launches (the bench
step) from the LS_DIAG_TIMES build: per launch, per-CTA phase stamps.

    tools/build_variant.sh diag "-DLS_DIAG_TIMES"
    LS_EVAL_LIB=ab/libls_eval_diag.so python tools/phase_pdl.py [n]

Stamps: 0 entry, 1 tables ready, 2 gate warp 0 done, 3 fp64 warp 0 done,
4 drain barrier, 5 CTA list published, 6 final merge start, 7 final merge done.
"""
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_00217_b200 import _native  # noqa: E402
from paper_2509_00217_b200.config import load_workload  # noqa: E402
from paper_2509_00217_b200.evaluator import Evaluator  # noqa: E402
from paper_2509_00217_b200.generator import GEN_UNIFORM  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1 << 27
ev = Evaluator(load_workload("moe_1p6t_h100x2048"), device=0)
lib = _native.lib()
words = ev.pack(ev.generate(GEN_UNIFORM, n, seed=0))
out = ev._alloc(n, ("throughput",))
buf = np.zeros((1024, 16), dtype=np.uint64)
for rep in range(3):
    lib.ls_diag_times(ctypes.c_void_p(buf.ctypes.data), 1024)  # also rewinds the launch counter
    torch.cuda.synchronize()
    for _ in range(4):
        ev.evaluate_packed_topk(words, k=8, out=out)
    torch.cuda.synchronize()
lib.ls_diag_times(ctypes.c_void_p(buf.ctypes.data), 1024)
t = buf.astype(np.int64)
t0 = t[t[:, 0] > 0, 0].min()
names = ["entry", "tables", "gate0 done", "fp0 done", "drain bar", "cta list", "final start", "final done"]
for L in range(4):
    rows = t[256 * L: 256 * L + 256]
    rows = rows[rows[:, 0] > 0]
    print(f"launch {L}: {len(rows)} CTAs")
    for j, name in enumerate(names):
        col = rows[:, j][rows[:, j] > 0]
        if len(col):
            col = (col - t0) / 1e3
            print(f"   {name:12s} min {col.min():9.2f}  median {np.median(col):9.2f}  max {col.max():9.2f} us")
