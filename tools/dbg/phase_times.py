"""Phase timeline of the fused evaluate+elite kernel from the LS_DIAG_TIMES build.

    tools/build_variant.sh diag "-DLS_DIAG_TIMES"
    LS_EVAL_LIB=ab/libls_eval_diag.so python tools/dbg/phase_times.py [n ...]

Stamps (globaltimer, per CTA): 0 entry, 1 gate table ready, 2 gate warp 0 done,
3 fp64 warp 0 done, 4 work warps past the drain barrier, 5 CTA list merge done,
6 last CTA starts the final merge, 7 final merge done, 8 CTA lists staged in
shared memory, 9 first head scan, 10 merge loop done (11: its round count).
"""
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_00217_b200 import _native  # noqa: E402
from paper_2509_00217_b200.config import load_workload  # noqa: E402
from paper_2509_00217_b200.evaluator import Evaluator  # noqa: E402

ev = Evaluator(load_workload("moe_1p6t_h100x2048"), device=0)
lib = _native.lib()
for n in [int(float(x)) for x in sys.argv[1:]] or [10**4, 10**6, 1 << 27]:
    planes = torch.stack([torch.randint(0, k, (n,), device="cuda", dtype=torch.uint8) for k in ev.head_sizes])
    words = ev.pack(planes)
    del planes
    out = ev._alloc(n, ("throughput",))
    for k in (8, 1):
        for _ in range(3):
            ev.evaluate_packed_topk(words, k=k, out=out)
        torch.cuda.synchronize()
        buf = np.zeros((1024, 16), dtype=np.uint64)
        lib.ls_diag_times(ctypes.c_void_p(buf.ctypes.data), 1024)
        grid = int((buf[:, 0] > 0).sum())
        t = buf[:grid].astype(np.int64)
        t0 = t[:, 0].min()
        rel = (t - t0) / 1e3
        last = int(np.argmax(t[:, 7]))
        print(f"n={n} k={k} grid={grid}")
        for j, name in enumerate(["entry", "table", "gate0 done", "fp0 done", "drain bar", "cta merge",
                                  "final start", "final done", "staged", "first scan", "merge loop"]):
            col = rel[:, j] if j < 6 else rel[last:last + 1, j]
            print(f"   {name:12s} min {col.min():8.2f}  median {np.median(col):8.2f}  max {col.max():8.2f} us")
        print(f"   final merge rounds {int(buf[last, 11])}")
        buf[:] = 0
        torch.cuda.synchronize()
