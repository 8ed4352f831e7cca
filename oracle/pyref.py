"""Time the reference's own Python evaluator on this host.

TEST INFRASTRUCTURE / CPU BASELINE ONLY (see oracle/__init__.py): bench.py
uses it for its CPU-baseline figures, never on the measured GPU path.

The reference package (``shardsearch``) is not part of this repo: it is
installed once, git-ignored, into ``baseline/_ref`` and
travels to the GPU box with the snapshot. Per candidate this runs exactly
what the reference's ``SearchEnv.step`` runs to score one strategy —
``decode_strategy`` (strategy.py:245-263) then ``simulate(SimRequest(...))``
(env.py:140-150, simulator.py:239-341) — in ``multiprocessing.Pool(P)``
(BASELINE.md §3), and returns the verdicts so the caller can compare them
with the GPU's.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import platform
import sys
import time
from pathlib import Path

import numpy as np

REF_ROOT = Path(__file__).resolve().parent.parent / "baseline" / "_ref"
_CODES = {"none": 0, "over_device_budget": 1, "layout_error": 2, "oom": 3, "slo_violation": 4}
_W = {}


def available() -> bool:
    return (REF_ROOT / "shardsearch" / "simulator.py").exists()


def _init(ref_root: str, cfg_path: str) -> None:
    if ref_root not in sys.path:
        sys.path.insert(0, ref_root)
    from shardsearch.config import load_config
    from shardsearch.simulator import SimRequest, simulate
    from shardsearch.strategy import decode_strategy

    cfg = load_config(cfg_path)
    _W.update(cfg=cfg, SimRequest=SimRequest, simulate=simulate, decode=decode_strategy)


def _score(vectors) -> tuple[np.ndarray, np.ndarray]:
    cfg, simulate, SimRequest, decode = _W["cfg"], _W["simulate"], _W["SimRequest"], _W["decode"]
    reason = np.empty(len(vectors), np.uint8)
    thr = np.empty(len(vectors), np.float64)
    for i, v in enumerate(vectors):
        s = decode(tuple(int(x) for x in v), cfg.space)
        r = simulate(SimRequest(model=cfg.model, hw=cfg.hardware, strategy=s,
                                context_len=cfg.simulation.context_len, slo_tpot=cfg.simulation.slo_tpot))
        reason[i] = _CODES[r.invalid_reason.value]
        thr[i] = r.throughput
    return reason, thr


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def time_reference(cfg_path: str, planes: np.ndarray, procs: int | None = None) -> dict:
    """Score the [A, n] candidates with the reference in Pool(procs); rate + verdicts."""
    procs = procs or os.cpu_count() or 1
    vecs = np.ascontiguousarray(planes.T)
    n = vecs.shape[0]
    chunks = np.array_split(vecs, procs * 4)
    ctx = mp.get_context("fork")
    with ctx.Pool(procs, initializer=_init, initargs=(str(REF_ROOT), str(cfg_path))) as pool:
        pool.map(_score, [c[:64] for c in chunks[:procs]])  # imports + first calls in every worker
        t0 = time.perf_counter()
        parts = pool.map(_score, chunks)
        el = time.perf_counter() - t0
    reason = np.concatenate([p[0] for p in parts])
    thr = np.concatenate([p[1] for p in parts])
    return {"value": n / el, "seconds": el, "n": n, "procs": procs, "per_core": n / el / procs,
            "python": platform.python_version(), "cpu": cpu_model(), "reason": reason, "throughput": thr}
