"""In-run parity checks of bench.py against the CPU oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): bench.py calls this after
its timed region, as the checker of what the GPU arm produced — never inside
the measurement.

* ``batch_parity``: regenerate a rank's whole batch on the host (the uniform
  stream twin, oracle/streams.c), score it with the C restatement of
  simulate() (simulator.py:239-341) and compare every reason byte and every
  raw float64 bit pattern with the GPU's verdicts; compute the oracle's top-k
  by raw over distinct vectors (build_report(by_raw) order, ppo.py:441-447:
  raw desc, earliest index first, first occurrence of a vector kept).
* ``rescore_elites``: every elite record's stream index regenerated and its
  vector re-scored by the oracle: same vector, valid, same raw bits.
* ``merge_topk``: the cross-rank merge rule on oracle lists.
"""

from __future__ import annotations

import numpy as np

from .cost_model import simulate_planes, uniform_planes


def vector_codes(planes: np.ndarray, head_sizes) -> np.ndarray:
    """Mixed-radix code of each column (head 0 most significant) — ls_elite_rec.code."""
    code = np.zeros(planes.shape[1], dtype=np.int64)
    for h, k in enumerate(head_sizes):
        code = code * int(k) + planes[h].astype(np.int64)
    return code


def _topk_sorted(raws: np.ndarray, idx: np.ndarray, codes: np.ndarray, k: int):
    order = np.lexsort((idx, -raws))
    raws, idx, codes = raws[order], idx[order], codes[order]
    _, first = np.unique(codes, return_index=True)
    keep = np.sort(first)[:k]
    return [(float(raws[i]), int(idx[i]), int(codes[i])) for i in keep]


def batch_parity(desc, head_sizes, seed: int, base: int, reason: np.ndarray, thr: np.ndarray, k: int,
                 threads: int) -> dict:
    """Whole-batch comparison of GPU verdicts (reason u8, throughput f64) for stream
    positions [base, base + n) with the oracle; returns counts and the oracle top-k."""
    n = reason.shape[0]
    planes = uniform_planes(desc, seed, base, n, threads=threads)
    want = simulate_planes(desc, planes, threads=threads, fields=("throughput",))
    bad_reason = int(np.count_nonzero(want["reason"] != reason))
    bad_raw = int(np.count_nonzero(want["throughput"].view(np.uint64) != thr.view(np.uint64)))
    valid = np.flatnonzero(want["reason"] == 0)
    codes = vector_codes(planes[:, valid], head_sizes)
    topk = _topk_sorted(want["throughput"][valid], valid.astype(np.int64) + base, codes, k)
    return {"checked": n, "reason_mismatches": bad_reason, "raw_mismatches": bad_raw,
            "valid": int(valid.size), "oracle_topk": topk}


def merge_topk(lists, k: int):
    """Merge per-rank (raw, index, code) lists: raw desc, index asc, distinct codes."""
    flat = [r for lst in lists for r in lst]
    if not flat:
        return []
    raws = np.asarray([r[0] for r in flat], dtype=np.float64)
    idx = np.asarray([r[1] for r in flat], dtype=np.int64)
    codes = np.asarray([r[2] for r in flat], dtype=np.int64)
    return _topk_sorted(raws, idx, codes, k)


def rescore_elites(desc, seed: int, elites) -> int:
    """Mismatches among elite records (vector, raw, index): the stream position must
    regenerate the record's vector, and the oracle must score it valid with that raw."""
    bad = 0
    for e in elites:
        planes = uniform_planes(desc, seed, e.index, 1, threads=1)
        if tuple(int(x) for x in planes[:, 0]) != tuple(e.vector):
            bad += 1
            continue
        r = simulate_planes(desc, planes, threads=1, fields=("throughput",))
        if int(r["reason"][0]) != 0 or r["throughput"].view(np.uint64)[0] != np.float64(e.raw).view(np.uint64):
            bad += 1
    return bad
