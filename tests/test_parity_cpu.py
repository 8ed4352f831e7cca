"""bench.py's in-run parity checker (oracle/parity.py) on the CPU: it must
count every reason / raw-bit mismatch it is shown, rank the oracle top-k by
(raw desc, index asc) over distinct vectors, merge per-rank lists by the same
rule, and reject elite records whose stream index, vector or raw is off."""

import numpy as np

from golden_io import load_eval
from oracle.cost_model import simulate_planes, uniform_planes
from oracle.parity import batch_parity, merge_topk, rescore_elites, vector_codes
from paper_2509_00217_b200.evaluator import Elite


def test_batch_parity_counts_mismatches_and_ranks_topk():
    wl, _, _ = load_eval("moe_1p6t_2048")
    desc, sizes = wl.desc(), wl.space.head_sizes
    n, base, seed = 200_000, 12345, 0
    planes = uniform_planes(desc, seed, base, n)
    truth = simulate_planes(desc, planes, fields=("throughput",))
    reason, thr = truth["reason"].copy(), truth["throughput"].copy()
    ok = batch_parity(desc, sizes, seed, base, reason, thr, 8, threads=2)
    assert ok["reason_mismatches"] == 0 and ok["raw_mismatches"] == 0 and ok["checked"] == n
    valid = np.flatnonzero(truth["reason"] == 0)
    order = valid[np.lexsort((valid, -truth["throughput"][valid]))]
    assert [t[1] - base for t in ok["oracle_topk"]][0] == order[0]
    assert all(a[0] >= b[0] for a, b in zip(ok["oracle_topk"], ok["oracle_topk"][1:]))
    codes = [t[2] for t in ok["oracle_topk"]]
    assert len(set(codes)) == len(codes)
    reason[7] ^= 1
    thr[valid[3]] = np.nextafter(thr[valid[3]], 0)
    bad = batch_parity(desc, sizes, seed, base, reason, thr, 8, threads=2)
    assert bad["reason_mismatches"] == 1 and bad["raw_mismatches"] == 1


def test_merge_and_rescore():
    wl, _, _ = load_eval("moe_1p6t_2048")
    desc, sizes = wl.desc(), wl.space.head_sizes
    a = [(5.0, 10, 1), (4.0, 3, 2)]
    b = [(5.0, 2, 7), (5.0, 11, 1), (1.0, 4, 9)]  # code 1 again later: dropped
    assert merge_topk([a, b], 3) == [(5.0, 2, 7), (5.0, 10, 1), (4.0, 3, 2)]
    planes = uniform_planes(desc, 0, 0, 50_000)
    res = simulate_planes(desc, planes, fields=("throughput",))
    i = int(np.flatnonzero(res["reason"] == 0)[0])
    vec = tuple(int(x) for x in planes[:, i])
    raw = float(res["throughput"][i])
    assert vector_codes(planes[:, [i]], sizes)[0] >= 0
    assert rescore_elites(desc, 0, [Elite(vec, raw, raw, i)]) == 0
    assert rescore_elites(desc, 0, [Elite(vec, raw, np.nextafter(raw, 0), i)]) == 1
    assert rescore_elites(desc, 0, [Elite(vec, raw, raw, i + 1)]) == 1
