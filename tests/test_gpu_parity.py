"""GPU parity: the CUDA evaluator (through libls_eval.so's C ABI) against the
reference's own golden verdicts and the CPU oracle — bit for bit.

Reference path: decode_strategy + simulate (pkg/src/shardsearch/strategy.py:
245-263, simulator.py:239-341). Bar: identical reason codes and identical
float64 bit patterns for every field (integer/byte work is exact; the fp64
formulas are reproduced with the reference's operation order, no FMA).
"""

import numpy as np
import pytest

from golden_io import FIELDS, eval_sets, load_eval, mismatches, search_sets, load_search

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ev_factory():
    from paper_2509_00217_b200.evaluator import Evaluator

    made = []

    def make(workload):
        e = Evaluator(workload, device=0)
        made.append(e)
        return e

    yield make
    for e in made:
        e.close()


def _dev(planes):
    return torch.from_numpy(np.ascontiguousarray(planes)).cuda()


@pytest.mark.parametrize("name", eval_sets())
def test_golden_bit_exact(name, ev_factory):
    wl, meta, data = load_eval(name)
    ev = ev_factory(wl)
    planes = _dev(data["vectors"].T)
    got = ev.evaluate(planes, fields="all").numpy()
    bad = mismatches(got, data)
    assert not bad.any(), f"{int(bad.sum())} mismatches, first at {np.nonzero(bad)[0][:5]}"


@pytest.mark.parametrize("name", ["moe_1p2t", "edge_odd", "llama3_8b_h100x8"])
def test_golden_generic_kernel_path(name, ev_factory):
    """Unaligned plane stride forces the one-candidate-per-thread kernel."""
    wl, meta, data = load_eval(name)
    ev = ev_factory(wl)
    A, n = data["vectors"].shape[1], data["vectors"].shape[0]
    buf = torch.zeros((A, n + 3), dtype=torch.uint8, device="cuda")
    buf[:, 1:n + 1] = _dev(data["vectors"].T)
    got = ev.evaluate(buf[:, 1:n + 1], fields="all").numpy()
    assert not mismatches(got, data).any()


@pytest.mark.parametrize("name", ["moe_1p6t_2048", "tiny", "unit_small_naive_sum"])
def test_host_pipeline_matches(name, ev_factory):
    wl, meta, data = load_eval(name)
    ev = ev_factory(wl)
    got = ev.evaluate_host(np.ascontiguousarray(data["vectors"].T), fields="all")
    assert not mismatches(got, data).any()


@pytest.mark.parametrize("name", ["moe_1p2t", "dsv3_style_h100x256", "edge_odd"])
def test_random_large_vs_oracle(name, ev_factory):
    """Fresh seeded candidates far beyond the fixtures, checked against the C oracle."""
    from oracle.cost_model import simulate_planes

    wl, meta, data = load_eval(name)
    ev = ev_factory(wl)
    rng = np.random.default_rng(123)
    n = 400_003  # ragged: not a multiple of 4
    sizes = ev.head_sizes
    planes = np.stack([rng.integers(0, k, size=n, dtype=np.uint8) for k in sizes])
    # bias half the axis heads to admissible values so the fp64 path is exercised
    planes[4:, : n // 2] = rng.integers(0, 3, size=(len(sizes) - 4, n // 2)) * (rng.random((len(sizes) - 4, n // 2)) < 0.5)
    want = simulate_planes(wl.desc(), planes)
    got = ev.evaluate(_dev(planes), fields="all").numpy()
    bad = mismatches(got, want)
    assert not bad.any(), f"{int(bad.sum())} mismatches"
    assert (want["reason"] == 0).sum() > 1000


def test_decode_errors_flagged(ev_factory):
    wl, meta, data = load_eval("moe_1p2t")
    ev = ev_factory(wl)
    planes = np.ascontiguousarray(data["vectors"][:64].T).copy()
    planes[0, 3] = 7      # tp domain has 7 entries: index 7 out of range
    planes[3, 10] = 11    # batch domain has 11
    planes[9, 20] = 3     # axis heads take 0..2
    got = ev.evaluate(_dev(planes), fields="all").numpy()
    assert got["reason"][3] == 255 and got["reason"][10] == 255 and got["reason"][20] == 255
    ok = np.ones(64, bool)
    ok[[3, 10, 20]] = False
    assert not mismatches({k: v[ok] for k, v in got.items()}, {k: data[k][:64][ok] for k in ["reason", *FIELDS]}).any()
    for i in (3, 10, 20):
        assert all(got[f][i] == 0.0 for f in FIELDS)


def test_empty_and_tiny_batches(ev_factory):
    wl, meta, data = load_eval("tiny")
    ev = ev_factory(wl)
    empty = torch.zeros((wl.space.vector_length, 0), dtype=torch.uint8, device="cuda")
    assert ev.evaluate(empty).reason.numel() == 0
    for n in (1, 2, 3, 5, 7):
        got = ev.evaluate(_dev(data["vectors"][:n].T), fields="all").numpy()
        assert not mismatches(got, {k: data[k][:n] for k in ["reason", *FIELDS]}).any()


def test_raw_only_output_matches_full(ev_factory):
    wl, meta, data = load_eval("moe_1p6t")
    ev = ev_factory(wl)
    planes = _dev(data["vectors"].T)
    raw = ev.evaluate(planes).numpy()
    assert set(raw) == {"reason", "throughput"}
    assert np.array_equal(raw["reason"], data["reason"])
    assert np.array_equal(raw["throughput"].view(np.uint64), data["throughput"].view(np.uint64))


@pytest.mark.parametrize("name", search_sets())
def test_reward_scan_matches_sequential_env(name, ev_factory):
    """Batched exclusive-prefix-max rewards == reference SearchEnv.step sequence."""
    wl, meta, data = load_search(name)
    ev = ev_factory(wl)
    planes = _dev(data["vectors"].T)
    res = ev.evaluate(planes)
    r = meta["reward"]
    reward, best = ev.reward_scan(res.reason, res.throughput, meta["b0"], r["alpha"], r["beta"], r["invalid_penalty"])
    assert np.array_equal(reward.cpu().numpy().view(np.uint64), data["rewards"].view(np.uint64))
    assert best.item() == meta["best_raw_final"]
    assert np.array_equal(res.reason.cpu().numpy() == 0, data["valid"])


@pytest.mark.parametrize("name", search_sets())
@pytest.mark.parametrize("cap", [1, 3, 8, 32])
def test_topk_matches_elite_buffer(name, cap, ev_factory):
    """Device top-k by reward == reference EliteBuffer after sequential offers."""
    wl, meta, data = load_search(name)
    ev = ev_factory(wl)
    planes = _dev(data["vectors"].T)
    res = ev.evaluate(planes)
    r = meta["reward"]
    reward, _ = ev.reward_scan(res.reason, res.throughput, meta["b0"], r["alpha"], r["beta"], r["invalid_penalty"])
    elites = ev.topk(planes, res.reason, res.throughput, key=reward, k=cap)
    want_v = [tuple(int(x) for x in v) for v in data[f"elite{cap}_vectors"]]
    want_r = list(data[f"elite{cap}_rewards"])
    assert [e.vector for e in elites] == want_v
    assert [e.key for e in elites] == want_r


def test_topk_by_raw_matches_report_winner(ev_factory):
    from oracle.search_semantics import best_by_raw

    wl, meta, data = load_eval("moe_1p2t")
    ev = ev_factory(wl)
    planes = _dev(data["vectors"].T)
    res = ev.evaluate(planes)
    best = ev.topk(planes, res.reason, res.throughput, k=1)[0]
    i = best_by_raw(data["reason"], data["throughput"])
    assert best.index == i and best.raw == data["throughput"][i]
    assert best.vector == tuple(int(x) for x in data["vectors"][i])


def test_topk_many_duplicates_and_merge(ev_factory):
    """A stream made of few distinct vectors repeated many times, split in
    shards and merged like the cross-GPU path."""
    from oracle.search_semantics import elite_offers

    wl, meta, data = load_eval("moe_1p2t")
    ev = ev_factory(wl)
    rng = np.random.default_rng(5)
    valid_rows = np.nonzero(data["reason"] == 0)[0][:40]
    pick = valid_rows[rng.integers(0, len(valid_rows), size=200_000)]
    vecs = data["vectors"][pick]
    planes = _dev(np.ascontiguousarray(vecs.T))
    res = ev.evaluate(planes)
    thr = res.throughput.cpu().numpy()
    want = elite_offers(vecs, thr, np.ones(len(vecs), bool), 16)
    got = ev.topk(planes, res.reason, res.throughput, k=16)
    assert [e.vector for e in got] == [w[0] for w in want]
    assert [e.index for e in got] == [w[2] for w in want]
    # shard into 4 pieces, top-k each, merge
    shards = np.array_split(np.arange(len(vecs)), 4)
    recs, counts = [], []
    for s in shards:
        lo, hi = int(s[0]), int(s[-1]) + 1
        r, c = ev.topk_records(planes[:, lo:hi], res.reason[lo:hi], res.throughput[lo:hi], k=16, index_base=lo)
        recs.append(r)
        counts.append(c)
    mrec, mcount = ev.merge_records(torch.cat(recs), torch.cat(counts), 16, 16)
    merged = ev.decode_records(mrec, mcount)
    assert [(e.vector, e.index, e.raw) for e in merged] == [(e.vector, e.index, e.raw) for e in got]


@pytest.mark.parametrize("name", ["moe_1p2t", "moe_1p6t_2048", "dsv3_style_h100x256", "tiny", "unit_small"])
@pytest.mark.parametrize("k", [1, 3, 8, 32])
def test_fused_evaluate_topk_matches_sequential_by_raw(name, k, ev_factory):
    """Fused sweep (evaluate + elite in one kernel) == sequential offers of
    every valid candidate keyed by raw, with and without verdict output."""
    from oracle.cost_model import simulate_planes
    from oracle.search_semantics import elite_offers

    wl, meta, data = load_eval(name)
    ev = ev_factory(wl)
    rng = np.random.default_rng(k)
    base = data["vectors"]
    vecs = np.concatenate([base, base[rng.integers(0, len(base), size=30_000)]])  # repeats
    planes_np = np.ascontiguousarray(vecs.T.astype(np.uint8))
    want_res = simulate_planes(wl.desc(), planes_np)
    want = elite_offers(vecs, want_res["throughput"], want_res["reason"] == 0, k)
    planes = _dev(planes_np)
    out, recs, count = ev.evaluate_topk(planes, k=k, index_base=1000)
    got = ev.decode_records(recs, count)
    assert [e.vector for e in got] == [w[0] for w in want]
    assert [e.index for e in got] == [w[2] + 1000 for w in want]
    assert [e.raw for e in got] == [w[1] for w in want]
    assert not mismatches(out.numpy(), want_res).any()
    _, recs2, count2 = ev.evaluate_topk(planes, k=k, index_base=1000, verdicts=False)
    assert [e.index for e in ev.decode_records(recs2, count2)] == [e.index for e in got]
