"""On-device candidate streams (ls_generate / ls_sweep) against the host twin
(generator.py) and the CPU oracle: generated vectors bit-identical, and the
fused sweep's elite equal to evaluating the materialised stream and offering
every valid candidate in order (by raw, earliest index on ties)."""

import itertools

import numpy as np
import pytest

from golden_io import load_eval

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def make_ev():
    from paper_2509_00217_b200.evaluator import Evaluator

    made = []

    def make(wl):
        ev = Evaluator(wl, device=0)
        made.append(ev)
        return ev

    yield make
    for ev in made:
        ev.close()


@pytest.mark.parametrize("name", ["tiny", "moe_1p2t", "llama3_8b_h100x8", "edge_odd"])
@pytest.mark.parametrize("mode", [1, 2, 3])
def test_generate_matches_host_twin(name, mode, make_ev):
    from paper_2509_00217_b200.generator import stream_size, stream_vectors

    wl, _, _ = load_eval(name)
    ev = make_ev(wl)
    size = stream_size(wl.model, wl.space, mode)
    if mode != 1:
        assert ev.stream_size(mode) == size
    n = min(300_001, size)
    start = 0 if mode == 1 else max(0, size - n - 17)
    got = ev.generate(mode, n, start=start, seed=99).cpu().numpy().T
    want = stream_vectors(wl.model, wl.space, mode, start, n, seed=99)
    assert np.array_equal(got, want)


def _elite_by_raw(wl, vectors, k, base=0):
    from oracle.cost_model import simulate_planes
    from oracle.search_semantics import elite_offers

    res = simulate_planes(wl.desc(), np.ascontiguousarray(vectors.T.astype(np.uint8)))
    el = elite_offers(vectors, list(res["throughput"]), res["reason"] == 0, k)
    return [(v, r, i + base) for v, r, i in el]


@pytest.mark.parametrize("name,mode,n,start", [
    ("moe_1p2t", 1, 2_000_003, 0),
    ("moe_1p6t_2048", 1, 1_000_000, 5_000_000),
    ("dsv3_style_h100x256", 3, 1_500_000, 7_777),
    ("edge_odd", 2, 364_500, 0),  # the whole space: 5*5*4*5 coarse x 3^6 axes
])
@pytest.mark.parametrize("k", [1, 8, 32])  # k = 32 over a full grid: the windowed last-CTA merge
def test_sweep_matches_sequential_elite(name, mode, n, start, k, make_ev):
    from paper_2509_00217_b200.generator import stream_vectors

    wl, _, _ = load_eval(name)
    ev = make_ev(wl)
    recs, count = ev.sweep(mode, n, start=start, seed=5, k=k)
    got = [(e.vector, e.raw, e.index) for e in ev.decode_records(recs, count)]
    vecs = stream_vectors(wl.model, wl.space, mode, start, n, seed=5)
    want = _elite_by_raw(wl, vecs, k, base=start)
    assert got == [(tuple(int(x) for x in v), r, i) for v, r, i in want]


def test_tiny_exhaustive_optimum(make_ev):
    """The tiny space's optimum 10322.359866532712 is a 3-way tie
    (1,0,2,2,{0,1,2},2,2,2) (reference test_acceptance.py:58):
    the sweep returns all three, earliest first."""
    wl, _, _ = load_eval("tiny")
    ev = make_ev(wl)
    recs, count = ev.sweep(2, 6561, k=3)
    el = ev.decode_records(recs, count)
    assert [e.vector for e in el] == [(1, 0, 2, 2, a, 2, 2, 2) for a in (0, 1, 2)]
    assert all(e.raw == 10322.359866532712 for e in el)


def test_llama8b_exhaustive_equals_oracle(make_ev):
    """BASELINE config 1: all 10,392,624 strategies of Llama-3-8B on one H100
    node, exhaustively; the device winner equals the CPU oracle's."""
    from oracle.cost_model import simulate_planes
    from paper_2509_00217_b200.generator import stream_vectors

    wl, _, _ = load_eval("llama3_8b_h100x8")
    ev = make_ev(wl)
    n = ev.stream_size(2)
    assert n == 10_392_624
    recs, count = ev.sweep(2, n, k=4)
    got = ev.decode_records(recs, count)
    planes = ev.generate(2, n).cpu().numpy()
    res = simulate_planes(wl.desc(), planes, threads=None)
    thr = np.where(res["reason"] == 0, res["throughput"], -1.0)
    best = int(np.argmax(thr))
    assert got[0].index == best and got[0].raw == res["throughput"][best]
    assert got[0].vector == tuple(int(x) for x in planes[:, best])


def test_stream_size_errors_and_empty_sweep():
    """a stream the library cannot enumerate raises instead of reporting
    0, and an empty sweep returns an empty elite."""
    from paper_2509_00217_b200._native import NativeError
    from paper_2509_00217_b200.baselines import random_sweep
    from paper_2509_00217_b200.evaluator import Evaluator
    from paper_2509_00217_b200.generator import GEN_UNIFORM

    wl, _, _ = load_eval("tiny")
    ev = Evaluator(wl, device=0)
    with pytest.raises(NativeError):
        ev.stream_size(GEN_UNIFORM)  # unbounded: no size
    rep = random_sweep(ev, 0)
    assert rep.evaluated == 0 and rep.elites == () and rep.best is None
