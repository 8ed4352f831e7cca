"""The CPU oracle (oracle/shardsim_oracle.c) pinned against the reference.

Every golden fixture was produced by the reference's own decode_strategy +
simulate (tests/golden/make_golden.py); the oracle must reproduce every
reason code and every float64 bit pattern.
"""

import numpy as np
import pytest

from golden_io import FIELDS, eval_sets, load_eval, load_search, mismatches, search_sets
from oracle.cost_model import layer_plan, simulate_planes
from oracle.search_semantics import elite_offers, rewards_sequential


@pytest.mark.parametrize("name", eval_sets())
def test_oracle_reproduces_reference_bits(name):
    wl, meta, data = load_eval(name)
    got = simulate_planes(wl.desc(), data["vectors"].T)
    bad = mismatches(got, data)
    assert not bad.any(), f"{int(bad.sum())} mismatches, first rows {np.nonzero(bad)[0][:5]}"


@pytest.mark.parametrize("name", search_sets())
def test_sequential_semantics_reproduce_reference(name):
    wl, meta, data = load_search(name)
    res = simulate_planes(wl.desc(), data["vectors"].T)
    r = meta["reward"]
    rewards, best = rewards_sequential(res["reason"], res["throughput"], meta["b0"], r["alpha"], r["beta"],
                                       r["invalid_penalty"])
    assert np.array_equal(np.asarray(rewards).view(np.uint64), data["rewards"].view(np.uint64))
    assert best == meta["best_raw_final"]
    for cap in (1, 3, 8, 32):
        want = [tuple(int(x) for x in v) for v in data[f"elite{cap}_vectors"]]
        got = elite_offers(data["vectors"], rewards, res["reason"] == 0, cap)
        assert [g[0] for g in got] == want
        assert [g[1] for g in got] == list(data[f"elite{cap}_rewards"])


def test_layer_plan_megatron_two_all_reduces():
    """reference tests/test_layout.py:162-172 on the unit model: tp=4 megatron
    layer = exactly two all_reduce (kind 1)."""
    wl, meta, data = load_eval("unit_small")
    # tp=4 (idx 2), ep=1, pp=1, batch=8 (idx 3), megatron axes over 12 ops
    vec = [2, 0, 0, 3, 0, 2, 0, 2, 1, 0, 2, 1, 2, 1, 0, 2]
    plan = layer_plan(wl.desc(), vec)
    assert [c[0] for c in plan] == [1, 1]


def test_layer_plan_expert_parallel_a2a_payload():
    """reference tests/test_layout.py:196-206: tp=1, ep=4 -> dispatch + combine
    all_to_all of 8*2/4*256*2 = 2048 bytes over a group of 4."""
    wl, meta, data = load_eval("unit_small")
    vec = [0, 2, 0, 3, 0, 2, 0, 2, 1, 0, 2, 1, 2, 1, 0, 2]
    plan = layer_plan(wl.desc(), vec)
    a2a = [c for c in plan if c[0] == 4]
    assert len(a2a) == 2 and all(c[1] == 4 and c[2] == 2048.0 for c in a2a)


def test_layer_plan_mixed_branches_align():
    """reference tests/test_layout.py:235-245: shared_ffn2 DIM1 under tp=4 ->
    2 all_reduce + 2 all_gather."""
    wl, meta, data = load_eval("unit_small")
    vec = [2, 0, 0, 3, 0, 2, 0, 2, 1, 0, 2, 1, 2, 2, 0, 2]
    kinds = [c[0] for c in layer_plan(wl.desc(), vec)]
    assert kinds.count(1) == 2 and kinds.count(2) == 2
