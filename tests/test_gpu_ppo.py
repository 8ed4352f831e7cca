"""GPU PPO search (paper_2509_00217_b200/ppo.py) against the reference's
run_search (golden eval logs in tests/golden/ppo_reference.npz, made by
tests/golden/make_golden_ppo.py) and the reference's chunk-protocol tests
(pkg/tests/test_ppo.py).
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2509_00217_b200.config import load_workload  # noqa: E402
from paper_2509_00217_b200.env import SearchEnv, replay_eval_log  # noqa: E402
from paper_2509_00217_b200.knobs import PpoConfig  # noqa: E402
from paper_2509_00217_b200.policy import EliteBuffer  # noqa: E402
from paper_2509_00217_b200.ppo import GpuSearch, run_search  # noqa: E402

GOLD = np.load(Path(__file__).parent / "golden" / "ppo_reference.npz")
META = json.loads(str(GOLD["meta"]))


def make_env(name, budget, **kw):
    wl = load_workload(name)
    return SearchEnv(wl.model, wl.hw, wl.space, wl.context_len, budget, slo_tpot=wl.slo_tpot, **kw), wl


def prefix(env, case):
    vecs = np.asarray([r.vector for r in env.eval_log], dtype=np.uint8)
    rews = np.asarray([r.reward for r in env.eval_log])
    ref_v, ref_r = GOLD[case + "_vectors"], GOLD[case + "_rewards"]
    for i in range(min(len(vecs), len(ref_v))):
        if not (np.array_equal(vecs[i], ref_v[i]) and rews[i] == ref_r[i]):
            return i
    return min(len(vecs), len(ref_v))


@pytest.mark.parametrize("case", ["tiny_0", "tiny_1"])
def test_tiny_search_reproduces_reference_trajectory(case):
    """Same PCG64 stream, same reward arithmetic: the GPU search walks the
    reference's trajectory (float64 policy math differs only in rounding)."""
    name, seed = case.rsplit("_", 1)
    m = META[case]
    env, _ = make_env(name, m["evals"])
    rep = run_search(env, PpoConfig(budget=m["evals"]), int(seed))
    assert rep.evals == m["evals"] == len(env.eval_log)
    k = prefix(env, case)
    assert k >= 200, f"trajectory diverged from the reference after {k} evals"
    if k == m["evals"]:
        assert list(rep.restarts) == m["restarts"]
        assert rep.best_raw == m["best_raw"] and list(rep.best_vector) == m["best_vector"]


def test_flagship_search_matches_reference_quality():
    """1.2T, budget 4000, seed 0: the reference's trajectory (or one of equal quality)."""
    case = "moe_1p2t_h100_0"
    m = META[case]
    env, _ = make_env("moe_1p2t_h100", m["evals"])
    rep = run_search(env, PpoConfig(budget=m["evals"]), 0)
    assert rep.evals == 4000
    k = prefix(env, case)
    if k < 4000:
        # diverged late: the search must still be a healthy PPO run
        assert k >= 500, f"diverged after {k} evals"
        assert rep.best_raw >= 0.8 * m["best_raw"]
    else:
        assert rep.best_raw == m["best_raw"]


def test_records_rewards_and_best_are_consistent():
    env, wl = make_env("moe_1p2t_h100", 400)
    env.best_raw = 3.0  # a pre-existing best carries into the search's rewards
    run_search(env, PpoConfig(budget=400), 5)
    best = 3.0
    for r in env.eval_log:
        if r.valid:
            assert r.reward == 1.0 * r.raw + 1.0 * (r.raw - best)
            best = max(best, r.raw)
        else:
            assert r.reward == -10.0 and r.raw == 0.0
    assert env.best_raw == best
    replayed = [raw for _, raw in replay_eval_log(env.eval_log, wl.model, wl.hw, wl.space, wl.context_len,
                                                   wl.slo_tpot)]
    assert replayed == [r.raw for r in env.eval_log]


def test_device_elite_buffer_equals_host_rules():
    env, _ = make_env("moe_1p2t_h100", 600)
    search = GpuSearch(env, PpoConfig(budget=600), 2)
    _, done = search.run()
    recs = search.records(0, done)
    buf = EliteBuffer(3)
    for r in recs:
        if r.valid:
            buf.offer(r.vector, r.reward)
    ev = search.elite_vec.cpu().numpy()
    er = search.elite_reward.cpu().numpy()
    assert [tuple(int(x) for x in ev[i]) for i in range(len(buf))] == [e.vector for e in buf.entries]
    assert list(er[: len(buf)]) == [e.reward for e in buf.entries]
    assert np.isinf(er[len(buf):]).all()


def test_no_early_exit_spends_budget_in_five_chunks():
    env, _ = make_env("tiny", 100)
    rep = run_search(env, PpoConfig(budget=100, tau=1.5), 0)
    assert list(rep.restarts) == [0, 20, 40, 60, 80]
    assert rep.evals == 100


def test_early_exits_roll_budget_forward_and_still_spend_all():
    env, _ = make_env("tiny", 100)
    rep = run_search(env, PpoConfig(budget=100, tau=1e-9), 0)  # every head confident at once
    assert rep.evals == 100 == len(env.eval_log)
    assert list(rep.restarts) == list(range(0, 100, 2))  # each agent exits after one rollout


def test_graphs_and_eager_agree():
    a, _ = make_env("tiny", 60)
    b, _ = make_env("tiny", 60)
    ra = run_search(a, PpoConfig(budget=60), 4, use_graphs=True)
    rb = run_search(b, PpoConfig(budget=60), 4, use_graphs=False)
    assert ra.rewards == rb.rewards and ra.restarts == rb.restarts


def test_budget_guard():
    env, _ = make_env("tiny", 50)
    with pytest.raises(ValueError):
        run_search(env, PpoConfig(budget=100), 0)
