"""Batched search baselines vs the reference's own runs
(tests/golden/baselines_reference.npz, made by make_golden_search.py):
random_walk and simulated_annealing consume the same numpy PCG64 stream, so
every record must match bit for bit; megatron_exhaustive picks the same
winner; the device-native exhaustive sweep finds the global optimum."""

import json
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden" / "baselines_reference.npz"


@pytest.fixture(scope="module")
def gold():
    z = np.load(GOLD)
    return json.loads(str(z["meta"])), {k: z[k] for k in z.files if k != "meta"}


def _env(name, budget):
    from paper_2509_00217_b200.config import load_config
    from paper_2509_00217_b200.env import SearchEnv

    cfg = load_config(f"paper_2509_00217_b200/configs/{name}.yaml")
    return cfg, SearchEnv(cfg.model, cfg.hardware, cfg.space, cfg.simulation.context_len, budget,
                          slo_tpot=cfg.simulation.slo_tpot)


@pytest.mark.parametrize("name,budget,seed", [("moe_1p2t_h100", 4000, 0), ("moe_1p2t_h100", 4000, 3),
                                              ("tiny", 1000, 0), ("tiny", 1000, 1)])
@pytest.mark.parametrize("algo", ["rw", "sa"])
def test_baseline_records_match_reference(name, budget, seed, algo, gold):
    from paper_2509_00217_b200.baselines import SaConfig, random_walk, simulated_annealing

    meta, data = gold
    key = f"{name}_{algo}_{seed}"
    cfg, env = _env(name, budget)
    rep = random_walk(env, budget, seed) if algo == "rw" else simulated_annealing(env, SaConfig(), budget, seed)
    assert np.array_equal(np.asarray([r.vector for r in env.eval_log]), data[key + "_vectors"])
    assert np.array_equal(np.asarray([r.reward for r in env.eval_log]).view(np.uint64),
                          data[key + "_rewards"].view(np.uint64))
    assert np.array_equal(np.asarray([r.raw for r in env.eval_log]).view(np.uint64), data[key + "_raws"].view(np.uint64))
    want = meta[key]
    assert list(rep.best_vector) == want["best_vector"]
    assert rep.best_raw == want["best_raw"] and rep.best_reward == want["best_reward"] and rep.evals == budget


@pytest.mark.parametrize("name", ["moe_1p2t_h100", "tiny"])
def test_megatron_exhaustive_matches_reference(name, gold):
    from paper_2509_00217_b200.baselines import megatron_exhaustive

    meta, _ = gold
    cfg, _ = _env(name, 1)
    rep = megatron_exhaustive(lambda b: _env(name, b)[1], cfg.space)
    want = meta[f"{name}_exhaustive"]
    assert list(rep.best_vector) == want["best_vector"] and rep.best_raw == want["best_raw"]
    assert rep.evals == want["evals"]


def test_device_exhaustive_finds_the_global_optimum():
    """The whole 2,005,126,893-point 1.2T space: the optimum is the Megatron
    layout at (tp 8, ep 4, pp 2, batch 64) — above the reference PPO's
    best-of-10 (47.99)."""
    from paper_2509_00217_b200.baselines import exhaustive_search
    from paper_2509_00217_b200.config import load_workload
    from paper_2509_00217_b200.evaluator import Evaluator

    ev = Evaluator(load_workload("moe_1p2t_h100"), device=0)
    rep = exhaustive_search(ev, k=4)
    assert rep.evaluated == 2_005_126_893
    assert rep.best.raw == 49.09885285712207
    assert rep.best.vector == (3, 2, 1, 6, 0, 2, 0, 2, 1, 0, 2, 1, 2, 1, 0, 2)
    adm = exhaustive_search(ev, admissible_only=True, k=4)
    assert adm.evaluated == 49_509_306 and adm.best.vector == rep.best.vector and adm.best.raw == rep.best.raw
    tiny = exhaustive_search(Evaluator(load_workload("tiny"), device=0), k=3)
    assert tiny.best.vector == (1, 0, 2, 2, 0, 2, 2, 2) and tiny.best.raw == 10322.359866532712
