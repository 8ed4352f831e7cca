"""The reference-side binding (refbind.gpu_search_env) driven through the
reference's OWN SearchEnv, installed in baseline/_ref:

* the seam contract of the reference's acceptance test
  (pkg/tests/test_acceptance.py:430-463: per-instance evaluate_raw stubs,
  reward shaping, exclusive best, penalty, budget) holds on the subclass;
* with the stock GPU seam, 2,000 steps produce the same rewards, raws and
  eval-log records as the reference's CPU env, and evaluate_raw returns the
  reference's SimResult field for field (detail text included);
* the reference's own random_walk / simulated_annealing drivers run on it.
Skipped when baseline/_ref is absent."""

import sys
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"
if not (REF / "shardsearch").exists():
    pytest.skip("reference package not installed in baseline/_ref", allow_module_level=True)
if str(REF) not in sys.path:
    sys.path.insert(0, str(REF))
import shardsearch  # noqa: E402
from shardsearch.config import load_config, packaged_config_path  # noqa: E402
from shardsearch.env import RewardConfig, SearchEnv  # noqa: E402
from shardsearch.simulator import InvalidReason, SimResult, TimeBreakdown  # noqa: E402

from paper_2509_00217_b200.refbind import gpu_search_env  # noqa: E402

GpuSearchEnv = gpu_search_env(shardsearch)


def _make(cls, cfg, budget):
    return cls(model=cfg.model, hw=cfg.hardware, space=cfg.space, context_len=cfg.simulation.context_len,
               budget=budget, slo_tpot=cfg.simulation.slo_tpot)


def test_reward_shaping_substitution_cases():
    """test_acceptance.py:430-463, verbatim in substance, on the GPU subclass."""
    cfg = load_config(packaged_config_path("tiny"))

    def stub(raw=None, reason=InvalidReason.NONE):
        valid = raw is not None
        return SimResult(valid=valid, invalid_reason=InvalidReason.NONE if valid else reason,
                         throughput=raw if valid else 0.0, tpot_s=0.001, memory_bytes=0.0,
                         breakdown=TimeBreakdown(0.001, 0.0, 0.0))

    action = (0,) * cfg.space.vector_length
    env = _make(GpuSearchEnv, cfg, 3)
    assert isinstance(env, SearchEnv)
    env.reward_cfg = RewardConfig(alpha=1.0, beta=1.0, invalid_penalty=-10.0)
    env.best_raw = 8.0
    env.evaluate_raw = lambda strategy: stub(raw=10.0)
    assert env.step(action) == (12.0, 10.0, True)
    assert env.best_raw == 10.0
    env.best_raw = 8.0
    env.evaluate_raw = lambda strategy: stub(raw=5.0)
    assert env.step(action) == (2.0, 5.0, True)
    assert env.best_raw == 8.0
    env.evaluate_raw = lambda strategy: stub(reason=InvalidReason.OOM)
    assert env.step(action) == (-10.0, 0.0, False)
    assert env.best_raw == 8.0 and env.evals_used == 3 and env.eval_log[-1].reason == "oom"


@pytest.mark.parametrize("name", ["tiny", "moe_1p2t_h100"])
def test_gpu_seam_equals_reference_env(name):
    cfg = load_config(packaged_config_path(name))
    n = 2000
    ref, gpu = _make(SearchEnv, cfg, n), _make(GpuSearchEnv, cfg, n)
    rng = np.random.default_rng(17)
    for _ in range(n):
        v = tuple(int(rng.integers(k)) for k in cfg.space.head_sizes)
        assert gpu.step(v) == ref.step(v)
    assert gpu.eval_log == ref.eval_log and gpu.best_raw == ref.best_raw
    for rec in ref.eval_log[:300]:
        s = shardsearch.strategy.decode_strategy(rec.vector, cfg.space)
        assert gpu.evaluate_raw(s) == ref.evaluate_raw(s)


def test_reference_drivers_on_the_gpu_env():
    from shardsearch.baselines import SaConfig, random_walk, simulated_annealing

    cfg = load_config(packaged_config_path("moe_1p2t_h100"))
    for algo in ("rw", "sa"):
        ref, gpu = _make(SearchEnv, cfg, 1500), _make(GpuSearchEnv, cfg, 1500)
        run = (lambda e: random_walk(e, 1500, 4)) if algo == "rw" else (
            lambda e: simulated_annealing(e, SaConfig(), 1500, 4))
        r1, r2 = run(ref), run(gpu)
        assert gpu.eval_log == ref.eval_log
        assert (r1.best_vector, r1.best_raw) == (r2.best_vector, r2.best_raw)
