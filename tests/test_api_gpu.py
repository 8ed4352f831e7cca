"""The reference's behavioural unit tests, re-run against the GPU-backed
drop-ins: simulate() (reference tests/test_simulator.py:157-328) and
SearchEnv (tests/test_env.py:88-253), plus SearchEnv.step_batch == n x step."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2509_00217_b200.env import BudgetExhausted, NoEvaluations, RewardConfig, SearchEnv, load_eval_log, replay_eval_log  # noqa: E402
from paper_2509_00217_b200.simulator import InvalidReason, SimRequest, simulate  # noqa: E402
from paper_2509_00217_b200.spec import HardwareSpec, ModelSpec  # noqa: E402
from paper_2509_00217_b200.strategy import (  # noqa: E402
    ActionSpaceSpec, AxisChoice, Strategy, canonical_fused_ops, encode_strategy, megatron_fine_dims)


def small_model(**kw):
    base = dict(name="unit", num_layers=4, hidden_dim=256, num_heads=8, head_dim=32, num_kv_heads=4, ffn_dim=128,
                num_experts=8, experts_per_token=2, has_shared_expert=True, vocab_size=4096, dtype_bytes=2)
    base.update(kw)
    return ModelSpec(**base)


def bare_hw(**kw):
    base = dict(name="bare", peak_flops=1e15, hbm_bandwidth=3e12, hbm_capacity=8e10, intra_node_bw=9e11,
                inter_node_bw=5e10, node_size=8, device_budget=24000, kernel_overhead=0.0, per_collective_latency=0.0)
    base.update(kw)
    return HardwareSpec(**base)


def make_strategy(model, tp=1, ep=1, pp=1, batch=8, overrides=None):
    ops = canonical_fused_ops(model)
    dims = dict(zip((op.name for op in ops), megatron_fine_dims(ops)))
    dims.update(overrides or {})
    return Strategy(tp, ep, pp, batch, tuple(op.name for op in ops), tuple(dims[op.name] for op in ops))


def req(model, hw, s, ctx=256, slo=0.050):
    return SimRequest(model=model, hw=hw, strategy=s, context_len=ctx, slo_tpot=slo)


class TestSimulate:
    def test_gate_order(self):
        m = small_model()
        r = simulate(req(m, bare_hw(device_budget=16, hbm_capacity=1.0), make_strategy(m, tp=8, ep=4)))
        assert r.invalid_reason is InvalidReason.OVER_DEVICE_BUDGET and not r.valid
        r = simulate(req(m, bare_hw(hbm_capacity=1.0), make_strategy(m, tp=16)))
        assert r.invalid_reason is InvalidReason.LAYOUT_ERROR and "not divisible" in r.detail
        r = simulate(req(m, bare_hw(), make_strategy(m, pp=8)))
        assert r.invalid_reason is InvalidReason.LAYOUT_ERROR and "num_layers" in r.detail
        r = simulate(req(m, bare_hw(hbm_capacity=1e5), make_strategy(m, batch=64), slo=1e-12))
        assert r.invalid_reason is InvalidReason.OOM and r.memory_bytes > 1e5
        r = simulate(req(m, bare_hw(), make_strategy(m), slo=1e-12))
        assert r.invalid_reason is InvalidReason.SLO_VIOLATION and r.tpot_s > 1e-12 and r.throughput == 0.0
        r = simulate(req(m, bare_hw(), make_strategy(m)))
        assert r.valid and r.invalid_reason is InvalidReason.NONE and r.throughput > 0.0
        with pytest.raises(ValueError, match="decode"):
            SimRequest(m, bare_hw(), make_strategy(m), context_len=256, phase="prefill")

    def test_hand_counted_memory(self):
        m = small_model(num_layers=2, hidden_dim=32, num_heads=4, head_dim=8, num_kv_heads=4, ffn_dim=16,
                        num_experts=2, experts_per_token=1, has_shared_expert=False, vocab_size=64)
        s = make_strategy(m, batch=2)
        s = s.replace_dims(tuple(AxisChoice.UNSHARDED for _ in s.op_dims))
        r = simulate(req(m, bare_hw(), s, ctx=16, slo=10.0))
        assert r.memory_bytes == 42176.0
        r2 = simulate(req(m, bare_hw(), s, ctx=32, slo=10.0))
        assert r2.memory_bytes - r.memory_bytes == 8192.0

    def test_accounting(self):
        m, hw = small_model(), bare_hw(kernel_overhead=1e-7, per_collective_latency=1e-6)
        for tp, ep, pp in [(1, 1, 1), (4, 1, 1), (2, 2, 2), (1, 8, 4)]:
            r = simulate(req(m, hw, make_strategy(m, tp=tp, ep=ep, pp=pp), slo=10.0))
            b = r.breakdown
            assert r.tpot_s == b.compute_s + b.comm_s + b.pipeline_s
        r1 = simulate(req(m, hw, make_strategy(m, pp=1), slo=10.0))
        r4 = simulate(req(m, hw, make_strategy(m, pp=4), slo=10.0))
        assert r1.breakdown.pipeline_s == 0.0
        assert r4.breakdown.pipeline_s == pytest.approx(3 * (8 * 256 * 2 / hw.intra_node_bw + 1e-6), rel=1e-12)
        first = simulate(req(m, hw, make_strategy(m, tp=4, ep=2, pp=2, batch=16), slo=10.0))
        assert first == simulate(req(m, hw, make_strategy(m, tp=4, ep=2, pp=2, batch=16), slo=10.0))

    def test_fine_dims_change_only_comm(self):
        m, hw = small_model(), bare_hw()
        meg = make_strategy(m, tp=4, batch=8)
        alt = make_strategy(m, tp=4, batch=8, overrides={"expert_ffn2": AxisChoice.DIM1, "shared_ffn2": AxisChoice.DIM1})
        rm, ra = simulate(req(m, hw, meg, slo=10.0)), simulate(req(m, hw, alt, slo=10.0))
        assert rm.breakdown.compute_s == ra.breakdown.compute_s
        assert rm.breakdown.comm_s - ra.breakdown.comm_s == pytest.approx(4 * (6144 - 7680) / hw.intra_node_bw,
                                                                          rel=1e-12)


def small_space():
    return ActionSpaceSpec(tp_domain=(1, 2, 4), ep_domain=(1, 2, 4), pp_domain=(1, 2, 4), batch_domain=(1, 4, 16))


def make_env(budget=16, log_path=None, hw=None, reward=RewardConfig()):
    return SearchEnv(small_model(), hw or bare_hw(device_budget=64), small_space(), 256, budget, reward=reward,
                     log_path=log_path)


def meg_vec(space, tp=1, ep=1, pp=1, batch=1):
    m = small_model()
    ops = canonical_fused_ops(m)
    return encode_strategy(Strategy(tp, ep, pp, batch, tuple(op.name for op in ops), megatron_fine_dims(ops)), space)


class TestEnv:
    def test_rewards_and_best(self):
        env = make_env()
        reward, raw, valid = env.step(meg_vec(env.space, tp=2, batch=4))
        assert valid and raw > 0 and reward == pytest.approx(2.0 * raw) and env.best_raw == raw
        env = make_env()
        r_good, raw_good, _ = env.step(meg_vec(env.space, tp=2, batch=16))
        r_ok, raw_ok, _ = env.step(meg_vec(env.space, tp=2, batch=4))
        assert raw_ok < raw_good and r_ok == pytest.approx(raw_ok + (raw_ok - raw_good))
        assert env.best_raw == raw_good

    def test_invalid_budget_and_selection(self):
        env = make_env(hw=bare_hw(device_budget=64, hbm_capacity=1e4))
        reward, raw, valid = env.step(meg_vec(env.space))
        assert (reward, raw, valid) == (env.reward_cfg.invalid_penalty, 0.0, False)
        assert env.eval_log[0].reason == "oom"
        env = make_env(budget=2)
        env.step(meg_vec(env.space, tp=2, batch=4))
        env.step(meg_vec(env.space, tp=2, batch=4))
        with pytest.raises(BudgetExhausted):
            env.step(meg_vec(env.space, tp=2, batch=4))
        with pytest.raises(NoEvaluations):
            make_env().final_selection()
        env = make_env()
        env.step(meg_vec(env.space, tp=2, batch=4))
        env.step(meg_vec(env.space, tp=2, batch=4))
        _, rec = env.final_selection()
        assert rec.index == 0

    def test_log_and_replay_bit_for_bit(self, tmp_path):
        log = tmp_path / "evals.ndjson"
        env = make_env(budget=8, log_path=log)
        for tp, batch in [(1, 4), (2, 16), (4, 16), (2, 1)]:
            env.step(meg_vec(env.space, tp=tp, batch=batch))
        env.close()
        records = load_eval_log(log)
        assert records == env.eval_log
        for record, recomputed in replay_eval_log(records, small_model(), bare_hw(device_budget=64), env.space, 256):
            assert recomputed == record.raw

    def test_step_batch_equals_sequential_steps(self):
        rng = np.random.default_rng(3)
        space = small_space()
        vecs = np.stack([rng.integers(0, k, size=3000) for k in space.head_sizes], axis=1)
        vecs = np.concatenate([vecs, vecs[:500]])  # repeats
        cfg = RewardConfig(alpha=0.5, beta=2.0, invalid_penalty=-3.0)
        seq = make_env(budget=4000, reward=cfg)
        seq.best_raw = 1.5
        for v in vecs[:400]:
            seq.step(v)
        bat = make_env(budget=4000, reward=cfg)
        bat.best_raw = 1.5
        bat.step_batch(vecs[:150])
        bat.step_batch(vecs[150:400])
        assert bat.eval_log == seq.eval_log
        assert bat.best_raw == seq.best_raw and bat.evals_used == 400
        with pytest.raises(BudgetExhausted):
            bat.step_batch(np.concatenate([vecs, vecs])[:3601])  # 3600 evaluations left
