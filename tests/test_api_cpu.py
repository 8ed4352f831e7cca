"""Host-side API parity with the reference (no GPU): spec validation
(reference tests/test_strategy.py:41-66), the strategy codec
(test_strategy.py:89-152), strict YAML configs (test_config.py) and the
workload descriptor the evaluator consumes."""

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2509_00217_b200.config import ConfigError, load_workload, packaged_configs, parse_config
from paper_2509_00217_b200.spec import HardwareSpec, ModelSpec, count_parameters
from paper_2509_00217_b200.strategy import (
    ActionSpaceSpec,
    AxisChoice,
    DecodingError,
    EncodingError,
    Strategy,
    canonical_fused_ops,
    codes_to_vectors,
    decode_strategy,
    encode_strategy,
    megatron_fine_dims,
    vector_codes,
)
from paper_2509_00217_b200.workload import build_desc


def small_model(**kw):
    base = dict(name="unit", num_layers=4, hidden_dim=256, num_heads=8, head_dim=32, num_kv_heads=4, ffn_dim=128,
                num_experts=8, experts_per_token=2, has_shared_expert=True, vocab_size=4096, dtype_bytes=2)
    base.update(kw)
    return ModelSpec(**base)


class TestSpecs:
    def test_validation_messages(self):
        with pytest.raises(ValueError, match="hidden_dim"):
            small_model(head_dim=16)
        with pytest.raises(ValueError, match="num_kv_heads"):
            small_model(num_kv_heads=3)
        with pytest.raises(ValueError, match="experts_per_token"):
            small_model(experts_per_token=9)
        with pytest.raises(ValueError, match="peak_flops"):
            HardwareSpec("h", 0.0, 1.0, 1.0, 1.0, 1.0, 8, 8, 0.0, 0.0)

    def test_parameter_count_hand_total(self):
        c = count_parameters(small_model())
        assert c.embedding == c.lm_head == 4096 * 256
        assert c.attention == 4 * (131072 + 65536)
        assert c.router == 4 * 2048
        assert c.routed_experts == 4 * 524288
        assert c.shared_expert == 4 * 65536
        assert c.norms == 4 * 1024 + 256
        assert c.total == c.dense + c.routed_experts

    def test_canonical_ops(self):
        assert len(canonical_fused_ops(small_model())) == 12
        assert len(canonical_fused_ops(small_model(has_shared_expert=False))) == 10
        ops = canonical_fused_ops(small_model())
        for op, axis in zip(ops, megatron_fine_dims(ops)):
            assert op.admits(axis)


class TestCodec:
    def test_space_size_and_fixed_vector(self):
        space = ActionSpaceSpec()
        assert space.size == 2_005_126_893 and space.vector_length == 16
        vec = (3, 1, 0, 5, 0, 2, 0, 2, 1, 0, 2, 1, 2, 1, 0, 2)
        s = decode_strategy(vec, space)
        assert (s.tp, s.ep, s.pp, s.batch) == (8, 2, 1, 32)
        assert encode_strategy(s, space) == vec

    def test_errors(self):
        space = ActionSpaceSpec()
        with pytest.raises(DecodingError, match="position 0"):
            decode_strategy((7,) + (0,) * 15, space)
        with pytest.raises(DecodingError, match="length"):
            decode_strategy((0,) * 15, space)
        s = decode_strategy((0,) * 16, space)
        with pytest.raises(EncodingError, match="tp=3"):
            encode_strategy(Strategy(3, s.ep, s.pp, s.batch, s.op_names, s.op_dims), space)
        with pytest.raises(ValueError, match="unique"):
            ActionSpaceSpec(tp_domain=(1, 2, 2))
        with pytest.raises(ValueError, match="pinned"):
            ActionSpaceSpec(pinned=(("qkv_proj", AxisChoice.DIM1),))

    def test_pins(self):
        space = ActionSpaceSpec(op_names=("qkv_proj", "attn_out_proj"), pinned=(("expert_ffn1", AxisChoice.DIM1),))
        s = decode_strategy((0, 0, 0, 0, 2, 1), space)
        assert s.axis_of("qkv_proj") is AxisChoice.DIM1
        assert s.axis_of("attn_out_proj") is AxisChoice.DIM0
        assert s.axis_of("expert_ffn1") is AxisChoice.DIM1
        assert s.axis_of("final_norm") is AxisChoice.UNSHARDED

    @given(st.data())
    @settings(max_examples=300, deadline=None)
    def test_round_trip_and_codes(self, data):
        space = ActionSpaceSpec()
        vec = tuple(data.draw(st.integers(0, k - 1)) for k in space.head_sizes)
        assert encode_strategy(decode_strategy(vec, space), space) == vec
        code = vector_codes([vec], space)
        assert tuple(codes_to_vectors(code, space)[0]) == vec


class TestConfig:
    def test_packaged_configs_load(self):
        names = packaged_configs()
        for required in ("tiny", "moe_1p2t_h100", "moe_1p6t_h100", "moe_1p6t_h100x2048", "llama3_8b_h100x8",
                         "llama3_70b_h100x64", "dsv3_style_h100x256"):
            assert required in names
        for name in names:
            wl = load_workload(name)
            build_desc(wl.model, wl.hw, wl.space, wl.context_len, wl.slo_tpot)

    def test_strict_keys_and_float_strings(self):
        doc = {
            "model": dict(name="m", num_layers=2, hidden_dim=32, num_heads=4, head_dim=8, num_kv_heads=4,
                          ffn_dim=16, num_experts=2, experts_per_token=1, has_shared_expert=False, vocab_size=64),
            "hardware": dict(name="h", peak_flops="989e12", hbm_bandwidth=3.35e12, hbm_capacity=8e10,
                             intra_node_bw=4.5e11, inter_node_bw=5e10, node_size=8, device_budget=64,
                             kernel_overhead=2e-6, per_collective_latency=1e-6),
            "simulation": {"context_len": 128},
        }
        cfg = parse_config(doc)
        assert cfg.hardware.peak_flops == 989e12
        bad = dict(doc, model=dict(doc["model"], hiden_dim=3))
        with pytest.raises(ConfigError, match="model.hiden_dim"):
            parse_config(bad)
        with pytest.raises(ConfigError, match="missing section 'simulation'"):
            parse_config({k: v for k, v in doc.items() if k != "simulation"})
        with pytest.raises(ConfigError, match="unknown operator"):
            parse_config(dict(doc, action_space={"ops": ["shared_ffn1"]}))


class TestDescriptor:
    def test_op_heads_and_pins(self):
        wl = load_workload("tiny")
        d = build_desc(wl.model, wl.hw, wl.space, wl.context_len, wl.slo_tpot)
        assert d.vector_length == 8
        assert [d.op_head[k] for k in range(12)] == [4, 5, -1, -1, -1, -1, 6, 7, -1, -1, -1, -1]
        assert list(d.domain_len) == [3, 3, 3, 3]

    def test_exactness_guard(self):
        huge = ModelSpec("huge", 2000, 65536, 512, 128, 8, 1 << 20, 1024, 8, True, 1 << 20, 8)
        hw = HardwareSpec("h", 1e15, 1e12, 1e11, 1e11, 1e10, 8, 1 << 20, 0.0, 0.0)
        with pytest.raises(ValueError, match="2\\^53"):
            build_desc(huge, hw, ActionSpaceSpec(), 1024, 0.05)
