"""Host layer planner (plan.py) against the reference's plan_layer /
LayerPlan.describe (golden text in tests/golden/plans_reference.json, made
by tests/golden/make_golden_plan.py from the reference itself), plus the
reference's plan-structure acceptance test (test_acceptance.py:179-230)."""

from __future__ import annotations

import json
from pathlib import Path

import pytest

from paper_2509_00217_b200.config import load_config, resolve_config_path
from paper_2509_00217_b200.plan import CollectiveKind, LayoutError, TensorLayout, plan_layer, transition
from paper_2509_00217_b200.strategy import AxisChoice, Strategy, canonical_fused_ops, decode_strategy, megatron_fine_dims

CASES = json.loads((Path(__file__).parent / "golden" / "plans_reference.json").read_text())


@pytest.fixture(scope="module")
def configs():
    return {name: load_config(resolve_config_path(name)) for name in {c["config"] for c in CASES}}


def test_every_reference_plan_description_and_error(configs):
    for case in CASES:
        cfg = configs[case["config"]]
        ops = canonical_fused_ops(cfg.model)
        segs = {"pre": tuple(op for op in ops if op.name == "embedding"),
                "layer": tuple(op for op in ops if op.per_layer),
                "post": tuple(op for op in ops if not op.per_layer and op.name != "embedding")}
        s = decode_strategy(tuple(case["vector"]), cfg.space)
        for seg, seg_ops in segs.items():
            try:
                got = plan_layer(cfg.model, seg_ops, s, s.batch, cfg.hardware.node_size).describe()
            except LayoutError as exc:
                got = "LayoutError: " + str(exc)
            assert got == case["plans"][seg], (case["config"], case["vector"], seg)


def test_transition_table():
    R, P = TensorLayout.replicated(4), TensorLayout.partial_sum(4)
    S0, S1 = TensorLayout.sharded(AxisChoice.DIM0, 4), TensorLayout.sharded(AxisChoice.DIM1, 4)
    kinds = {(a, b): transition(x, y, 1.0, "intra").kind for a, x in (("R", R), ("S0", S0), ("P", P))
             for b, y in (("R", R), ("S1", S1)) if not (a == "R" and b == "R")}
    assert kinds == {("R", "S1"): CollectiveKind.NO_OP, ("S0", "R"): CollectiveKind.ALL_GATHER,
                     ("S0", "S1"): CollectiveKind.ALL_TO_ALL, ("P", "R"): CollectiveKind.ALL_REDUCE,
                     ("P", "S1"): CollectiveKind.REDUCE_SCATTER}
    with pytest.raises(LayoutError):
        transition(R, P, 1.0, "intra")
    assert TensorLayout.sharded(AxisChoice.DIM1, 1) == TensorLayout.replicated(1)


def test_allgather_between_ffn_matmuls_replaces_the_mlp_allreduce():
    cfg = load_config(resolve_config_path("moe_1p2t_h100"))
    ops = canonical_fused_ops(cfg.model)
    names = tuple(op.name for op in ops)
    by_name = dict(zip(names, megatron_fine_dims(ops)))
    ffn_ops = {"expert_ffn1", "expert_ffn2", "shared_ffn1", "shared_ffn2"}

    def plan_with(dims):
        s = Strategy(tp=4, ep=1, pp=1, batch=64, op_names=names, op_dims=tuple(dims[n] for n in names))
        return plan_layer(cfg.model, ops, s, batch_tokens=64, node_size=cfg.hardware.node_size)

    def mlp_collectives(plan):
        kinds = [c.kind for st in plan.steps if st.op.name in ffn_ops for c in st.collectives_before]
        return kinds + [c.kind for c in plan.exit_collectives]

    alt = dict(by_name, expert_ffn2=AxisChoice.DIM1, shared_ffn2=AxisChoice.DIM1)
    alt_plan = plan_with(alt)
    ffn2 = next(s for s in alt_plan.steps if s.op.name == "expert_ffn2")
    assert any(c.kind is CollectiveKind.ALL_GATHER for c in ffn2.collectives_before)
    assert CollectiveKind.ALL_REDUCE not in mlp_collectives(alt_plan)
    mega = plan_with(dict(by_name))
    assert mlp_collectives(mega).count(CollectiveKind.ALL_REDUCE) == 1
    mega_ffn2 = next(s for s in mega.steps if s.op.name == "expert_ffn2")
    assert not any(c.kind in (CollectiveKind.ALL_GATHER, CollectiveKind.ALL_REDUCE, CollectiveKind.REDUCE_SCATTER)
                   for c in mega_ffn2.collectives_before)
