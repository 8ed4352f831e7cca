"""Scalar ``simulate()`` facade over the batched GPU evaluator.

Same types and contract as the reference (pkg/src/shardsearch/simulator.py:
48-97, :239-341): ``InvalidReason``, ``SimRequest`` (validated the same way),
``TimeBreakdown``, ``SimResult`` and ``simulate(req)``. The numbers come from
libls_eval.so — a one-candidate batch — and are bit-identical to the
reference's; only the human-readable ``detail`` text is produced on the host
(the reference never logs it, env.py:165-172).

A ``Strategy`` is self-describing (degree values, op axes, pins), so the
facade keeps one evaluator per (model, hardware, context, SLO, op list, pins)
whose domains grow to cover every degree value it has been asked about.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass
from enum import Enum


from .evaluator import Evaluator
from .spec import HardwareSpec, ModelSpec
from .strategy import (
    CANONICAL_OP_NAMES,
    DEFAULT_BATCH_DOMAIN,
    DEFAULT_DEGREE_DOMAIN,
    ActionSpaceSpec,
    AxisChoice,
    Strategy,
    canonical_fused_ops,
)
from .workload import LS_MAX_DOMAIN, Workload

__all__ = ["InvalidReason", "SimRequest", "TimeBreakdown", "SimResult", "simulate", "simulate_vector",
           "result_from_row", "layout_error_detail", "explain"]


class InvalidReason(str, Enum):
    NONE = "none"
    OVER_DEVICE_BUDGET = "over_device_budget"
    LAYOUT_ERROR = "layout_error"
    OOM = "oom"
    SLO_VIOLATION = "slo_violation"


_BY_CODE = {0: InvalidReason.NONE, 1: InvalidReason.OVER_DEVICE_BUDGET, 2: InvalidReason.LAYOUT_ERROR,
            3: InvalidReason.OOM, 4: InvalidReason.SLO_VIOLATION}


@dataclass(frozen=True)
class SimRequest:
    model: ModelSpec
    hw: HardwareSpec
    strategy: Strategy
    context_len: int
    slo_tpot: float = 0.050
    phase: str = "decode"

    def __post_init__(self) -> None:
        if self.phase != "decode":
            raise ValueError(f"only the decode phase is modeled, got phase={self.phase!r}")
        if self.context_len < 1:
            raise ValueError(f"context_len must be positive, got {self.context_len}")
        if self.slo_tpot <= 0:
            raise ValueError(f"slo_tpot must be positive, got {self.slo_tpot}")


@dataclass(frozen=True)
class TimeBreakdown:
    compute_s: float
    comm_s: float
    pipeline_s: float

    @property
    def total_s(self) -> float:
        return self.compute_s + self.comm_s + self.pipeline_s


@dataclass(frozen=True)
class SimResult:
    valid: bool
    invalid_reason: InvalidReason
    throughput: float
    tpot_s: float
    memory_bytes: float
    breakdown: TimeBreakdown
    detail: str = ""


# ---------------------------------------------------------------------------
# host-side detail text (layout.py / simulator.py messages, first failing check)


def _extent(model, op: str, axis: AxisChoice):
    h = model.hidden_dim
    table = {
        "embedding": {AxisChoice.DIM0: model.vocab_size, AxisChoice.DIM1: h},
        "qkv_proj": {AxisChoice.DIM0: h, AxisChoice.DIM1: model.num_heads},
        "attn_core": {AxisChoice.DIM1: model.num_heads},
        "attn_out_proj": {AxisChoice.DIM0: model.num_heads, AxisChoice.DIM1: h},
        "expert_ffn1": {AxisChoice.DIM0: h, AxisChoice.DIM1: model.ffn_dim},
        "expert_ffn2": {AxisChoice.DIM0: model.ffn_dim, AxisChoice.DIM1: h},
        "shared_ffn1": {AxisChoice.DIM0: h, AxisChoice.DIM1: model.ffn_dim},
        "shared_ffn2": {AxisChoice.DIM0: model.ffn_dim, AxisChoice.DIM1: h},
        "lm_head": {AxisChoice.DIM0: h, AxisChoice.DIM1: model.vocab_size},
    }
    return table.get(op, {}).get(axis)


def layout_error_detail(model, strategy) -> str:
    """Message of the first LayoutError the reference walk would raise
    (simulator.py:268-276, layout.py:368-374, :214-221)."""
    s = strategy
    if model.num_layers % s.pp:
        return f"pp={s.pp} does not divide num_layers={model.num_layers}"
    if s.ep > model.num_experts:
        return f"ep={s.ep} exceeds num_experts={model.num_experts}"
    if model.num_experts % s.ep:
        return f"ep={s.ep} does not divide num_experts={model.num_experts}"
    ops = canonical_fused_ops(model)
    walk = [op for op in ops if op.per_layer] + [ops[0]] + [op for op in ops if not op.per_layer and op.name != "embedding"]
    for op in walk:
        axis = AxisChoice(s.axis_of(op.name))
        if not op.admits(axis):
            return f"{op.name} does not admit shard axis {axis.name}"
        if axis != AxisChoice.UNSHARDED and s.tp > 1:
            ext = _extent(model, op.name, axis)
            if ext is None:
                return f"{op.name} has no shardable extent on {axis.name}"
            if ext % s.tp:
                return f"{op.name} cannot shard {axis.name}: extent {ext} not divisible by tp={s.tp}"
    return "layout error"


_FIELDS = ("throughput", "tpot_s", "memory_bytes", "compute_s", "comm_s", "pipeline_s")


def result_from_row(row: dict, i: int, model=None, hw=None, strategy=None, slo=None) -> SimResult:
    """SimResult of candidate i of a numpy result dict (reason + six fields)."""
    return result_from_verdict(int(row["reason"][i]), tuple(float(row[k][i]) if k in row else 0.0 for k in _FIELDS),
                               model, hw, strategy, slo)


def result_from_verdict(code: int, fields, model=None, hw=None, strategy=None, slo=None) -> SimResult:
    """SimResult of one verdict: reason code + the six numbers in _FIELDS order."""
    if code == 255:
        from .strategy import DecodingError

        raise DecodingError("index vector out of range for the action space")
    reason = _BY_CODE[code]
    f = dict(zip(_FIELDS, fields))
    detail = ""
    if strategy is not None:
        if reason is InvalidReason.OVER_DEVICE_BUDGET:
            detail = f"needs {strategy.world_size} devices, budget is {hw.device_budget}"
        elif reason is InvalidReason.LAYOUT_ERROR:
            detail = layout_error_detail(model, strategy)
        elif reason is InvalidReason.OOM:
            detail = f"needs {f['memory_bytes'] / 1e9:.2f} GB, capacity is {hw.hbm_capacity / 1e9:.2f} GB"
        elif reason is InvalidReason.SLO_VIOLATION:
            detail = f"tpot {f['tpot_s'] * 1e3:.2f} ms exceeds SLO {slo * 1e3:.2f} ms"
    return SimResult(
        valid=reason is InvalidReason.NONE,
        invalid_reason=reason,
        throughput=f["throughput"],
        tpot_s=f["tpot_s"],
        memory_bytes=f["memory_bytes"],
        breakdown=TimeBreakdown(f["compute_s"], f["comm_s"], f["pipeline_s"]),
        detail=detail,
    )


# ---------------------------------------------------------------------------
# evaluator cache for free-standing strategies


class _FacadeCache:
    def __init__(self) -> None:
        self._lock = threading.Lock()
        self._entries: dict = {}

    def evaluator_for(self, req: SimRequest):
        s = req.strategy
        key = (req.model, req.hw, int(req.context_len), float(req.slo_tpot), tuple(s.op_names),
               tuple(s.pinned_dims))
        with self._lock:
            ent = self._entries.get(key)
            doms = ent[1] if ent else [list(DEFAULT_DEGREE_DOMAIN), list(DEFAULT_DEGREE_DOMAIN),
                                       list(DEFAULT_DEGREE_DOMAIN), list(DEFAULT_BATCH_DOMAIN)]
            grew = False
            for h, v in enumerate((s.tp, s.ep, s.pp, s.batch)):
                if v not in doms[h]:
                    if len(doms[h]) >= LS_MAX_DOMAIN:
                        doms[h] = doms[h][: LS_MAX_DOMAIN // 2]
                    doms[h].append(v)
                    grew = True
            if ent is None or grew:
                space = ActionSpaceSpec(tuple(doms[0]), tuple(doms[1]), tuple(doms[2]), tuple(doms[3]),
                                        op_names=tuple(s.op_names) if s.op_names else ("embedding",),
                                        pinned=tuple(s.pinned_dims))
                # a replaced evaluator is not closed here: another thread may be
                # scoring with it; reference counting frees it
                ev = Evaluator(Workload(req.model, req.hw, space, req.context_len, req.slo_tpot))
                ent = (ev, doms)
                self._entries[key] = ent
            # the domains frozen into this evaluator (a later growth builds a new one)
            return ent[0], tuple(tuple(d) for d in doms)


_CACHE = _FacadeCache()


def simulate(req: SimRequest) -> SimResult:
    """Score one strategy on the GPU (reference simulator.py:239-341)."""
    ev, doms = _CACHE.evaluator_for(req)
    s = req.strategy
    vec = [doms[0].index(s.tp), doms[1].index(s.ep), doms[2].index(s.pp), doms[3].index(s.batch)]
    vec += [int(a) for a in s.op_dims] if s.op_names else [0]
    code, fields = ev.evaluate_one(vec)
    return result_from_verdict(code, fields, req.model, req.hw, s, req.slo_tpot)


def simulate_vector(ev: Evaluator, vector, model=None, hw=None, strategy=None, slo=None) -> SimResult:
    """Score one index vector of ``ev``'s action space (ls_evaluate_one: no
    allocation, no copy, no stream sync — the scalar seam's fast path)."""
    code, fields = ev.evaluate_one(vector)
    return result_from_verdict(code, fields, model, hw, strategy, slo)


def explain(req: SimRequest) -> str:
    """Human-readable account of one strategy (reference simulator.py:344-374):
    verdict and times from the GPU evaluator, per-layer plan from the host
    planner (plan.py)."""
    from .plan import plan_layer

    model, hw, s = req.model, req.hw, req.strategy
    result = simulate(req)
    lines = [f"strategy: tp={s.tp} ep={s.ep} pp={s.pp} batch={s.batch} world_size={s.world_size}",
             "fine dims: " + " ".join(f"{n}={AxisChoice(a).name.lower()}" for n, a in zip(s.op_names, s.op_dims)),
             f"valid: {result.valid}" + ("" if result.valid else f" ({result.invalid_reason.value}: {result.detail})")]
    if result.invalid_reason in (InvalidReason.OVER_DEVICE_BUDGET, InvalidReason.LAYOUT_ERROR):
        return "\n".join(lines)
    lines.append(f"memory per device: {result.memory_bytes / 1e9:.3f} GB")
    if result.invalid_reason is InvalidReason.OOM:
        return "\n".join(lines)
    lines.append(f"tpot: {result.tpot_s * 1e3:.4f} ms")
    b = result.breakdown
    lines.append(f"breakdown: compute {b.compute_s * 1e3:.4f} ms, comm {b.comm_s * 1e3:.4f} ms, "
                 f"pipeline {b.pipeline_s * 1e3:.4f} ms")
    if result.valid:
        lines.append(f"throughput: {result.throughput:.4f} tokens/s/chip")
    layer_ops = tuple(op for op in canonical_fused_ops(model) if op.per_layer)
    plan = plan_layer(model, layer_ops, s, s.batch, hw.node_size)
    lines.append("per-layer plan:")
    lines.extend("  " + ln for ln in plan.describe().splitlines())
    return "\n".join(lines)
