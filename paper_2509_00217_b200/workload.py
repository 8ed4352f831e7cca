"""Workload compiler: (model, hardware, action space, context, SLO) -> POD.

Produces the ``ls_workload_desc`` struct of include/ls_eval.h as a ctypes
structure. The evaluator context builds all per-workload tables from it; the
test oracle consumes the same struct, so both read one definition of "the
workload". Accepts the reference's own spec objects as well as ours (field
names are identical), which is what makes the evaluator a drop-in behind
``SearchEnv.evaluate_raw`` (reference env.py:140-150).
"""

from __future__ import annotations

import ctypes
import sys
from dataclasses import dataclass

from .strategy import CANONICAL_OP_NAMES, AxisChoice

__all__ = [
    "LS_ABI_VERSION", "LS_MAX_DOMAIN", "LS_MAX_HEADS", "LS_NUM_OPS", "SUM_NAIVE", "SUM_NEUMAIER",
    "default_sum_mode", "WorkloadDesc", "Workload", "build_desc",
]

LS_ABI_VERSION = 1
LS_MAX_DOMAIN = 64
LS_MAX_HEADS = 64
LS_NUM_OPS = 12
SUM_NAIVE = 0
SUM_NEUMAIER = 1


def default_sum_mode() -> int:
    """Python's float ``sum()`` is Neumaier-compensated from 3.12 on.

    The reference's ``_plan_times`` (simulator.py:232-235) inherits whichever
    the interpreter does; parity is with the interpreter running beside us.
    """
    return SUM_NEUMAIER if sys.version_info >= (3, 12) else SUM_NAIVE


class WorkloadDesc(ctypes.Structure):
    """ctypes mirror of ``ls_workload_desc`` (include/ls_eval.h)."""

    _fields_ = [
        ("abi_version", ctypes.c_uint32),
        ("sum_mode", ctypes.c_uint32),
        ("num_layers", ctypes.c_int64),
        ("hidden_dim", ctypes.c_int64),
        ("num_heads", ctypes.c_int64),
        ("head_dim", ctypes.c_int64),
        ("num_kv_heads", ctypes.c_int64),
        ("ffn_dim", ctypes.c_int64),
        ("num_experts", ctypes.c_int64),
        ("experts_per_token", ctypes.c_int64),
        ("vocab_size", ctypes.c_int64),
        ("dtype_bytes", ctypes.c_int64),
        ("has_shared_expert", ctypes.c_int32),
        ("reserved0", ctypes.c_int32),
        ("peak_flops", ctypes.c_double),
        ("hbm_bandwidth", ctypes.c_double),
        ("hbm_capacity", ctypes.c_double),
        ("intra_node_bw", ctypes.c_double),
        ("inter_node_bw", ctypes.c_double),
        ("node_size", ctypes.c_int64),
        ("device_budget", ctypes.c_int64),
        ("kernel_overhead", ctypes.c_double),
        ("per_collective_latency", ctypes.c_double),
        ("context_len", ctypes.c_int64),
        ("slo_tpot", ctypes.c_double),
        ("domain_len", ctypes.c_int32 * 4),
        ("domain", (ctypes.c_int64 * LS_MAX_DOMAIN) * 4),
        ("vector_length", ctypes.c_int32),
        ("op_head", ctypes.c_int8 * LS_NUM_OPS),
        ("op_pinned", ctypes.c_int8 * LS_NUM_OPS),
    ]


_INT53 = 1 << 53


def build_desc(model, hw, space, context_len: int, slo_tpot: float, sum_mode: int | None = None) -> WorkloadDesc:
    """Flatten one workload; raises ValueError for what the kernel cannot represent."""
    d = WorkloadDesc()
    d.abi_version = LS_ABI_VERSION
    d.sum_mode = default_sum_mode() if sum_mode is None else int(sum_mode)
    for name in (
        "num_layers", "hidden_dim", "num_heads", "head_dim", "num_kv_heads", "ffn_dim",
        "num_experts", "experts_per_token", "vocab_size", "dtype_bytes",
    ):
        setattr(d, name, int(getattr(model, name)))
    d.has_shared_expert = 1 if model.has_shared_expert else 0
    for name in ("peak_flops", "hbm_bandwidth", "hbm_capacity", "intra_node_bw", "inter_node_bw",
                 "kernel_overhead", "per_collective_latency"):
        setattr(d, name, float(getattr(hw, name)))
    d.node_size = int(hw.node_size)
    d.device_budget = int(hw.device_budget)
    d.context_len = int(context_len)
    d.slo_tpot = float(slo_tpot)
    domains = (space.tp_domain, space.ep_domain, space.pp_domain, space.batch_domain)
    for h, dom in enumerate(domains):
        if len(dom) > LS_MAX_DOMAIN:
            raise ValueError(f"domain {h} has {len(dom)} entries; the evaluator supports {LS_MAX_DOMAIN}")
        d.domain_len[h] = len(dom)
        for j, v in enumerate(dom):
            d.domain[h][j] = int(v)
    A = 4 + len(space.op_names)
    if A > LS_MAX_HEADS:
        raise ValueError(f"vector length {A} exceeds {LS_MAX_HEADS}")
    d.vector_length = A
    pins = dict(space.pinned)
    for k, name in enumerate(CANONICAL_OP_NAMES):
        if name in space.op_names:
            d.op_head[k] = 4 + list(space.op_names).index(name)
            d.op_pinned[k] = 0
        else:
            d.op_head[k] = -1
            d.op_pinned[k] = int(pins.get(name, AxisChoice.UNSHARDED))
    _check_exactness(d)
    return d


def _check_exactness(d: WorkloadDesc) -> None:
    """Every integer the cost model turns into a double must be exact (< 2^53).

    Python's int/int true division is correctly rounded for any size; IEEE
    double division of the converted operands equals it only when both
    conversions are exact. The largest products are the weight byte counts.
    """
    h = d.hidden_dim
    qkv = (d.num_heads + 2 * d.num_kv_heads) * d.head_dim
    expert = 2 * h * d.ffn_dim
    dense = (2 * d.vocab_size * h + d.num_layers * (h * qkv + d.num_heads * d.head_dim * h)
             + d.num_layers * h * d.num_experts + (d.num_layers * expert if d.has_shared_expert else 0)
             + d.num_layers * 4 * h + h)
    routed = d.num_layers * d.num_experts * expert
    max_batch = max(d.domain[3][j] for j in range(d.domain_len[3]))
    biggest = max(dense * d.dtype_bytes, routed * d.dtype_bytes,
                  max_batch * max(h, d.vocab_size, qkv, d.ffn_dim) * d.dtype_bytes * max(1, d.experts_per_token))
    if biggest >= _INT53:
        raise ValueError("workload integers exceed 2^53; exact double conversion is not guaranteed")


@dataclass(frozen=True)
class Workload:
    """Everything a simulate() call fixes except the strategy."""

    model: object
    hw: object
    space: object
    context_len: int
    slo_tpot: float = 0.050
    sum_mode: int | None = None

    def desc(self) -> WorkloadDesc:
        return build_desc(self.model, self.hw, self.space, self.context_len, self.slo_tpot, self.sum_mode)

    def key(self) -> bytes:
        """Identity of the workload as the evaluator sees it (for context caches)."""
        return bytes(self.desc())
