"""B200-native batched strategy evaluation for Learn to Shard (arXiv 2509.00217).

The reference's per-candidate cost-model path (SearchEnv.step ->
evaluate_raw -> simulate, pkg/src/shardsearch/env.py:140-180,
simulator.py:239-341) rebuilt as hand-written sm_100a CUDA behind a C ABI
(include/ls_eval.h, libls_eval.so), with the reference's Python API on top.
"""

from .spec import HardwareSpec, ModelSpec, ParameterCount, count_parameters
from .strategy import (
    ActionSpaceSpec,
    AxisChoice,
    DecodingError,
    EncodingError,
    FusedOpDescriptor,
    OpClass,
    Strategy,
    canonical_fused_ops,
    decode_strategy,
    encode_strategy,
    megatron_fine_dims,
)
from .workload import Workload

__all__ = [
    "ActionSpaceSpec", "AxisChoice", "DecodingError", "EncodingError", "FusedOpDescriptor", "HardwareSpec",
    "ModelSpec", "OpClass", "ParameterCount", "Strategy", "Workload", "canonical_fused_ops", "count_parameters",
    "decode_strategy", "encode_strategy", "megatron_fine_dims",
]

__version__ = "0.1.0"
