"""Generate golden fixtures from the REFERENCE implementation itself.

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

For each workload it draws candidate index vectors (uniform over every head,
uniform over admissible axes, and structured grids), scores them with the
reference's own ``decode_strategy`` + ``simulate`` (pkg/src/shardsearch/
strategy.py:245-263, simulator.py:239-341) and stores the verdicts as exact
float64 bit patterns. A second family of fixtures records the reference's
sequential ``SearchEnv.step`` rewards (env.py:152-180) and the final
``EliteBuffer`` contents (policy.py:86-102) over candidate streams with
duplicates. The fixtures travel with the repo; the reference does not.
"""

from __future__ import annotations

import dataclasses
import itertools
import json
import sys
from pathlib import Path

import numpy as np

import shardsearch
from shardsearch import simulator as ref_sim
from shardsearch.config import load_config, packaged_config_path
from shardsearch.env import RewardConfig, SearchEnv
from shardsearch.model import HardwareSpec, ModelSpec
from shardsearch.policy import EliteBuffer
from shardsearch.simulator import SimRequest, simulate
from shardsearch.strategy import (
    ActionSpaceSpec,
    AxisChoice,
    canonical_fused_ops,
    decode_strategy,
    megatron_fine_dims,
)

OUT = Path(__file__).resolve().parent
REASONS = {"none": 0, "over_device_budget": 1, "layout_error": 2, "oom": 3, "slo_violation": 4}
FIELDS = ("throughput", "tpot_s", "memory_bytes", "compute_s", "comm_s", "pipeline_s")

H100 = dict(
    name="h100-sxm-cluster", peak_flops=989.0e12, hbm_bandwidth=3.35e12, hbm_capacity=80.0e9,
    intra_node_bw=450.0e9, inter_node_bw=50.0e9, node_size=8, device_budget=24000,
    kernel_overhead=2.0e-6, per_collective_latency=1.0e-6,
)
DENSE_OPS = ("embedding", "qkv_proj", "kv_cache_io", "attn_core", "attn_out_proj", "router_gate",
             "expert_ffn1", "expert_ffn2", "final_norm", "lm_head")


def packaged(name, **hw_over):
    cfg = load_config(packaged_config_path(name))
    hw = dataclasses.replace(cfg.hardware, **hw_over) if hw_over else cfg.hardware
    return cfg.model, hw, cfg.space, cfg.simulation.context_len, cfg.simulation.slo_tpot


def appendix_b(name):
    """SURVEY.md Appendix B workloads (BASELINE configs the reference does not ship)."""
    if name == "llama3_8b_h100x8":
        model = ModelSpec("llama3-8b", 32, 4096, 32, 128, 8, 21504, 1, 1, False, 128256, 2)
        hw = HardwareSpec(**{**H100, "device_budget": 8})
        space = ActionSpaceSpec(tp_domain=(1, 2, 4, 8), ep_domain=(1,), pp_domain=(1, 2, 4, 8), op_names=DENSE_OPS)
        return model, hw, space, 8192, 0.05
    if name == "llama3_70b_h100x64":
        model = ModelSpec("llama3-70b", 80, 8192, 64, 128, 8, 43008, 1, 1, False, 128256, 2)
        hw = HardwareSpec(**{**H100, "device_budget": 64})
        return model, hw, ActionSpaceSpec(op_names=DENSE_OPS), 16384, 0.05
    if name.startswith("dsv3_style_h100x256"):
        model = ModelSpec("dsv3-style", 61, 7168, 56, 128, 8, 3072, 256, 8, True, 129280, 2)
        hw = HardwareSpec(**{**H100, "device_budget": 256})
        slo = 0.02 if name.endswith("slo20ms") else 0.05
        return model, hw, ActionSpaceSpec(), 16384, slo
    raise KeyError(name)


def unit_small():
    """The reference unit tests' small_model/bare_hw pair (test_simulator.py:29-62)."""
    model = ModelSpec("unit", 4, 256, 8, 32, 4, 128, 8, 2, True, 4096, 2)
    hw = HardwareSpec("bare", 1e15, 3e12, 8e10, 9e11, 5e10, 8, 24000, 1e-7, 1e-6)
    return model, hw, ActionSpaceSpec(), 256, 0.050


def edge_odd():
    """Non-power-of-two degrees, odd dims, pins and a partial op list."""
    model = ModelSpec("odd", 6, 384, 12, 32, 4, 300, 15, 3, True, 1000, 4)
    hw = HardwareSpec("odd-hw", 3.3e14, 1.7e12, 2.5e8, 2.9e11, 3.1e10, 6, 90, 1.3e-6, 7e-7)
    space = ActionSpaceSpec(
        tp_domain=(1, 2, 3, 6, 12), ep_domain=(1, 3, 5, 15, 30), pp_domain=(1, 2, 3, 4),
        batch_domain=(1, 3, 7, 100, 333),
        op_names=("lm_head", "qkv_proj", "expert_ffn2", "attn_core", "shared_ffn1", "kv_cache_io"),
        pinned=(("expert_ffn1", AxisChoice.DIM1), ("attn_out_proj", AxisChoice.DIM0),
                ("shared_ffn2", AxisChoice.DIM0)),
    )
    return model, hw, space, 777, 1.5e-4


def noshared_default_space():
    """Default 12-op space over a model without shared experts (extra heads ignored)."""
    model = ModelSpec("noshared", 8, 1024, 16, 64, 4, 2048, 16, 2, False, 32000, 2)
    hw = HardwareSpec(**{**H100, "hbm_capacity": 4.0e9, "device_budget": 512})
    return model, hw, ActionSpaceSpec(), 4096, 6e-4


def workload_meta(model, hw, space, ctx, slo):
    return {
        "model": dataclasses.asdict(model),
        "hw": dataclasses.asdict(hw),
        "space": {
            "tp_domain": list(space.tp_domain), "ep_domain": list(space.ep_domain),
            "pp_domain": list(space.pp_domain), "batch_domain": list(space.batch_domain),
            "op_names": list(space.op_names),
            "pinned": [[n, int(a)] for n, a in space.pinned],
        },
        "context_len": ctx,
        "slo_tpot": slo,
    }


def admissible_sampler(model, space, rng, n):
    ops = {op.name: op for op in canonical_fused_ops(model)}
    cols = [rng.integers(0, k, size=n) for k in space.head_sizes[:4]]
    for name in space.op_names:
        op = ops.get(name)
        choices = [a for a in (0, 1, 2) if op is None or op.admits(AxisChoice(a))]
        cols.append(np.asarray(choices)[rng.integers(0, len(choices), size=n)])
    return np.stack(cols, axis=1)


def uniform_sampler(space, rng, n):
    return np.stack([rng.integers(0, k, size=n) for k in space.head_sizes], axis=1)


def megatron_grid(model, space):
    ops = canonical_fused_ops(model)
    by_name = dict(zip((op.name for op in ops), megatron_fine_dims(ops)))
    tail = [int(by_name.get(n, AxisChoice.UNSHARDED)) for n in space.op_names]
    grid = itertools.product(*(range(k) for k in space.head_sizes[:4]))
    return np.asarray([list(c) + tail for c in grid])


def score(model, hw, space, ctx, slo, vectors):
    out = {"reason": np.zeros(len(vectors), np.uint8)}
    for f in FIELDS:
        out[f] = np.zeros(len(vectors), np.float64)
    for i, vec in enumerate(vectors):
        r = simulate(SimRequest(model=model, hw=hw, strategy=decode_strategy(tuple(int(v) for v in vec), space),
                                context_len=ctx, slo_tpot=slo))
        out["reason"][i] = REASONS[r.invalid_reason.value]
        vals = (r.throughput, r.tpot_s, r.memory_bytes, r.breakdown.compute_s, r.breakdown.comm_s,
                r.breakdown.pipeline_s)
        for f, v in zip(FIELDS, vals):
            out[f][i] = float(v)
    return out


def save_eval(name, spec, vectors, sum_mode):
    model, hw, space, ctx, slo = spec
    vectors = np.asarray(vectors, dtype=np.int64)
    res = score(model, hw, space, ctx, slo, vectors)
    meta = workload_meta(model, hw, space, ctx, slo)
    meta["sum_mode"] = sum_mode
    meta["python"] = list(sys.version_info[:3])
    np.savez_compressed(
        OUT / f"eval_{name}.npz",
        meta=np.asarray(json.dumps(meta)),
        vectors=vectors.astype(np.uint8),
        **res,
    )
    counts = np.bincount(res["reason"], minlength=5)
    print(f"{name}: n={len(vectors)} reasons={counts.tolist()}")


def eval_fixtures():
    rng = np.random.default_rng(20250900217)
    neumaier = 1 if sys.version_info >= (3, 12) else 0
    sets = {
        "tiny": (packaged("tiny"), None),
        "moe_1p2t": (packaged("moe_1p2t_h100"), (5000, 5000, True)),
        "moe_1p6t": (packaged("moe_1p6t_h100"), (3000, 3000, False)),
        "moe_1p6t_2048": (packaged("moe_1p6t_h100", device_budget=2048), (5000, 5000, True)),
        "llama3_8b_h100x8": (appendix_b("llama3_8b_h100x8"), (2000, 5000, True)),
        "llama3_70b_h100x64": (appendix_b("llama3_70b_h100x64"), (2000, 4000, True)),
        "dsv3_style_h100x256": (appendix_b("dsv3_style_h100x256"), (2000, 4000, True)),
        "dsv3_style_h100x256_slo20ms": (appendix_b("dsv3_style_h100x256_slo20ms"), (1000, 3000, False)),
        "unit_small": (unit_small(), (2000, 4000, True)),
        "edge_odd": (edge_odd(), (3000, 5000, False)),
        "noshared_default_space": (noshared_default_space(), (2000, 3000, False)),
    }
    for name, (spec, plan) in sets.items():
        model, hw, space, ctx, slo = spec
        if plan is None:
            vectors = np.asarray(list(itertools.product(*(range(k) for k in space.head_sizes))))
        else:
            n_u, n_a, grid = plan
            parts = [uniform_sampler(space, rng, n_u), admissible_sampler(model, space, rng, n_a)]
            if grid:
                parts.append(megatron_grid(model, space))
            vectors = np.concatenate(parts)
        save_eval(name, spec, vectors, neumaier)

    # Python <= 3.11 semantics: the simulator's sum() as a naive left fold.
    spec = packaged("moe_1p2t_h100")
    ref_sim.sum = lambda xs: _naive_sum(xs)
    try:
        vectors = np.concatenate([admissible_sampler(spec[0], spec[2], rng, 4000), megatron_grid(spec[0], spec[2])])
        save_eval("moe_1p2t_naive_sum", spec, vectors, 0)
        spec = unit_small()
        save_eval("unit_small_naive_sum", spec, admissible_sampler(spec[0], spec[2], rng, 3000), 0)
    finally:
        del ref_sim.sum


def _naive_sum(xs):
    total = 0
    for x in xs:
        total = total + x
    return total


def search_fixtures():
    """Sequential env.step rewards + EliteBuffer contents over streams with repeats."""
    rng = np.random.default_rng(7)
    cases = []
    model, hw, space, ctx, slo = packaged("moe_1p2t_h100")
    base = admissible_sampler(model, space, rng, 3000)
    # repeats: re-offer earlier vectors later in the stream
    reps = base[rng.integers(0, 3000, size=1000)]
    stream = np.concatenate([base, reps])
    stream = stream[rng.permutation(len(stream))]
    cases.append(("moe_1p2t_stream", (model, hw, space, ctx, slo), stream, 0.0, RewardConfig()))
    cases.append(("moe_1p2t_stream_b0", (model, hw, space, ctx, slo), stream[:2000], 35.0,
                  RewardConfig(alpha=0.5, beta=2.0, invalid_penalty=-3.0)))
    tiny = packaged("tiny")
    tv = np.asarray(list(itertools.product(*(range(k) for k in tiny[2].head_sizes))))
    tstream = tv[rng.integers(0, len(tv), size=4000)]
    cases.append(("tiny_stream", tiny, tstream, 0.0, RewardConfig()))

    for name, (model, hw, space, ctx, slo), stream, b0, rcfg in cases:
        env = SearchEnv(model, hw, space, ctx, budget=len(stream), reward=rcfg, slo_tpot=slo)
        env.best_raw = b0
        rewards, raws, valid = [], [], []
        for vec in stream:
            r, raw, ok = env.step(tuple(int(v) for v in vec))
            rewards.append(r)
            raws.append(raw)
            valid.append(ok)
        elites = {}
        for cap in (1, 3, 8, 32):
            buf = EliteBuffer(cap)
            for vec, r, ok in zip(stream, rewards, valid):
                if ok:
                    buf.offer(vec, r)
            elites[cap] = buf.entries
        meta = workload_meta(model, hw, space, ctx, slo)
        meta["sum_mode"] = 1 if sys.version_info >= (3, 12) else 0
        meta["reward"] = dataclasses.asdict(rcfg)
        meta["b0"] = b0
        meta["best_raw_final"] = env.best_raw
        payload = {}
        for cap, entries in elites.items():
            payload[f"elite{cap}_vectors"] = np.asarray([e.vector for e in entries], dtype=np.uint8).reshape(-1, space.vector_length)
            payload[f"elite{cap}_rewards"] = np.asarray([e.reward for e in entries], dtype=np.float64)
        np.savez_compressed(
            OUT / f"search_{name}.npz",
            meta=np.asarray(json.dumps(meta)),
            vectors=np.asarray(stream, dtype=np.uint8),
            rewards=np.asarray(rewards, dtype=np.float64),
            raws=np.asarray(raws, dtype=np.float64),
            valid=np.asarray(valid, dtype=bool),
            **payload,
        )
        print(f"{name}: n={len(stream)} valid={int(np.sum(valid))} best={env.best_raw}")


if __name__ == "__main__":
    print("reference", shardsearch.__file__, "python", sys.version.split()[0])
    eval_fixtures()
    search_fixtures()
