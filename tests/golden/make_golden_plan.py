"""Golden layer plans and explain() text from the REFERENCE (layout.py
plan_layer / LayerPlan.describe, simulator.py explain), made in this container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_plan.py

For each config, seeded random index vectors (uniform, and admissible-axis
biased so most plans exist): the index vector, the pre/layer/post plan
descriptions (or the LayoutError message), and the full explain() text.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from shardsearch.config import load_config, packaged_config_path
from shardsearch.layout import LayoutError, plan_layer
from shardsearch.simulator import SimRequest, explain
from shardsearch.strategy import AxisChoice, canonical_fused_ops, decode_strategy

OUT = Path(__file__).resolve().parent
CONFIGS = ("tiny", "moe_1p2t_h100", "moe_1p6t_h100", "llama3_70b_h100x64", "dsv3_style_h100x256")


def main():
    cases = []
    for ci, name in enumerate(CONFIGS):
        try:
            cfg = load_config(packaged_config_path(name))
        except Exception:  # BASELINE Appendix-B workloads: this repo's YAML, parsed by the reference
            cfg = load_config(Path(__file__).resolve().parents[2] / "paper_2509_00217_b200" / "configs" / f"{name}.yaml")
        ops = canonical_fused_ops(cfg.model)
        by_name = {op.name: op for op in ops}
        segs = {"pre": tuple(op for op in ops if op.name == "embedding"),
                "layer": tuple(op for op in ops if op.per_layer),
                "post": tuple(op for op in ops if not op.per_layer and op.name != "embedding")}
        rng = np.random.default_rng(100 + ci)
        sizes = cfg.space.head_sizes
        for i in range(120):
            vec = [int(rng.integers(k)) for k in sizes]
            if i % 2:  # admissible axes only
                for h, op_name in enumerate(cfg.space.op_names):
                    op = by_name[op_name]
                    allowed = [a for a in (0, 1, 2) if op.admits(AxisChoice(a))]
                    vec[4 + h] = int(allowed[int(rng.integers(len(allowed)))])
            s = decode_strategy(tuple(vec), cfg.space)
            plans = {}
            for seg, seg_ops in segs.items():
                try:
                    plans[seg] = plan_layer(cfg.model, seg_ops, s, s.batch, cfg.hardware.node_size).describe()
                except LayoutError as exc:
                    plans[seg] = "LayoutError: " + str(exc)
            text = explain(SimRequest(cfg.model, cfg.hardware, s, cfg.simulation.context_len,
                                      cfg.simulation.slo_tpot))
            cases.append({"config": name, "vector": vec, "plans": plans, "explain": text})
    (OUT / "plans_reference.json").write_text(json.dumps(cases))
    print(len(cases), "cases")


if __name__ == "__main__":
    main()
