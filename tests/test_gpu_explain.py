"""explain() (simulator.py) against the reference's explain text for 600
strategies over five workloads (tests/golden/plans_reference.json): GPU
verdict and times, host plan."""

from __future__ import annotations

import json
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

pytest.importorskip("torch")

from paper_2509_00217_b200.config import load_config, resolve_config_path  # noqa: E402
from paper_2509_00217_b200.simulator import SimRequest, explain  # noqa: E402
from paper_2509_00217_b200.strategy import decode_strategy  # noqa: E402

CASES = json.loads((Path(__file__).parent / "golden" / "plans_reference.json").read_text())


def test_explain_text_matches_reference():
    cfgs = {name: load_config(resolve_config_path(name)) for name in {c["config"] for c in CASES}}
    for case in CASES:
        cfg = cfgs[case["config"]]
        s = decode_strategy(tuple(case["vector"]), cfg.space)
        text = explain(SimRequest(cfg.model, cfg.hardware, s, cfg.simulation.context_len, cfg.simulation.slo_tpot))
        assert text == case["explain"], (case["config"], case["vector"])
