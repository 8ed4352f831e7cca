"""Run-directory reading and the comparison report (runs.py) against the
reference CLI's own `report` output on run directories it wrote
(tests/golden/report_runs, tests/golden/report_expected; made by
tests/golden/make_golden_report.py)."""

from __future__ import annotations

import json
import shutil
from pathlib import Path

import numpy as np
import pytest

from paper_2509_00217_b200.runs import RunError, read_eval_arrays, read_run, report

GOLD = Path(__file__).parent / "golden"
RUNS = [GOLD / "report_runs" / a for a in ("rw", "sa", "ppo", "exhaustive")]


def test_report_matches_reference_byte_for_byte(tmp_path):
    text = report(RUNS, tmp_path)
    assert text + "\n" == (GOLD / "report_expected" / "table.txt").read_text()
    for name in ("table.csv", "curves.csv"):
        assert (tmp_path / name).read_bytes() == (GOLD / "report_expected" / name).read_bytes(), name


def test_curves_are_running_max_of_valid_raw():
    run = read_run(RUNS[0])
    arr = read_eval_arrays(RUNS[0] / "seed_0" / "evals.ndjson")
    best, want = 0.0, []
    for raw, ok in zip(arr["raw"], arr["valid"]):
        if ok and raw > best:
            best = raw
        want.append(best)
    np.testing.assert_array_equal(run.seeds[0].curve, want)
    assert [s.seed for s in run.seeds] == [0, 1, 2]


def test_unfinished_and_incompatible_runs_are_refused(tmp_path):
    with pytest.raises(RunError):
        read_run(tmp_path)
    other = tmp_path / "other"
    shutil.copytree(RUNS[0], other)
    cfg = (other / "config.yaml").read_text().replace("slo_tpot:", "slo_tpot: 0.07 #", 1)
    (other / "config.yaml").write_text(cfg)
    summary = json.loads((other / "summary.json").read_text())
    assert summary["algorithm"] == "rw"
    with pytest.raises(RunError):
        report([RUNS[0], other])
