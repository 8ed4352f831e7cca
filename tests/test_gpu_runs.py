"""run_searches (runs.py) writes the same run directories as the reference
CLI's `search` (tests/golden/report_runs, made by the reference): identical
eval logs and summaries; reports equal except their wall-clock field."""

from __future__ import annotations

import json
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

pytest.importorskip("torch")

from paper_2509_00217_b200.runs import report, run_searches  # noqa: E402

GOLD = Path(__file__).parent / "golden" / "report_runs"
JOBS = (("rw", dict(budget=150, seeds=3)), ("sa", dict(budget=150, seeds=2, seed0=5)),
        ("ppo", dict(budget=100, seeds=2)), ("exhaustive", {}))


@pytest.mark.parametrize("algo,kw", JOBS)
def test_run_directory_matches_reference(tmp_path, algo, kw):
    out = tmp_path / algo
    run_searches("tiny", algo, out, **kw)
    ref = GOLD / algo
    assert json.loads((out / "summary.json").read_text()) == json.loads((ref / "summary.json").read_text())
    subs = sorted(p.name for p in ref.iterdir() if p.is_dir())
    assert sorted(p.name for p in out.iterdir() if p.is_dir()) == subs
    for sub in subs:
        assert (out / sub / "evals.ndjson").read_bytes() == (ref / sub / "evals.ndjson").read_bytes(), sub
        got = json.loads((out / sub / "report.json").read_text())
        want = json.loads((ref / sub / "report.json").read_text())
        got.pop("wall_clock_s"), want.pop("wall_clock_s")
        assert got == want, sub


def test_report_over_gpu_runs_equals_reference_report(tmp_path):
    for algo, kw in JOBS:
        run_searches("tiny", algo, tmp_path / algo, **kw)
    ours = report([tmp_path / a for a, _ in JOBS], tmp_path / "rep")
    theirs = report([GOLD / a for a, _ in JOBS])
    assert ours == theirs
