"""Golden run directories and report outputs from the REFERENCE CLI
(cli.py cmd_search / cmd_report), made in this container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_report.py

Writes tests/golden/report_runs/{rw,sa,ppo,exhaustive}/ (config.yaml,
summary.json, per-seed evals.ndjson + report.json) for the tiny config, and
tests/golden/report_expected/{table.txt,table.csv,curves.csv}.
"""

from __future__ import annotations

import contextlib
import io
import shutil
from pathlib import Path

from shardsearch.cli import main as cli

OUT = Path(__file__).resolve().parent
RUNS = OUT / "report_runs"
EXPECTED = OUT / "report_expected"


def main():
    shutil.rmtree(RUNS, ignore_errors=True)
    shutil.rmtree(EXPECTED, ignore_errors=True)
    RUNS.mkdir()
    EXPECTED.mkdir()
    jobs = (("rw", ["--budget", "150", "--seeds", "3"]), ("sa", ["--budget", "150", "--seeds", "2", "--seed0", "5"]),
            ("ppo", ["--budget", "100", "--seeds", "2"]), ("exhaustive", []))
    for algo, extra in jobs:
        with contextlib.redirect_stdout(io.StringIO()):
            rc = cli(["search", "--config", "tiny", "--algo", algo, "--out", str(RUNS / algo)] + extra)
        assert rc == 0, (algo, rc)
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli(["report"] + [str(RUNS / a) for a, _ in jobs] + ["--out", str(EXPECTED)])
    assert rc == 0
    text = buf.getvalue().splitlines()
    (EXPECTED / "table.txt").write_text("\n".join(text[:-1]) + "\n")  # drop the "wrote ..." line
    print("\n".join(text[:-1]))


if __name__ == "__main__":
    main()
