"""Run directories and the comparison report.

Same on-disk layout and report as the reference CLI's ``search`` / ``report``
commands (cli.py:263-534), so run directories from either side mix:

    <run>/config.yaml            copy of the experiment config
    <run>/summary.json           per-seed best raw, mean, best-of-k
    <run>/seed_<s>/evals.ndjson  one EvalRecord per evaluation (env.py:54-87)
    <run>/seed_<s>/report.json   SearchReport
    <run>/grid/...               the exhaustive (Megatron-grid) sweep

Searches run on the GPU (ppo.run_search, baselines.*); eval logs are written
in one block per search. Reading a run parses each log once into arrays and
computes best-so-far curves with a running maximum instead of per-record
Python loops, so reports over millions of evaluations stay cheap.
"""

from __future__ import annotations

import csv
import dataclasses
import io
import json
import shutil
import statistics
from pathlib import Path
from typing import Sequence

import numpy as np

from .baselines import megatron_exhaustive, random_walk, simulated_annealing
from .config import ExperimentConfig, load_config, resolve_config_path
from .env import EvalRecord, SearchEnv
from .report import SearchReport

__all__ = ["RunError", "SeedRun", "RunDir", "run_searches", "read_eval_arrays", "read_run", "comparison_table",
           "render_text", "render_table_csv", "render_curves_csv", "report"]

TABLE_COLUMNS = ("workload", "algorithm", "runs", "mean_best_raw", "best_of_k_raw", "normalized_over_rw",
                 "vs_exhaustive")


class RunError(ValueError):
    """A run directory is missing, unfinished, or incompatible."""


def _best_valid_record(records: Sequence[EvalRecord]) -> EvalRecord | None:
    best = None
    for r in records:
        if r.valid and (best is None or r.raw > best.raw):
            best = r
    return best


def _summarize(algo: str, budget: int, rows: list[dict]) -> dict:
    bests = [row["best_raw"] for row in rows]
    k = max(range(len(bests)), key=lambda i: (bests[i], -i))
    return {"algorithm": algo, "budget": budget, "runs": len(rows), "per_seed": rows,
            "mean_best_raw": statistics.fmean(bests), "best_of_k_raw": bests[k],
            "best_of_k_seed": rows[k]["seed"], "best_of_k_vector": rows[k]["best_vector"]}


def run_searches(config: str, algo: str, out_dir: str | Path, budget: int | None = None, seeds: int = 1,
                 seed0: int = 0) -> dict:
    """Seeded searches into a run directory (reference cmd_search, cli.py:263-347)."""
    config_path = resolve_config_path(config)
    cfg = load_config(config_path)
    if algo not in ("ppo", "sa", "rw", "exhaustive"):
        raise RunError(f"unknown algorithm {algo!r}")
    budget = cfg.ppo.budget if budget is None else budget
    if budget < 1 or seeds < 1:
        raise RunError("budget and seeds must be positive")
    out = Path(out_dir)
    if (out / "summary.json").exists():
        raise RunError(f"refusing to overwrite finished run directory {out}")
    out.mkdir(parents=True, exist_ok=True)
    shutil.copyfile(config_path, out / "config.yaml")

    def make_env(env_budget: int, log_path: Path) -> SearchEnv:
        return SearchEnv(cfg.model, cfg.hardware, cfg.space, context_len=cfg.simulation.context_len,
                         budget=env_budget, reward=cfg.reward, slo_tpot=cfg.simulation.slo_tpot,
                         log_path=log_path)

    rows = []
    if algo == "exhaustive":
        run_dir = out / "grid"
        run_dir.mkdir(exist_ok=True)
        rep = megatron_exhaustive(lambda b: make_env(b, run_dir / "evals.ndjson"), cfg.space)
        (run_dir / "report.json").write_text(rep.to_json() + "\n", encoding="utf-8")
        rows.append({"seed": None, "best_raw": rep.best_raw, "best_vector": list(rep.best_vector),
                     "evals": rep.evals})
        budget = rep.budget
    else:
        from .ppo import run_search

        for seed in range(seed0, seed0 + seeds):
            run_dir = out / f"seed_{seed}"
            run_dir.mkdir(exist_ok=True)
            with make_env(budget, run_dir / "evals.ndjson") as env:
                if algo == "ppo":
                    rep = run_search(env, dataclasses.replace(cfg.ppo, budget=budget), seed)
                elif algo == "sa":
                    rep = simulated_annealing(env, cfg.sa, budget, seed)
                else:
                    rep = random_walk(env, budget, seed)
            (run_dir / "report.json").write_text(rep.to_json() + "\n", encoding="utf-8")
            best = _best_valid_record(env.eval_log)
            rows.append({"seed": seed, "best_raw": best.raw if best else 0.0,
                         "best_vector": list(best.vector) if best else None, "evals": rep.evals})
    summary = _summarize(algo, budget, rows)
    (out / "summary.json").write_text(json.dumps(summary, indent=2) + "\n", encoding="utf-8")
    return summary


def read_eval_arrays(path: str | Path) -> dict[str, np.ndarray]:
    """An NDJSON eval log as arrays: index, vector [n, A], raw, reward, valid, reason."""
    idx, vec, raw, rew, valid, reason = [], [], [], [], [], []
    with open(path, encoding="utf-8") as fh:
        for line in fh:
            line = line.strip()
            if not line:
                continue
            d = json.loads(line)
            idx.append(d["index"])
            vec.append(d["vector"])
            raw.append(d["raw"])
            rew.append(d["reward"])
            valid.append(d["valid"])
            reason.append(d["reason"])
    return {"index": np.asarray(idx, dtype=np.int64), "vector": np.asarray(vec, dtype=np.int64),
            "raw": np.asarray(raw, dtype=np.float64), "reward": np.asarray(rew, dtype=np.float64),
            "valid": np.asarray(valid, dtype=bool), "reason": np.asarray(reason, dtype=object)}


@dataclasses.dataclass(frozen=True)
class SeedRun:
    seed: int | None
    best_raw: float
    curve: np.ndarray  # best-so-far valid raw after each evaluation


@dataclasses.dataclass(frozen=True)
class RunDir:
    path: Path
    cfg: ExperimentConfig
    workload: str
    algorithm: str
    seeds: tuple[SeedRun, ...]


def read_run(path: str | Path) -> RunDir:
    """One finished run directory (reference _read_run, cli.py:370-406)."""
    path = Path(path)
    config_path, summary_path = path / "config.yaml", path / "summary.json"
    if not config_path.is_file() or not summary_path.is_file():
        raise RunError(f"{path} is not a finished run directory (missing config.yaml or summary.json)")
    cfg = load_config(config_path)
    summary = json.loads(summary_path.read_text(encoding="utf-8"))
    seeds = []
    for sub in sorted(p for p in path.iterdir() if p.is_dir()):
        log = sub / "evals.ndjson"
        if not log.is_file():
            continue
        arr = read_eval_arrays(log)
        curve = np.maximum.accumulate(np.where(arr["valid"], arr["raw"], 0.0)) if arr["raw"].size else arr["raw"]
        if curve.size:
            curve = np.maximum(curve, 0.0)
        seed = None
        rp = sub / "report.json"
        if rp.is_file():
            seed = SearchReport.from_json(rp.read_text(encoding="utf-8")).seed
        seeds.append(SeedRun(seed, float(curve[-1]) if curve.size else 0.0, curve))
    if not seeds:
        raise RunError(f"{path} contains no eval logs")
    seeds.sort(key=lambda s: (s.seed is None, s.seed if s.seed is not None else 0))
    return RunDir(path, cfg, f"{cfg.model.name}@{cfg.simulation.context_len}", str(summary["algorithm"]),
                  tuple(seeds))


def _check_compatible(runs: Sequence[RunDir]) -> None:
    first: dict[str, RunDir] = {}
    for run in runs:
        prior = first.setdefault(run.workload, run)
        if prior is run:
            continue
        a, b = prior.cfg, run.cfg
        if not (a.model == b.model and a.hardware == b.hardware and a.space == b.space
                and a.simulation == b.simulation and a.reward == b.reward):
            raise RunError(f"run directories {prior.path} and {run.path} both claim workload {run.workload!r} "
                           "but their configs disagree; refusing to compare")


def comparison_table(runs: Sequence[RunDir]) -> list[dict]:
    """Per (workload, algorithm): runs, mean best raw, best-of-k, ratio to
    random walk's mean and to the exhaustive grid's best (cli.py:430-479)."""
    _check_compatible(runs)
    merged: dict[tuple[str, str], list[SeedRun]] = {}
    for run in runs:
        merged.setdefault((run.workload, run.algorithm), []).extend(run.seeds)
    rw_mean, ex_best = {}, {}
    for (workload, algo), seeds in merged.items():
        bests = [s.best_raw for s in seeds]
        if algo == "rw":
            rw_mean[workload] = statistics.fmean(bests)
        elif algo == "exhaustive":
            ex_best[workload] = max(bests)
    rows = []
    for (workload, algo), seeds in merged.items():
        bests = [s.best_raw for s in seeds]
        mean_best, best_k = statistics.fmean(bests), max(bests)
        rw, ex = rw_mean.get(workload, 0.0), ex_best.get(workload, 0.0)
        rows.append({"workload": workload, "algorithm": algo, "runs": len(bests), "mean_best_raw": mean_best,
                     "best_of_k_raw": best_k, "normalized_over_rw": mean_best / rw if rw > 0 else None,
                     "vs_exhaustive": best_k / ex if ex > 0 else None})
    return rows


def _cell(v) -> str:
    if v is None:
        return "-"
    if isinstance(v, float):
        return f"{v:.6f}"
    return str(v)


def render_text(rows: list[dict]) -> str:
    cells = [[_cell(row[c]) for c in TABLE_COLUMNS] for row in rows]
    widths = [max([len(h)] + [len(line[i]) for line in cells]) for i, h in enumerate(TABLE_COLUMNS)]

    def fmt(line):
        return "  ".join(t.ljust(w) for t, w in zip(line, widths)).rstrip()

    return "\n".join([fmt(TABLE_COLUMNS)] + [fmt(line) for line in cells])


def render_table_csv(rows: list[dict]) -> str:
    buf = io.StringIO()
    w = csv.writer(buf)
    w.writerow(TABLE_COLUMNS)
    for row in rows:
        w.writerow(["" if row[c] is None else row[c] for c in TABLE_COLUMNS])
    return buf.getvalue()


def render_curves_csv(runs: Sequence[RunDir]) -> str:
    """workload,algorithm,seed,eval_index,best_so_far_raw — one row per evaluation."""
    parts = ["workload,algorithm,seed,eval_index,best_so_far_raw\r\n"]
    for run in runs:
        for sr in run.seeds:
            label = "" if sr.seed is None else str(sr.seed)
            prefix = f"{_csv_field(run.workload)},{_csv_field(run.algorithm)},{label},"
            parts.append("".join(f"{prefix}{i},{b!r}\r\n" for i, b in enumerate(sr.curve.tolist())))
    return "".join(parts)


def _csv_field(text: str) -> str:
    buf = io.StringIO()
    csv.writer(buf).writerow([text])
    return buf.getvalue()[:-2]


def report(run_dirs: Sequence[str | Path], out: str | Path | None = None) -> str:
    """The comparison table as text; with ``out`` also table.csv and curves.csv."""
    runs = [read_run(d) for d in run_dirs]
    rows = comparison_table(runs)
    if out is not None:
        o = Path(out)
        o.mkdir(parents=True, exist_ok=True)
        (o / "table.csv").write_text(render_table_csv(rows), encoding="utf-8")
        (o / "curves.csv").write_text(render_curves_csv(runs), encoding="utf-8")
    return render_text(rows)
