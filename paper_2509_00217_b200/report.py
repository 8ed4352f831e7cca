"""Search reports (reference ppo.py:362-463): the winner of an eval-record
stream — by reward (learning searches) or by raw over valid records
(exhaustive baseline) — earliest record on ties."""

from __future__ import annotations

import json
from dataclasses import dataclass
from typing import Sequence

from .env import EvalRecord

__all__ = ["SearchReport", "build_report"]


@dataclass(frozen=True)
class SearchReport:
    algorithm: str
    seed: int | None
    budget: int
    evals: int
    best_vector: tuple[int, ...]
    best_raw: float
    best_reward: float
    best_valid: bool
    restarts: tuple[int, ...]
    rewards: tuple[float, ...]
    raws: tuple[float, ...]
    wall_clock_s: float

    def best_so_far_raw(self) -> tuple[float, ...]:
        best, curve = 0.0, []
        for raw in self.raws:
            best = max(best, raw)
            curve.append(best)
        return tuple(curve)

    def to_json(self) -> str:
        return json.dumps({
            "algorithm": self.algorithm, "seed": self.seed, "budget": self.budget, "evals": self.evals,
            "best_vector": list(self.best_vector), "best_raw": self.best_raw, "best_reward": self.best_reward,
            "best_valid": self.best_valid, "restarts": list(self.restarts), "rewards": list(self.rewards),
            "raws": list(self.raws), "wall_clock_s": self.wall_clock_s,
        })

    @staticmethod
    def from_json(text: str) -> "SearchReport":
        p = json.loads(text)
        return SearchReport(p["algorithm"], p["seed"], p["budget"], p["evals"], tuple(p["best_vector"]),
                            p["best_raw"], p["best_reward"], p["best_valid"], tuple(p["restarts"]),
                            tuple(p["rewards"]), tuple(p["raws"]), p["wall_clock_s"])


def build_report(algorithm: str, seed, records: Sequence[EvalRecord], restarts, budget: int, wall_clock_s: float,
                 by_raw: bool = False) -> SearchReport:
    if not records:
        raise ValueError("cannot report on zero evaluations")
    best = None
    for record in records:
        if by_raw and not record.valid:
            continue
        key = record.raw if by_raw else record.reward
        if best is None or key > (best.raw if by_raw else best.reward):
            best = record
    if best is None:
        best = records[0]  # nothing valid: report the first penalty record
    return SearchReport(algorithm, seed, budget, len(records), best.vector, best.raw, best.reward, best.valid,
                        tuple(restarts), tuple(r.reward for r in records), tuple(r.raw for r in records),
                        wall_clock_s)
