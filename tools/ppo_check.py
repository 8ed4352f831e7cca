"""GPU PPO search vs the reference's recorded trajectories, plus wall time.

    python tools/ppo_check.py [--no-graphs] [--cases tiny_0,moe_1p2t_h100_0]

For each case prints how many leading eval records equal the reference's
(vector, reward, raw), the restart points, best raw and wall time.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2509_00217_b200.config import load_workload  # noqa: E402
from paper_2509_00217_b200.env import SearchEnv  # noqa: E402
from paper_2509_00217_b200.knobs import PpoConfig  # noqa: E402
from paper_2509_00217_b200.ppo import run_search  # noqa: E402


def common_prefix(a_vec, a_rew, b_vec, b_rew):
    n = min(len(a_vec), len(b_vec))
    for i in range(n):
        if not (np.array_equal(a_vec[i], b_vec[i]) and a_rew[i] == b_rew[i]):
            return i
    return n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--no-graphs", action="store_true")
    ap.add_argument("--cases", default="")
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--engine", default="fused")
    args = ap.parse_args()
    gold = np.load(ROOT / "tests" / "golden" / "ppo_reference.npz")
    meta = json.loads(str(gold["meta"]))
    cases = [c for c in args.cases.split(",") if c] or list(meta)
    for case in cases:
        name, seed = case.rsplit("_", 1)
        m = meta[case]
        wl = load_workload(name)
        for rep in range(args.repeat):
            env = SearchEnv(wl.model, wl.hw, wl.space, wl.context_len, m["evals"], slo_tpot=wl.slo_tpot)
            env.evaluator  # build tables outside the timed search
            t0 = time.perf_counter()
            report = run_search(env, PpoConfig(budget=m["evals"]), int(seed), use_graphs=not args.no_graphs)
            wall = time.perf_counter() - t0
            vecs = np.asarray([r.vector for r in env.eval_log], dtype=np.uint8)
            rews = np.asarray([r.reward for r in env.eval_log])
            k = common_prefix(vecs, rews, gold[case + "_vectors"], gold[case + "_rewards"])
            print(json.dumps({"case": case, "engine": args.engine, "rep": rep, "wall_s": round(wall, 4), "evals": report.evals,
                              "match_prefix": k, "restarts": list(report.restarts), "ref_restarts": m["restarts"],
                              "best_raw": report.best_raw, "ref_best_raw": m["best_raw"],
                              "best_vector": list(report.best_vector), "ref_wall_s": round(m["wall_s"], 2)}),
                  flush=True)


if __name__ == "__main__":
    main()
