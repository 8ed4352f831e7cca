"""Short fused-PPO search for kernel launch lists under ncu:

    ncu --metrics gpu__time_duration.sum --csv --log-file out.csv python tools/ppo_profile.py --budget 100
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2509_00217_b200.config import load_workload  # noqa: E402
from paper_2509_00217_b200.env import SearchEnv  # noqa: E402
from paper_2509_00217_b200.knobs import PpoConfig  # noqa: E402
from paper_2509_00217_b200.ppo import run_search  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--budget", type=int, default=100)
    ap.add_argument("--config", default="moe_1p2t_h100")
    ap.add_argument("--no-graphs", action="store_true")
    ap.add_argument("--engine", default="fused")
    ap.add_argument("--chunks", type=int, default=1)
    args = ap.parse_args()
    wl = load_workload(args.config)
    env = SearchEnv(wl.model, wl.hw, wl.space, wl.context_len, args.budget, slo_tpot=wl.slo_tpot)
    env.evaluator
    stats = {}
    t0 = time.perf_counter()
    rep = run_search(env, PpoConfig(budget=args.budget, chunks=args.chunks), 0, use_graphs=not args.no_graphs, stats=stats)
    print(f"budget {args.budget} wall {time.perf_counter() - t0:.4f}s best {rep.best_raw} {stats}")


if __name__ == "__main__":
    main()
