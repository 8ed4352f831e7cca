"""Golden PPO searches on the BASELINE configs beyond the 1.2T flagship, made
by running the REFERENCE in this container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_ppo_configs.py

* ppo_reference_llama70b.npz — BASELINE.json config 2 (Llama-3-70B dense on 64
  simulated H100s, ``configs/llama3_70b_h100x64.yaml``): the reference's
  ``run_search`` (ppo.py:466-528), budget 4000, seeds 0-9 — every eval
  record (vectors, rewards, raws), the restarts, the winner and the
  reference's own wall time per seed on this container's cores (one process
  per seed).
"""

from __future__ import annotations

import json
import time
from multiprocessing import Pool
from pathlib import Path

import numpy as np

from shardsearch.config import load_config
from shardsearch.env import SearchEnv
from shardsearch.ppo import PpoConfig, run_search

OUT = Path(__file__).resolve().parent
CFG = OUT.parent.parent / "paper_2509_00217_b200" / "configs" / "llama3_70b_h100x64.yaml"
BUDGET = 4000
SEEDS = tuple(range(10))


def one(seed):
    cfg = load_config(CFG)
    env = SearchEnv(cfg.model, cfg.hardware, cfg.space, cfg.simulation.context_len, BUDGET,
                    slo_tpot=cfg.simulation.slo_tpot)
    t0 = time.perf_counter()
    rep = run_search(env, PpoConfig(budget=BUDGET), seed)
    wall = time.perf_counter() - t0
    arrays = {"vectors": np.asarray([r.vector for r in env.eval_log], dtype=np.uint8),
              "rewards": np.asarray([r.reward for r in env.eval_log]),
              "raws": np.asarray([r.raw for r in env.eval_log])}
    meta = {"best_vector": list(rep.best_vector), "best_raw": rep.best_raw, "best_reward": rep.best_reward,
            "restarts": list(rep.restarts), "evals": rep.evals, "wall_s": wall}
    return seed, arrays, meta


def main():
    payload, meta = {}, {}
    with Pool(min(len(SEEDS), 8)) as pool:
        for seed, arrays, m in pool.imap_unordered(one, SEEDS):
            key = f"llama3_70b_h100x64_{seed}"
            for k, v in arrays.items():
                payload[f"{key}_{k}"] = v
            meta[key] = m
            print(key, m["best_raw"], f"{m['wall_s']:.1f}s", flush=True)
    np.savez_compressed(OUT / "ppo_reference_llama70b.npz", meta=np.asarray(json.dumps(meta)), **payload)


if __name__ == "__main__":
    main()
