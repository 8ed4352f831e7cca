"""Golden outputs of the reference's search baselines (baselines.py:92-194),
made by running the REFERENCE in this container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_search.py

random_walk and simulated_annealing draw from numpy's PCG64 with the given
seed, so a batched re-implementation that consumes the same random stream and
the same evaluator must reproduce every record; megatron_exhaustive is
deterministic.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from shardsearch.baselines import SaConfig, megatron_exhaustive, random_walk, simulated_annealing
from shardsearch.config import load_config, packaged_config_path
from shardsearch.env import SearchEnv

OUT = Path(__file__).resolve().parent


def env_for(cfg, budget):
    return SearchEnv(cfg.model, cfg.hardware, cfg.space, cfg.simulation.context_len, budget,
                     slo_tpot=cfg.simulation.slo_tpot)


def main():
    payload = {}
    meta = {}
    for name, budget, seeds in (("moe_1p2t_h100", 4000, (0, 3)), ("tiny", 1000, (0, 1))):
        cfg = load_config(packaged_config_path(name))
        for seed in seeds:
            for algo in ("rw", "sa"):
                env = env_for(cfg, budget)
                rep = random_walk(env, budget, seed) if algo == "rw" else simulated_annealing(env, SaConfig(), budget, seed)
                key = f"{name}_{algo}_{seed}"
                payload[key + "_vectors"] = np.asarray([r.vector for r in env.eval_log], dtype=np.uint8)
                payload[key + "_rewards"] = np.asarray([r.reward for r in env.eval_log])
                payload[key + "_raws"] = np.asarray([r.raw for r in env.eval_log])
                meta[key] = {"best_vector": list(rep.best_vector), "best_raw": rep.best_raw,
                             "best_reward": rep.best_reward, "evals": rep.evals}
                print(key, rep.best_raw, rep.best_reward)
        rep = megatron_exhaustive(lambda b: env_for(cfg, b), cfg.space)
        meta[f"{name}_exhaustive"] = {"best_vector": list(rep.best_vector), "best_raw": rep.best_raw,
                                      "best_reward": rep.best_reward, "evals": rep.evals}
        print(name, "exhaustive", rep.best_raw, rep.best_vector)
    np.savez_compressed(OUT / "baselines_reference.npz", meta=np.asarray(json.dumps(meta)), **payload)


if __name__ == "__main__":
    main()
