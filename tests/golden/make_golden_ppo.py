"""Golden outputs of the reference's policy and PPO search (policy.py, ppo.py),
made by running the REFERENCE in this container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_ppo.py

* policy_reference.npz — a small PolicyNetwork (width 16, ffn 8) built from a
  seeded generator: its parameters, forward outputs on two observations, the
  exact gradients of loss_and_grads on a two-sample rollout, and the
  parameters after one ppo_update (2 epochs of Adam).
* ppo_reference.npz — full run_search eval logs (vectors, rewards, raws,
  restarts) for tiny (budget 1000, seeds 0, 1) and the 1.2T flagship
  (budget 4000, seeds 0, 3).
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

from shardsearch.config import load_config, packaged_config_path
from shardsearch.env import SearchEnv
from shardsearch.policy import EliteBuffer, PolicyNetwork, build_observation
from shardsearch.ppo import Adam, PpoConfig, RolloutBatch, RolloutSample, loss_and_grads, ppo_update, run_search
from shardsearch.strategy import canonical_fused_ops

OUT = Path(__file__).resolve().parent


def env_for(cfg, budget):
    return SearchEnv(cfg.model, cfg.hardware, cfg.space, cfg.simulation.context_len, budget,
                     slo_tpot=cfg.simulation.slo_tpot)


def policy_fixture():
    cfg = load_config(packaged_config_path("moe_1p2t_h100"))
    ops = canonical_fused_ops(cfg.model)
    rng = np.random.default_rng(11)
    pol = PolicyNetwork(cfg.space, ops, rng=rng, history_len=3, width=16, ffn_width=8)
    out = {"param." + k: v.copy() for k, v in pol.params.items()}
    buf = EliteBuffer(3)
    obs0 = build_observation(buf, cfg.space)
    buf.offer(tuple(int(rng.integers(k)) for k in cfg.space.head_sizes), 12.5)
    buf.offer(tuple(int(rng.integers(k)) for k in cfg.space.head_sizes), 30.25)
    obs1 = build_observation(buf, cfg.space)
    samples = []
    for i, obs in enumerate((obs0, obs1)):
        o = pol.forward(obs)
        out[f"obs{i}"] = obs
        out[f"logits{i}"] = np.stack([np.pad(h, (0, 11 - h.size), constant_values=np.nan) for h in o.logits])
        out[f"probs{i}"] = np.stack([np.pad(p, (0, 11 - p.size), constant_values=np.nan) for p in o.probs])
        out[f"value{i}"] = np.asarray(o.value)
        action, logprob, entropy = pol.sample(o, rng)
        out[f"action{i}"] = np.asarray(action)
        out[f"logprob{i}"] = np.asarray(logprob)
        out[f"entropy{i}"] = np.asarray(entropy)
        samples.append(RolloutSample(obs=obs, action=action, logprob_old=logprob, reward=[3.0, -10.0][i],
                                     value_old=o.value))
    batch = RolloutBatch(tuple(samples))
    pcfg = PpoConfig()
    report, grads = loss_and_grads(pol, batch, pcfg)
    out.update({"grad." + k: v for k, v in grads.items()})
    out["loss"] = np.asarray([report.policy_loss, report.value_loss, report.entropy, report.total_loss])
    ppo_update(pol, batch, pcfg, 1e-3, Adam(pol.params))
    out.update({"updated." + k: v.copy() for k, v in pol.params.items()})
    np.savez_compressed(OUT / "policy_reference.npz", **out)


def ppo_fixture():
    payload, meta = {}, {}
    for name, budget, seeds in (("tiny", 1000, (0, 1)), ("moe_1p2t_h100", 4000, (0, 3))):
        cfg = load_config(packaged_config_path(name))
        for seed in seeds:
            env = env_for(cfg, budget)
            t0 = time.perf_counter()
            rep = run_search(env, PpoConfig(budget=budget), seed)
            key = f"{name}_{seed}"
            payload[key + "_vectors"] = np.asarray([r.vector for r in env.eval_log], dtype=np.uint8)
            payload[key + "_rewards"] = np.asarray([r.reward for r in env.eval_log])
            payload[key + "_raws"] = np.asarray([r.raw for r in env.eval_log])
            meta[key] = {"best_vector": list(rep.best_vector), "best_raw": rep.best_raw,
                         "best_reward": rep.best_reward, "restarts": list(rep.restarts), "evals": rep.evals,
                         "wall_s": time.perf_counter() - t0}
            print(key, meta[key], flush=True)
    np.savez_compressed(OUT / "ppo_reference.npz", meta=np.asarray(json.dumps(meta)), **payload)


if __name__ == "__main__":
    which = sys.argv[1:] or ["policy", "ppo"]
    if "policy" in which:
        policy_fixture()
    if "ppo" in which:
        ppo_fixture()
