"""Where the GPU PPO search first leaves the reference's Llama-3-70B trajectory."""
import json, sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2509_00217_b200.config import load_workload
from paper_2509_00217_b200.env import SearchEnv
from paper_2509_00217_b200.knobs import PpoConfig
from paper_2509_00217_b200.ppo import run_search

G = np.load(ROOT / "tests/golden/ppo_reference_llama70b.npz")
M = json.loads(str(G["meta"]))
wl = load_workload("llama3_70b_h100x64")
for seed in [int(s) for s in sys.argv[1:]] or [0, 4, 9]:
    case = f"llama3_70b_h100x64_{seed}"
    for engine in ("fused", "torch"):
        env = SearchEnv(wl.model, wl.hw, wl.space, wl.context_len, 4000, slo_tpot=wl.slo_tpot)
        rep = run_search(env, PpoConfig(budget=4000), seed, engine=engine)
        v = np.asarray([r.vector for r in env.eval_log], dtype=np.uint8)
        ref = G[case + "_vectors"]
        bad = np.nonzero((v != ref).any(1))[0]
        print(seed, engine, "restarts ours", list(rep.restarts)[:12], "ref", M[case]["restarts"][:12])
        print(seed, engine, "mismatch records", bad[:20].tolist(), "count", len(bad))
        for i in bad[:3]:
            print("   rec", i, "ours", v[i].tolist(), "ref", ref[i].tolist(), "reward ref", G[case + "_rewards"][i])
