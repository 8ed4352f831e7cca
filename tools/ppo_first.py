"""Where a fresh process spends its first PPO search (cold start)."""
import sys
import time
from pathlib import Path

T0 = time.perf_counter()
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2509_00217_b200.config import load_workload  # noqa: E402
from paper_2509_00217_b200.env import SearchEnv  # noqa: E402
from paper_2509_00217_b200.knobs import PpoConfig  # noqa: E402
from paper_2509_00217_b200.ppo import GpuSearch  # noqa: E402


def mark(what, t=[T0]):
    torch.cuda.synchronize() if torch.cuda.is_initialized() else None
    now = time.perf_counter()
    print(f"{what:32s} {1e3 * (now - t[0]):9.1f} ms", flush=True)
    t[0] = now


mark("imports")
torch.zeros(1, device="cuda")
mark("cuda init")
wl = load_workload("moe_1p2t_h100")
env = SearchEnv(wl.model, wl.hw, wl.space, wl.context_len, 4000, slo_tpot=wl.slo_tpot)
env.evaluator
mark("evaluator (tables)")
s = GpuSearch(env, PpoConfig(budget=4000), 0)
mark("GpuSearch init")
with torch.cuda.stream(s.stream):
    s._start_chunk(800)
    mark("start chunk (params, prime)")
    s._run_round(2)
    mark("first round (capture+replay)")
    for _ in range(10):
        s._run_round(2)
    mark("10 rounds")
