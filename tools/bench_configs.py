"""Per-config measurements of every BASELINE.json config on one B200.

    python tools/bench_configs.py [--out gpurun_out/configs.json] [--seeds 10] [--quick]

One JSON object per line, each timed with CUDA events on the evaluator's
stream after a warm-up call (the fused step of bench.py on each config):

* ``uniform``: resident packed batch of 10^8 i.i.d. uniform candidates
  (baselines.uniform_vector semantics), fused evaluate + elite top-8 with
  per-candidate verdicts to HBM — configs 2, 3 (SLO 0.05 s and 0.02 s), 4 and
  the 1.2T flagship;
* ``enumerate``: on-device enumeration streams (0 B of candidate input):
  config 1's exhaustive 10,392,624-point Llama-3-8B space and every config's
  admissible-axis subspace, with the winner;
* ``sizes``: config 5, the synthetic sweep 10^4 .. 10^9 on 1.6T@2048 through
  the resident packed fused step (the 10^9 batch is 8 GB of words plus 9 GB
  of verdicts);
* ``search``: config 2, the 4000-round PPO ``run_search`` on Llama-3-70B for
  seeds 0..S-1: wall time and winner, next to the reference's own run
  (tests/golden/ppo_reference_llama70b.npz, made on the CPU by
  tests/golden/make_golden_ppo_configs.py).
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_00217_b200.baselines import exhaustive_search  # noqa: E402
from paper_2509_00217_b200.config import load_workload  # noqa: E402
from paper_2509_00217_b200.env import SearchEnv  # noqa: E402
from paper_2509_00217_b200.evaluator import Evaluator  # noqa: E402
from paper_2509_00217_b200.knobs import PpoConfig  # noqa: E402
from paper_2509_00217_b200.ppo import run_search  # noqa: E402


def emit(fh, obj):
    line = json.dumps(obj)
    print(line, flush=True)
    fh.write(line + "\n")
    fh.flush()


def uniform_words(ev, n, seed=0):
    gen = torch.Generator(device=ev.device)
    gen.manual_seed(seed)
    planes = torch.empty((ev.vector_length, n), dtype=torch.uint8, device=ev.device)
    for h, k in enumerate(ev.head_sizes):
        planes[h] = torch.randint(0, k, (n,), generator=gen, device=ev.device, dtype=torch.uint8)
    words = ev.pack(planes)
    del planes
    return words


def time_fused(ev, words, reps):
    n = words.shape[0]
    out = ev._alloc(n, ("throughput",))
    stream = torch.cuda.current_stream(ev.device)
    ev.evaluate_packed_topk(words, k=8, out=out)  # warm-up
    torch.cuda.synchronize(ev.device)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        _, recs, count = ev.evaluate_packed_topk(words, k=8, out=out)
    b.record(stream)
    torch.cuda.synchronize(ev.device)
    ms = a.elapsed_time(b) / reps
    best = ev.decode_records(recs, count)
    valid = float((out.reason == 0).float().mean().item())
    return ms, best[0] if best else None, valid


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "configs.jsonl"))
    ap.add_argument("--seeds", type=int, default=10)
    ap.add_argument("--quick", action="store_true", help="smaller batches, 2 seeds")
    args = ap.parse_args()
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    fh = open(args.out, "w")
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    n_uni = 10**7 if args.quick else 10**8
    seeds = 2 if args.quick else args.seeds

    workloads = [
        ("llama3_8b_h100x8", "config 1", None),
        ("llama3_70b_h100x64", "config 2", None),
        ("dsv3_style_h100x256", "config 3 (SLO 0.05 s)", None),
        ("dsv3_style_h100x256", "config 3 (SLO 0.02 s)", 0.02),
        ("moe_1p6t_h100x2048", "config 4", None),
        ("moe_1p2t_h100", "flagship 1.2T", None),
    ]
    for name, label, slo in workloads:
        wl = load_workload(name)
        if slo is not None:
            wl = dataclasses.replace(wl, slo_tpot=slo)
        with Evaluator(wl, device=0) as ev:
            words = uniform_words(ev, n_uni)
            ms, best, valid = time_fused(ev, words, 5)
            del words
            emit(fh, {"kind": "uniform", "config": label, "workload": name, "slo_tpot": wl.slo_tpot, "n": n_uni,
                      "ms": ms, "evals_per_s": n_uni / ms * 1e3, "valid_frac": valid,
                      "best": None if best is None else {"vector": list(best.vector), "raw": best.raw,
                                                         "index": best.index}})
            for admissible in ((False, True) if name == "llama3_8b_h100x8" else (True,)):
                exhaustive_search(ev, admissible_only=admissible)  # warm-up
                rep = exhaustive_search(ev, admissible_only=admissible)
                b = rep.best
                emit(fh, {"kind": "enumerate", "config": label, "workload": name, "slo_tpot": wl.slo_tpot,
                          "space": "admissible-axis" if admissible else "full", "n": rep.evaluated, "ms": rep.device_ms,
                          "evals_per_s": rep.evaluated / rep.device_ms * 1e3,
                          "best": None if b is None else {"vector": list(b.vector), "raw": b.raw, "index": b.index}})
                if admissible:  # the fp32 fast mode of the same sweep (raw within 1e-5, reasons exact)
                    ev.set_precision("fp32")
                    exhaustive_search(ev, admissible_only=True)
                    rep = exhaustive_search(ev, admissible_only=True)
                    ev.set_precision("fp64")
                    b = rep.best
                    emit(fh, {"kind": "enumerate_fp32", "config": label, "workload": name, "slo_tpot": wl.slo_tpot,
                              "space": "admissible-axis", "n": rep.evaluated, "ms": rep.device_ms,
                              "evals_per_s": rep.evaluated / rep.device_ms * 1e3,
                              "best": None if b is None else {"vector": list(b.vector), "raw": b.raw,
                                                               "index": b.index}})
        torch.cuda.empty_cache()

    wl = load_workload("moe_1p6t_h100x2048")
    with Evaluator(wl, device=0) as ev:
        top = 10**8 if args.quick else 10**9
        n = 10**4
        while n <= top:
            words = uniform_words(ev, n)
            reps = 200 if n <= 10**6 else (20 if n <= 10**8 else 3)
            ms, best, _ = time_fused(ev, words, reps)
            del words
            emit(fh, {"kind": "sizes", "config": "config 5", "workload": "moe_1p6t_h100x2048", "n": n, "ms": ms,
                      "evals_per_s": n / ms * 1e3, "reps": reps,
                      "l2": "resident" if n * 17 < 126e6 else "streamed from HBM"})
            if n <= 10**6:  # one call on its own (launch + table staging + merges): the latency floor
                words = uniform_words(ev, n)
                out = ev._alloc(n, ("throughput",))
                ev.evaluate_packed_topk(words, k=8, out=out)
                lat = []
                for _ in range(50):
                    torch.cuda.synchronize(ev.device)
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    ev.evaluate_packed_topk(words, k=8, out=out)
                    b.record()
                    torch.cuda.synchronize(ev.device)
                    lat.append(a.elapsed_time(b))
                emit(fh, {"kind": "latency", "config": "config 5", "workload": "moe_1p6t_h100x2048", "n": n,
                          "ms_median": float(np.median(lat)), "note": "one fused call, synchronised, events around it"})
                del words, out
            torch.cuda.empty_cache()
            n *= 10

    gold_path = ROOT / "tests" / "golden" / "ppo_reference_llama70b.npz"
    gold = json.loads(str(np.load(gold_path)["meta"])) if gold_path.exists() else {}
    wl = load_workload("llama3_70b_h100x64")
    for seed in range(seeds):
        env = SearchEnv(wl.model, wl.hw, wl.space, wl.context_len, 4000, slo_tpot=wl.slo_tpot)
        t0 = time.perf_counter()
        rep = run_search(env, PpoConfig(budget=4000), seed)
        wall = time.perf_counter() - t0
        ref = gold.get(f"llama3_70b_h100x64_{seed}")
        emit(fh, {"kind": "search", "config": "config 2", "workload": "llama3_70b_h100x64", "seed": seed,
                  "budget": 4000, "wall_s": wall, "best_raw": rep.best_raw, "best_vector": list(rep.best_vector),
                  "reference_wall_s": None if ref is None else ref["wall_s"],
                  "reference_best_raw": None if ref is None else ref["best_raw"],
                  "same_best_raw_as_reference": None if ref is None else rep.best_raw == ref["best_raw"],
                  "same_best_vector_as_reference": None if ref is None else (
                      list(rep.best_vector) == ref["best_vector"])})
    fh.close()


if __name__ == "__main__":
    main()
