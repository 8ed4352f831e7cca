"""Benchmark: batched strategy evaluation (evals/s) on B200, 1..8 GPUs.

Metric (BASELINE.json): strategy evaluations per second, whole job.
Workload: BASELINE config 4 — the 1.6T-parameter MoE on 2048 simulated H100s
(packaged config ``moe_1p6t_h100x2048``), candidates i.i.d. uniform over every
head (baselines.uniform_vector semantics, reference baselines.py:50-54),
generated on each GPU from a per-rank seed. Weak scaling: each rank scores
its own batch of ``--n`` candidates per step (contiguous global index range),
so inputs (16 B/candidate, ~2 GB) dwarf the 126 MB L2 — no flush needed.

One step = the hot path over one batch:
  evaluate (reason + raw throughput per candidate, HBM SoA in/out)
  -> device top-k by raw over distinct vectors (elite of the batch)
  -> (N > 1) one NCCL all-gather of the per-rank top-k (records + count) and
     a device merge.

Also reported: ``e2e`` — the same metric through the public API with HOST
buffers (Evaluator.evaluate_host -> ls_evaluate_host: pinned H2D of the
planes, kernels, D2H of reason + raw, inside the timed region);
``roofline`` of the evaluate kernel (25 algorithmic bytes per candidate ÷
its CUDA-event time vs the measured HBM copy peak); ``cpu_baseline`` — the
C restatement of the reference cost model (oracle/, a "port") on this
host's cores over a bounded sample.

``--impl reference`` times that CPU port alone (the reference is pure
Python with no native path to build).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "strategy evals/sec"
UNIT = "evals/s"
CONFIG = "moe_1p6t_h100x2048"
# per candidate: one packed 8-byte candidate word in, reason u8 + raw f64 out
# (planes: 16 head bytes in instead of 8)
ALGO_BYTES = {"packed": 8 + 1 + 8, "planes": 16 + 1 + 8}
ELITE_K = 8
SEED = 0  # uniform candidate stream seed (seed 0)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=CONFIG)
    ap.add_argument("--candidates-per-gpu", "--n", dest="n", type=int, default=1 << 27,
                    help="candidates per GPU per step (use the long name under torchrun: --n is ambiguous there)")
    ap.add_argument("--e2e-n", type=int, default=1 << 26, help="candidates per GPU per e2e step")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="CPU baseline sample budget")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-search", action="store_true", help="skip the PPO search wall-time line")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle check of the timed batch")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer (end-to-end) measurement")
    ap.add_argument("--diag-no-exchange", action="store_true", help=argparse.SUPPRESS)  # N>1 diagnostics only
    ap.add_argument("--diag-reserve", type=int, default=None, help=argparse.SUPPRESS)
    ap.add_argument("--no-pyref", action="store_true", help="skip timing the reference's Python evaluator")
    ap.add_argument("--pyref-n", type=int, default=1 << 19, help="candidates for the Python reference timing")
    ap.add_argument("--format", default="packed", choices=["packed", "planes"],
                    help="resident candidate format: 8-byte packed words or uint8 SoA planes")
    return ap.parse_args()


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


def stream_planes(desc, start, n, threads=None):
    """Host twin of the GPU arm's candidates: uniform stream positions [start, start + n)
    (oracle/streams.c == generator.py GEN_UNIFORM == the device's ls_generate)."""
    from oracle.cost_model import uniform_planes

    return uniform_planes(desc, SEED, start, n, threads=threads)


# ----------------------------------------------------------------- CPU side


def python_reference_block(args, desc, gpu_reason=None, gpu_thr=None, sample=None):
    """The reference's own Python evaluator (baseline/_ref, decode_strategy +
    simulate per candidate) in Pool(os.cpu_count()) on the first `sample`
    candidates of rank 0's batch; its verdicts are compared with the GPU's."""
    from oracle import pyref

    if not pyref.available():
        return {"unavailable": "the reference package is not installed in baseline/_ref (DESIGN.md section 7)"}
    sample = sample or args.pyref_n
    cfg = ROOT / "paper_2509_00217_b200" / "configs" / f"{args.config}.yaml"
    r = pyref.time_reference(str(cfg), stream_planes(desc, 0, sample))
    blk = {"value": r["value"], "unit": UNIT, "cores": r["procs"], "per_core": r["per_core"], "kind": "reference",
           "sample": f"first {sample} candidates of rank 0's batch; rate measured on that sample (a full batch "
                     f"of {args.n} would take {args.n / r['value']:.0f} s at this rate)",
           "seconds": r["seconds"], "python": r["python"], "cpu": r["cpu"],
           "api": "shardsearch.strategy.decode_strategy + shardsearch.simulator.simulate (env.py:140-158)"}
    if gpu_reason is not None:
        blk["gpu_mismatches"] = int(np.count_nonzero(gpu_reason[:sample] != r["reason"]) + np.count_nonzero(
            gpu_thr[:sample].view(np.uint64) != r["throughput"].view(np.uint64)))
    return blk


def cpu_rate(workload, seconds, sample=1 << 23):
    """Oracle C port over all host cores: evals/s on a bounded prefix of rank 0's batch."""
    from oracle.cost_model import simulate_planes

    threads = os.cpu_count() or 1
    desc = workload.desc()
    planes = stream_planes(desc, 0, sample, threads)
    out = simulate_planes(desc, planes[:, : 1 << 16], threads=threads, fields=("throughput",))  # warm
    out = {"reason": np.empty(sample, np.uint8), "throughput": np.empty(sample, np.float64)}
    done, t0 = 0, time.perf_counter()
    while True:
        simulate_planes(desc, planes, threads=threads, out=out)
        done += sample
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return done / el, threads, done


def run_reference(args, rank):
    """The reference's CPU evaluator (C restatement, all host threads) on the GPU arm's
    exact candidates: rank 0's batch, stream positions [0, n), every step."""
    from paper_2509_00217_b200.config import load_workload
    from oracle.cost_model import simulate_planes

    if rank != 0:
        return
    wl = load_workload(args.config)
    threads = os.cpu_count() or 1
    n = args.n
    desc = wl.desc()
    planes = stream_planes(desc, 0, n, threads)
    out = {"reason": np.empty(n, np.uint8), "throughput": np.empty(n, np.float64)}
    for _ in range(args.warmup):
        simulate_planes(desc, planes, threads=threads, out=out)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        simulate_planes(desc, planes, threads=threads, out=out)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = n * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, 1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"the GPU arm's rank-0 batch ({n} candidates: uniform stream seed {SEED}, "
                                   f"positions [0, {n})) x {args.steps} steps through oracle/shardsim_oracle.c "
                                   f"(C restatement of simulator.py:239-341), {threads} threads"},
        "same_config": True,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_pyref:
        # the reference's own Python evaluator on the same candidates, checked against the port
        pr = python_reference_block(args, desc, out["reason"], out["throughput"])
        if "gpu_mismatches" in pr:
            pr["port_mismatches"] = pr.pop("gpu_mismatches")
        line["python_reference"] = pr
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU side


class Clocks:
    """SM clock + throttle-reason sampler over the timed region: once the
    steps are queued, the host polls NVML until the region's end event
    completes (so even a few-millisecond region gets samples); nvidia-smi at
    its 200 ms floor when NVML is unavailable. No reads between step
    launches: an NVML read there delayed the launches (N=1 step 0.42 ->
    0.48 ms, N=4 0.45 -> 0.72 ms)."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.sampler = None
        self.sm, self.smax, self.reasons = [], None, set()

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.smax = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}

            def sample():
                self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.reasons.update(n for n, bit in bits.items() if r & bit)

            self.sampler = sample
            return
        except Exception:
            self.sampler = None
        try:
            q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def poll_until(self, event):
        """Sample on the calling thread until ``event`` has completed: every
        sample falls inside the region the event closes."""
        if self.sampler is None:
            return
        while not event.query():
            self.sampler()

    def stop(self):
        if self.sampler is not None:
            src = "nvml, polled until the end event completed"
        elif self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            for line in out.strip().splitlines():
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    self.sm.append(float(parts[1]))
                    self.smax = float(parts[2])
                except ValueError:
                    continue
                for name, flag in zip(self.NAMES, parts[5:9]):
                    if flag.lower().startswith("active"):
                        self.reasons.add(name)
            src = "nvidia-smi 200 ms"
        else:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock source"]}
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.smax,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": src}


# reference run_search on moe_1p2t_h100, budget 4000, seed 0, in this image's CPU
# container (BASELINE.md "Search-level reference points")
REF_SEARCH_WALL_S = 105.8
REF_SEARCH_BEST_RAW = 41.90363518619595


def ppo_search_line():
    """Wall time of one full PPO search through the public
    API: ppo.run_search on the flagship 1.2T config, budget 4000, seed 0 — the
    first (cold) call in this process, which pays the context, table build and
    graph capture, and a second (warm) call."""
    from paper_2509_00217_b200.config import load_workload
    from paper_2509_00217_b200.env import SearchEnv
    from paper_2509_00217_b200.knobs import PpoConfig
    from paper_2509_00217_b200.ppo import run_search

    wl = load_workload("moe_1p2t_h100")

    def one(budget):
        t0 = time.perf_counter()
        env = SearchEnv(wl.model, wl.hw, wl.space, wl.context_len, budget, slo_tpot=wl.slo_tpot)
        rep = run_search(env, PpoConfig(budget=budget), 0)
        return time.perf_counter() - t0, rep

    cold, rep0 = one(4000)
    warm = [one(4000) for _ in range(3)]
    wall = statistics.median(w for w, _ in warm)
    rep = warm[0][1]
    return {"workload": "moe_1p2t_h100 PPO run_search, budget 4000, seed 0 (fused policy kernels + CUDA graphs)",
            "wall_s": wall, "wall_s_runs": [w for w, _ in warm], "cold_wall_s": cold,
            "cold": "first run_search of the bench process: its context, tables, buffers and graph captures",
            "evals": rep.evals, "evals_per_s": rep.evals / wall,
            "best_raw": rep.best_raw, "reference_wall_s": REF_SEARCH_WALL_S, "reference_best_raw": REF_SEARCH_BEST_RAW,
            "same_best_as_reference": all(r.best_raw == REF_SEARCH_BEST_RAW for r in [rep0] + [r for _, r in warm])}


# reference per-call costs on this workload family (63-85 us per
# candidate through SearchEnv.step; SA 4000 steps 0.57 s)
REF_STEP_US = (63.0, 85.0)
REF_SA_4000_S = 0.57


def seam_line():
    """Latency of the per-candidate drop-in seam (reference env.py:140-180) and the
    device SA chain (baselines.py:112-145), through the public API."""
    from paper_2509_00217_b200.baselines import SaConfig, simulated_annealing, uniform_vector
    from paper_2509_00217_b200.config import load_workload
    from paper_2509_00217_b200.env import SearchEnv
    from paper_2509_00217_b200.simulator import SimRequest, simulate
    from paper_2509_00217_b200.strategy import decode_strategy

    wl = load_workload("moe_1p2t_h100")
    n = 4000
    env = SearchEnv(wl.model, wl.hw, wl.space, wl.context_len, 3 * n, slo_tpot=wl.slo_tpot)
    rng = np.random.default_rng(0)
    vecs = [uniform_vector(wl.space, rng) for _ in range(n)]
    for v in vecs[:200]:
        env.step(v)
    t0 = time.perf_counter()
    for v in vecs:
        env.step(v)
    step_us = (time.perf_counter() - t0) / n * 1e6
    ev = env.evaluator
    t0 = time.perf_counter()
    for v in vecs:
        ev.evaluate_one(v)
    one_us = (time.perf_counter() - t0) / n * 1e6
    reqs = [SimRequest(wl.model, wl.hw, decode_strategy(v, wl.space), wl.context_len, wl.slo_tpot) for v in vecs]
    simulate(reqs[0])
    t0 = time.perf_counter()
    for r in reqs:
        simulate(r)
    sim_us = (time.perf_counter() - t0) / n * 1e6
    sa_env = SearchEnv(wl.model, wl.hw, wl.space, wl.context_len, 4000, slo_tpot=wl.slo_tpot)
    sa_env.evaluator
    t0 = time.perf_counter()
    rep = simulated_annealing(sa_env, SaConfig(), 4000, 0)
    sa_s = time.perf_counter() - t0
    return {"workload": "moe_1p2t_h100, uniform vectors, one call per candidate",
            "search_env_step_us": step_us, "simulate_us": sim_us, "evaluate_one_us": one_us,
            "reference_step_us": list(REF_STEP_US),
            "sa_4000_wall_s": sa_s, "sa_best_raw": rep.best_raw, "reference_sa_4000_s": REF_SA_4000_S}


def workload_config(args, world):
    return {"workload": f"{args.config}: uniform candidates (baselines.uniform_vector semantics), counter-based "
                        f"stream seed {SEED}, rank r scores positions [r*n, (r+1)*n), n = {args.n} per GPU per step, "
                        + ("packed 8-byte candidate words" if args.format == "packed" else "SoA uint8 planes")
                        + " resident in HBM",
            "format": args.format, "candidates_per_gpu": args.n, "elite_k": ELITE_K,
            "parallelism": f"dp{world} (index-range shards)",
            "l2": f"inputs {ALGO_BYTES[args.format] - 9} B x n per GPU >> 126 MB L2; no flush"}


def parity_block(args, ev, wl, out, elite, local_elite, base, rank, world):
    """Check what the timed steps produced against the CPU oracle (after the timed
    region): every verdict of this rank's batch, the rank's top-k, the merged elite."""
    import torch
    import torch.distributed as dist

    from oracle.parity import batch_parity, merge_topk, rescore_elites, vector_codes

    t0 = time.perf_counter()
    threads = max(1, (os.cpu_count() or 1) // world)
    desc = wl.desc()
    sizes = ev.head_sizes

    def triples(elites):
        if not elites:
            return []
        codes = vector_codes(np.asarray([e.vector for e in elites], dtype=np.uint8).T, sizes)
        return [(float(e.raw), int(e.index), int(c)) for e, c in zip(elites, codes)]

    bp = batch_parity(desc, sizes, SEED, base, out.reason.cpu().numpy(), out.throughput.cpu().numpy(), ELITE_K,
                      threads)
    mine = {"checked": bp["checked"], "reason": bp["reason_mismatches"], "raw": bp["raw_mismatches"],
            "valid": bp["valid"], "topk": bp["oracle_topk"], "local_equal": triples(local_elite) == bp["oracle_topk"]}
    allv = [mine]
    if world > 1:
        allv = [None] * world
        dist.all_gather_object(allv, mine)
    if rank != 0:
        return None
    merged = merge_topk([v["topk"] for v in allv], ELITE_K)
    return {
        "oracle": "oracle/shardsim_oracle.c (C restatement of simulator.py:239-341), candidates regenerated by "
                  "oracle/streams.c",
        "scope": "every candidate of every rank's batch (the verdict buffers of the last timed step), each "
                 "rank's top-k, and the merged elite",
        "candidates_checked": sum(v["checked"] for v in allv),
        "mismatches": sum(v["reason"] + v["raw"] for v in allv),
        "reason_mismatches": sum(v["reason"] for v in allv),
        "raw_mismatches": sum(v["raw"] for v in allv),
        "valid_candidates": sum(v["valid"] for v in allv),
        "rank_topk_equal": all(v["local_equal"] for v in allv),
        "elite_equal": triples(elite) == merged,
        "elite_rescored": len(elite),
        "elite_mismatches": rescore_elites(desc, SEED, elite),
        "seconds": time.perf_counter() - t0,
    }


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2509_00217_b200.config import load_workload
    from paper_2509_00217_b200.dist import ShardedSweep
    from paper_2509_00217_b200.evaluator import BatchResult, Evaluator
    from paper_2509_00217_b200.generator import GEN_UNIFORM

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    wl = load_workload(args.config)
    ev = Evaluator(wl, device=local_rank)
    sizes = ev.head_sizes
    n = args.n
    base = rank * n  # contiguous global index range per rank
    # the uniform stream's positions [base, base + n), generated on the device
    # (the host twin oracle/streams.c regenerates them for the parity block and the reference arm)
    planes = ev.generate(GEN_UNIFORM, n, start=base, seed=SEED)
    cands = planes
    if args.format == "packed":
        cands = ev.pack(planes)  # same candidates, 8 B each
    out = BatchResult(reason=torch.empty(n, dtype=torch.uint8, device=dev),
                      throughput=torch.empty(n, dtype=torch.float64, device=dev))
    # N > 1: each step's elite all-gather + merge runs on a side stream beside the
    # next step's evaluate (which leaves one SM free for it)
    # N > 1: the elite exchange — "nccl" (grouped all-gather on a side stream; measured faster at
    # 20 steps) or "p2p" (the fused launch writes its block into every rank's ring over NVLink,
    # one merge launch per lap of 16 steps)
    xchg = os.environ.get("LS_XCHG", "nccl")
    sweep = ShardedSweep(ev, k=ELITE_K, overlap=world > 1, group_steps=int(os.environ.get("LS_XCHG_GROUP", "4")),
                         transport=xchg if world > 1 else "nccl")
    if args.diag_reserve is not None:
        ev.reserve_sms(args.diag_reserve)
    if args.diag_no_exchange:  # diagnostics: each rank's fused launches alone (no elite exchange)
        sweep = ShardedSweep(ev, k=ELITE_K, overlap=False)
        sweep.world = 1
    stream = torch.cuda.current_stream(dev)

    def step():
        # no events between steps: consecutive fused launches overlap (PDL), and a
        # stream operation between them would serialise them
        _, recs, count = sweep.run(cands, index_base=base, out=out)
        # our kernels per step: the fused evaluate (its last CTA merges the CTA lists);
        # N > 1: + per group of steps one NCCL all-gather and one merge launch (side stream)
        if world == 1:
            return recs, count, 1
        if sweep.transport == "p2p":  # + one merge launch per lap (and one in wait())
            return recs, count, 1 + 1 / sweep._lap
        return recs, count, 1 + 2 / sweep.group_steps

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks = Clocks(local_rank)
    clocks.start()  # NVML init before the barrier: its cost must not skew the ranks' starts
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t_start.record(stream)
    launches = 0.0
    for _ in range(args.steps):
        recs, count, nl = step()
        launches += nl
    sweep.wait()  # the last step's exchange is part of the timed region
    t_end.record(stream)
    clocks.poll_until(t_end)
    torch.cuda.synchronize(dev)
    sweep.check()  # a p2p merge that timed out waiting for a peer fails the run
    sweep.close()  # p2p: unmap the peers' rings (collective)
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    elapsed_ms = t_start.elapsed_time(t_end)
    elite = ev.decode_records(recs, count)
    local_elite = ev.decode_records(*sweep.last_local()) if world > 1 else elite

    # max over ranks of the device time
    if world > 1:
        t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t[0])
    # the fused launches overlap back to back (PDL): the average launch takes one step
    kern_avg = elapsed_ms / args.steps

    parity = None if args.no_parity else parity_block(args, ev, wl, out, elite, local_elite, base, rank, world)
    out_reason_h = out_thr_h = None
    if rank == 0 and not args.no_pyref:
        out_reason_h = out.reason[: args.pyref_n].cpu().numpy()
        out_thr_h = out.throughput[: args.pyref_n].cpu().numpy()

    # end-to-end through the public host API (Evaluator.evaluate_host_compact ->
    # ls_evaluate_host_compact): the step's candidates in pinned HOST memory in the
    # reference's wire format (uint8 index-vector planes), packed into 8-byte words
    # on host threads, H2D, evaluate, D2H of the reason bytes + the valid raws —
    # all inside the timed region; the same from host packed words as a second figure
    e2e_value = e2e_words = None
    nvalid, e2e_check, e2e_n = 0, None, min(args.e2e_n, n)
    if args.no_e2e:
        del planes
    else:
        e2e_n = min(args.e2e_n, n)
        host_planes = torch.empty((len(sizes), e2e_n), dtype=torch.uint8).pin_memory()
        host_planes.copy_(planes[:, :e2e_n].cpu())
        host_words = torch.empty(e2e_n, dtype=torch.int64).pin_memory()
        host_words.copy_(cands[:e2e_n].cpu() if cands.dim() == 1 else ev.pack(planes[:, :e2e_n]).cpu())
        del planes
        reason_h = torch.empty(e2e_n, dtype=torch.uint8).pin_memory().numpy()
        vraw_h = torch.empty(e2e_n, dtype=torch.float64).pin_memory().numpy()
        e2e_steps = max(3, min(args.steps, 10))

        def e2e_run(src):
            ev.evaluate_host_compact(src, reason_h, vraw_h)  # warm: allocates the pipeline buffers
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            nv = 0
            for _ in range(e2e_steps):
                r, v = ev.evaluate_host_compact(src, reason_h, vraw_h)
                nv = len(v)
            el = time.perf_counter() - t0
            if world > 1:
                t = torch.tensor([el], dtype=torch.float64, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                el = float(t[0])
            return world * e2e_n * e2e_steps / el, nv

        e2e_value, nvalid = e2e_run(host_planes.numpy())
        e2e_words, _ = e2e_run(host_words.numpy())
        e2e_check = bool(np.array_equal(reason_h, out.reason[:e2e_n].cpu().numpy()))

    if rank != 0:
        return
    value = world * n * args.steps / (elapsed_ms / 1e3)
    pk, pk_kind = peaks()
    algo_bytes = ALGO_BYTES[args.format]
    achieved_gbs = algo_bytes * n / (kern_avg / 1e3) / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "roofline_traffic.json"
    if tfile.exists():
        try:
            for tj in json.loads(tfile.read_text()).get("entries", []):
                if tj.get("config") == args.config and tj.get("n") == n and tj.get("format") == args.format:
                    traffic = tj.get("bytes_per_launch")
        except Exception:
            traffic = None
    cfg = workload_config(args, world)
    cfg["elite_exchange"] = sweep.transport
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": world * e2e_n * 8,
                "d2h_bytes_per_step": world * (e2e_n + 8 * nvalid), "candidates_per_gpu": e2e_n,
                "input": "pinned host uint8 planes [16, n] (the reference's index vectors), copied as they are",
                "output": "reason byte per candidate + raw of the valid ones (compact host results)",
                "api": "Evaluator.evaluate_host_compact -> ls_evaluate_host_compact(LS_HOST_PLANES)",
                "from_packed_words": e2e_words, "reason_equal_device_batch": e2e_check},
        "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": pk.get("hbm_gbs"), "unit": "GB/s",
                     "frac": achieved_gbs / pk.get("hbm_gbs"), "traffic": traffic,
                     "kernel": "eval_ws_kernel<GEN_WORDS> (fused evaluate + elite, last-CTA merge)"
                               if args.format == "packed" else
                               "eval_ws_kernel (fused evaluate + elite, last-CTA merge)", "algorithmic_bytes_per_candidate": algo_bytes,
                     "kernel_ms_avg": kern_avg, "peak_source": f"{pk_kind} hbm_gbs (MEASURED_PEAKS.json)",
                     "timing": "CUDA events around the K back-to-back fused launches on their stream, / K "
                               "(consecutive launches overlap under programmatic dependent launch)"},
        "gpu_launches": int(round(launches)),
        "clocks": clk,
        "parity": parity,
        "elite_best": {"vector": list(elite[0].vector), "raw": elite[0].raw, "index": elite[0].index} if elite else None,
    }
    if not args.no_search:
        line["search"] = ppo_search_line()
        line["seam"] = seam_line()
    if not args.no_pyref:
        line["python_reference"] = python_reference_block(args, wl.desc(), out_reason_h, out_thr_h)
    if not args.no_cpu:
        rate, cores, done = cpu_rate(wl, args.cpu_seconds)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
                                "sample": f"{done} candidates (a prefix of rank 0's batch, repeated) of {args.config} "
                                          f"through oracle/shardsim_oracle.c (C restatement of the reference cost "
                                          f"model), {cores} threads"}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
