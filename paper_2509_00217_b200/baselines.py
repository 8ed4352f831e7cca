"""Search baselines over the GPU evaluator, batched where the reference's
algorithm allows it (reference baselines.py:50-194).

* ``random_walk`` draws the same i.i.d. uniform vectors as the reference
  (numpy PCG64, one ``integers(k)`` per head in order), then scores the whole
  budget in ONE batched pass (``SearchEnv.step_batch``: device evaluate +
  exclusive-max reward scan) — records identical to the reference's.
* ``simulated_annealing`` is a sequential Metropolis chain (each proposal
  depends on the last acceptance) and steps one candidate at a time.
* ``megatron_exhaustive`` scores the coarse grid with Megatron-pinned axes in
  one batched pass and picks the best valid raw, earliest on ties.
* ``exhaustive_search`` / ``random_sweep`` are the device-native callers:
  candidates generated on the GPU (``ls_sweep``), no per-candidate traffic —
  the whole 2.0e9-point 1.2T space in milliseconds.
"""

from __future__ import annotations

import itertools
import math
import time
from dataclasses import dataclass
from typing import Callable

import numpy as np

from .env import BudgetExhausted, EvalRecord, SearchEnv
from .evaluator import REASON_NAMES, Elite, Evaluator
from .generator import GEN_ENUM, GEN_ENUM_ADMISSIBLE, GEN_UNIFORM
from .knobs import SaConfig
from .report import SearchReport, build_report
from .strategy import ActionSpaceSpec, canonical_fused_ops, megatron_fine_dims

__all__ = ["NoValidConfiguration", "SaConfig", "uniform_vector", "mutate_vector", "acceptance_probability",
           "cosine_decay", "random_walk", "simulated_annealing", "sa_draws", "megatron_exhaustive", "SweepReport",
           "exhaustive_search", "random_sweep"]


class NoValidConfiguration(RuntimeError):
    """An exhaustive sweep found nothing that passes the validity gates."""


def cosine_decay(initial: float, progress: float) -> float:
    """Cosine decay from ``initial`` at progress 0 to 0 at 1 (reference ppo.py:164-167)."""
    clamped = min(max(progress, 0.0), 1.0)
    return initial * 0.5 * (1.0 + math.cos(math.pi * clamped))


def uniform_vector(space: ActionSpaceSpec, rng: np.random.Generator) -> tuple[int, ...]:
    return tuple(int(rng.integers(k)) for k in space.head_sizes)


def mutate_vector(vector, space: ActionSpaceSpec, rng: np.random.Generator, moves: int = 1) -> tuple[int, ...]:
    mutable = [i for i, k in enumerate(space.head_sizes) if k > 1]
    if not mutable:
        return tuple(vector)
    picks = rng.choice(len(mutable), size=min(moves, len(mutable)), replace=False)
    out = list(vector)
    for pick in np.atleast_1d(picks):
        coord = mutable[int(pick)]
        drawn = int(rng.integers(space.head_sizes[coord] - 1))
        out[coord] = drawn if drawn < out[coord] else drawn + 1
    return tuple(out)


def acceptance_probability(delta: float, temperature: float) -> float:
    if delta >= 0:
        return 1.0
    if temperature <= 0:
        return 0.0
    return math.exp(delta / temperature)


def random_walk(env: SearchEnv, budget: int, seed: int) -> SearchReport:
    """Budget-many i.i.d. uniform samples, best by reward — one GPU pass."""
    if budget < 1:
        raise ValueError("random walk budget must be >= 1")
    start = time.perf_counter()
    rng = np.random.default_rng(seed)
    vectors = np.asarray([uniform_vector(env.space, rng) for _ in range(budget)], dtype=np.int64)
    first = env.evals_used
    env.step_batch(vectors)
    records = env.eval_log[first:first + budget]
    return build_report("rw", seed, records, (), budget, time.perf_counter() - start)


def simulated_annealing(env: SearchEnv, cfg: SaConfig, budget: int, seed: int) -> SearchReport:
    """Single-chain annealing on the shaped reward, cosine temperature
    (reference baselines.py:112-145).

    The chain runs on the device in ONE kernel (ls_sa_chain): the randomness
    is drawn here first, in the reference's order — it does not depend on the
    chain's accept/reject decisions — so the records equal the reference's.
    An environment whose ``evaluate_raw`` seam was overridden runs the
    sequential host loop through that seam instead."""
    if budget < 1:
        raise ValueError("simulated annealing budget must be >= 1")
    if not env._stock_seam():
        return _simulated_annealing_host(env, cfg, budget, seed)
    start = time.perf_counter()
    rng = np.random.default_rng(seed)
    first = env.evals_used
    steps = min(budget, env.budget_left)
    if steps < 1:
        raise BudgetExhausted(f"budget of {env.budget} evaluations spent")
    init, coords, drawn, u, temperature, moves = sa_draws(env.space, cfg, budget, steps, rng)
    rc = env.reward_cfg
    vecs, raws, rewards, reasons, best = env.evaluator.sa_chain(
        init, coords, drawn, u, temperature, moves, env.best_raw, rc.alpha, rc.beta, rc.invalid_penalty)
    for i in range(steps):
        env._append(EvalRecord(env.evals_used, tuple(int(x) for x in vecs[i]), float(raws[i]), float(rewards[i]),
                               bool(reasons[i] == 0), REASON_NAMES[int(reasons[i])]))
    env.best_raw = best
    if steps < budget:  # the reference's next env.step would raise here
        raise BudgetExhausted(f"budget of {env.budget} evaluations spent")
    records = env.eval_log[first:first + budget]
    return build_report("sa", seed, records, (), budget, time.perf_counter() - start)


def sa_draws(space: ActionSpaceSpec, cfg: SaConfig, budget: int, steps: int, rng: np.random.Generator):
    """The randomness of a simulated-annealing chain of ``steps`` evaluations, drawn
    from ``rng`` exactly as the reference's loop draws it (baselines.py:131-139):
    the first vector (``uniform_vector``), then per proposal ``mutate_vector``'s
    ``choice`` + ``integers(k - 1)`` draws and the acceptance ``random()`` — none
    depends on the chain's decisions. Returns (init, coords, drawn, u,
    temperature, moves) for ``ls_sa_chain``."""
    init = uniform_vector(space, rng)
    mutable = [i for i, k in enumerate(space.head_sizes) if k > 1]
    moves = min(cfg.neighbor_moves, len(mutable)) if mutable else 0
    coords = np.zeros((steps - 1, moves), dtype=np.int32)
    drawn = np.zeros((steps - 1, moves), dtype=np.int32)
    u = np.zeros(steps - 1, dtype=np.float64)
    temperature = np.zeros(steps - 1, dtype=np.float64)
    for step in range(1, steps):  # mutate_vector's and the acceptance test's draws, in order
        temperature[step - 1] = cosine_decay(cfg.t_initial, step / budget)
        if mutable:
            picks = np.atleast_1d(rng.choice(len(mutable), size=moves, replace=False))
            for j, pick in enumerate(picks):
                coord = mutable[int(pick)]
                coords[step - 1, j] = coord
                drawn[step - 1, j] = int(rng.integers(space.head_sizes[coord] - 1))
        u[step - 1] = rng.random()
    return init, coords, drawn, u, temperature, moves


def _simulated_annealing_host(env: SearchEnv, cfg: SaConfig, budget: int, seed: int) -> SearchReport:
    start = time.perf_counter()
    rng = np.random.default_rng(seed)
    first = env.evals_used
    current = uniform_vector(env.space, rng)
    current_reward, _, _ = env.step(current)
    for step in range(1, budget):
        temperature = cosine_decay(cfg.t_initial, step / budget)
        candidate = mutate_vector(current, env.space, rng, cfg.neighbor_moves)
        candidate_reward, _, _ = env.step(candidate)
        if rng.random() < acceptance_probability(candidate_reward - current_reward, temperature):
            current, current_reward = candidate, candidate_reward
    records = env.eval_log[first:first + budget]
    return build_report("sa", seed, records, (), budget, time.perf_counter() - start)


def megatron_exhaustive(env_factory: Callable[[int], SearchEnv], space: ActionSpaceSpec) -> SearchReport:
    """Every coarse degree tuple with Megatron-pinned axes, best valid by raw."""
    grid_size = len(space.tp_domain) * len(space.ep_domain) * len(space.pp_domain) * len(space.batch_domain)
    start = time.perf_counter()
    with env_factory(grid_size) as env:
        if env.space != space:
            raise ValueError("env_factory produced an environment over a different space")
        ops = canonical_fused_ops(env.model)
        dims = dict(zip((op.name for op in ops), megatron_fine_dims(ops)))
        tail = tuple(int(dims[name]) for name in space.op_names)
        grid = itertools.product(*(range(k) for k in space.head_sizes[:4]))
        env.step_batch(np.asarray([c + tail for c in grid], dtype=np.int64))
        records = env.eval_log[-grid_size:]
        if not any(r.valid for r in records):
            raise NoValidConfiguration(f"no valid configuration among {grid_size} megatron-pinned points")
    return build_report("exhaustive", None, records, (), grid_size, time.perf_counter() - start, by_raw=True)


@dataclass(frozen=True)
class SweepReport:
    """Outcome of a device-native sweep: the elite by raw, best first."""

    mode: int
    evaluated: int
    elites: tuple[Elite, ...]
    device_ms: float

    @property
    def best(self) -> Elite | None:
        return self.elites[0] if self.elites else None


def _sweep(ev: Evaluator, mode: int, n: int, start: int, seed: int, k: int, chunk: int) -> SweepReport:
    import torch

    if n <= 0:  # nothing to evaluate: an empty elite
        return SweepReport(mode, 0, (), 0.0)
    recs, counts = [], []
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(torch.cuda.current_stream(ev.device))
    for lo in range(start, start + n, chunk):
        r, c = ev.sweep(mode, min(chunk, start + n - lo), start=lo, seed=seed, k=k)
        recs.append(r)
        counts.append(c)
    if len(recs) > 1:
        r, c = ev.merge_records(torch.cat(recs), torch.cat(counts), k, k)
    else:
        r, c = recs[0], counts[0]
    t1.record(torch.cuda.current_stream(ev.device))
    elites = ev.decode_records(r, c)
    return SweepReport(mode, n, tuple(elites), t0.elapsed_time(t1))


def exhaustive_search(ev: Evaluator, admissible_only: bool = False, k: int = 8,
                      chunk: int = 1 << 34) -> SweepReport:
    """Score the whole action space (or its admissible-axis subspace) on the GPU;
    the elite by raw, earliest itertools.product position on ties."""
    mode = GEN_ENUM_ADMISSIBLE if admissible_only else GEN_ENUM
    return _sweep(ev, mode, ev.stream_size(mode), 0, 0, k, chunk)


def random_sweep(ev: Evaluator, n: int, seed: int = 0, k: int = 8, chunk: int = 1 << 34) -> SweepReport:
    """n i.i.d. uniform candidates generated on the GPU (counter-based stream)."""
    return _sweep(ev, GEN_UNIFORM, n, 0, seed, k, chunk)
