"""Chunked PPO strategy search on the GPU (reference pkg/src/shardsearch/ppo.py).

Same algorithm and protocol as the reference's ``run_search`` (:466-528):
one-step episodes, the elite buffer (capacity ``history_len``) as the
observation, ``n_steps`` samples per rollout, ``epochs_per_update`` clipped-PPO
epochs with Adam under a cosine learning rate (:164-167, :297-327), an
early exit once every head is confident (:356-358), fresh parameters and
optimizer per chunk with unspent allowance rolled forward (:489-518), and
exactly ``budget`` evaluations.

What is B200-native:

* Every sample, update and confidence check runs on the device. The env
  step — strategy scoring, Eq.-1 reward against the running best, eval-log
  append and the elite-buffer offer — is one fused kernel (``ls_env_step``),
  so nothing per-sample crosses PCIe; the host reads one status word per
  round (the early-exit / numerics flag).
* One PPO round (sample, step, sample, step, two update epochs, confidence)
  is captured once into a CUDA graph and replayed; per-round inputs (the
  learning rate, the uniform draws) are indexed on the device from a
  chunk-local counter.
* The uniform stream is the reference's: one numpy PCG64 generator drives
  parameter initialisation and one ``random()`` per head per sample, in the
  reference's order. Each chunk pre-draws its allowance's worth of uniforms and
  rewinds the generator to the position the reference would have reached, so
  later chunks see the same draws as the reference's restarts. The sampled
  trajectory therefore equals the reference's for as long as the float64
  probabilities agree — they differ only in BLAS rounding order.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _native
from .baselines import cosine_decay
from .env import EvalRecord, SearchEnv
from .evaluator import REASON_NAMES
from .knobs import PpoConfig
from .policy import NumericsError, TorchPolicy
from .report import SearchReport, build_report
from .strategy import DecodingError, canonical_fused_ops

__all__ = ["PpoConfig", "ChunkExit", "ChunkOutcome", "GpuSearch", "run_search"]

_CONFIDENT, _NONFINITE = 1, 2


class ChunkExit(str, Enum):
    EXHAUSTED = "exhausted"
    EARLY_EXIT = "early_exit"


@dataclass(frozen=True)
class ChunkOutcome:
    exit: ChunkExit
    evals_used: int


class GpuSearch:
    """Device-resident state of one PPO search over ``env``."""

    # rounds run eagerly (per round size) before one is captured into a CUDA graph
    capture_warmup = 0

    def __init__(self, env: SearchEnv, cfg: PpoConfig, seed: int, *, use_graphs: bool = True) -> None:
        if env.budget_left < cfg.budget:
            raise ValueError(f"environment has {env.budget_left} evals left, need {cfg.budget}")
        self.env, self.cfg, self.seed = env, cfg, seed
        ev = env.evaluator
        self.ev = ev
        dev = self.device = ev.device
        self.rng = np.random.default_rng(seed)
        self.policy = TorchPolicy(env.space, canonical_fused_ops(env.model), history_len=cfg.history_len,
                                  width=cfg.width, ffn_width=cfg.ffn_width, device=dev)
        self.H = H = env.space.vector_length
        T, B = cfg.history_len, cfg.budget
        f64 = dict(dtype=torch.float64, device=dev)
        i64 = dict(dtype=torch.int64, device=dev)
        # environment / elite / log state (ls_search_state)
        self.best = torch.tensor([env.best_raw], **f64)
        self.elite_vec = torch.zeros((T, H), **i64)
        self.elite_reward = torch.full((T,), float("-inf"), **f64)
        self.log_pos = torch.zeros(1, **i64)
        self.log_vec = torch.zeros((B, H), dtype=torch.uint8, device=dev)
        self.log_raw = torch.zeros(B, **f64)
        self.log_reward = torch.zeros(B, **f64)
        self.log_reason = torch.zeros(B, dtype=torch.uint8, device=dev)
        rc = env.reward_cfg
        self._state = _native.SearchState(self.best.data_ptr(), self.elite_vec.data_ptr(), self.elite_reward.data_ptr(),
                                          T, self.log_pos.data_ptr(), B, self.log_vec.data_ptr(),
                                          self.log_raw.data_ptr(), self.log_reward.data_ptr(),
                                          self.log_reason.data_ptr(), rc.alpha, rc.beta, rc.invalid_penalty)
        # chunk-local inputs, indexed on the device by the chunk's sample counter
        self.spent = torch.zeros(1, **i64)
        self.uniforms = torch.zeros(B * H, **f64)
        self.lr_table = torch.zeros(B, **f64)
        self.lr = torch.zeros((), **f64)
        self.head_offsets = torch.arange(H, **i64)
        self.size_cap = self.policy.sizes - 1
        # rollout batch
        n = cfg.n_steps
        self.b_obs = torch.zeros((n, T, H), **f64)
        self.b_act = torch.zeros((n, H), **i64)
        self.b_logp = torch.zeros(n, **f64)
        self.b_value = torch.zeros(n, **f64)
        self.b_reward = torch.zeros(n, **f64)
        self.action = torch.zeros(H, **i64)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.status_host = torch.zeros(1, dtype=torch.int32).pin_memory()
        self.use_graphs = use_graphs
        self.stream = torch.cuda.Stream(device=dev)
        self._graphs: dict[int, torch.cuda.CUDAGraph] = {}
        self._eager_rounds: dict[int, int] = {}
        self._lib = _native.lib(require_gpu=True)
        self.rounds = 0
        self.round_events: list | None = None  # set to [] to record (start, end) CUDA events per round
        self._init_engine()

    def _init_engine(self) -> None:
        """Buffers and the ls_ppo_plan of the fused-kernel engine (ls_policy.cu)."""
        cfg, pol, dev = self.cfg, self.policy, self.device
        dims = _native.PolicyDims(self.H, cfg.width, cfg.ffn_width, cfg.history_len, pol.num_heads, pol.kmax,
                                  cfg.n_steps)
        layout = _native.PolicyLayout()
        _native.check(self._lib.ls_policy_layout_of(ctypes.byref(dims), ctypes.byref(layout)))
        if list(layout.off) != pol.offsets or layout.total != pol.flat.numel():
            raise RuntimeError("policy arena layout disagrees with ls_policy_layout_of")
        ws = int(self._lib.ls_ppo_workspace_bytes(ctypes.byref(dims)))
        if ws == 0:
            raise _native.NativeError(4, "policy dims unsupported by the fused PPO kernels")
        self.adam_m = torch.zeros_like(pol.flat)
        self.adam_v = torch.zeros_like(pol.flat)
        self.adam_step = torch.zeros(1, dtype=torch.int64, device=dev)
        self.workspace = torch.zeros(ws, dtype=torch.uint8, device=dev)
        self.blocked_u8 = pol.blocked.to(torch.uint8).contiguous()
        self.head_size_i32 = pol.sizes.to(torch.int32).contiguous()
        ptr = lambda t: t.data_ptr()  # noqa: E731
        self.plan = _native.PpoPlan(
            dims, ptr(pol.flat), ptr(self.adam_m), ptr(self.adam_v), None, ptr(self.workspace), ptr(self.blocked_u8),
            ptr(self.head_size_i32), ptr(pol.obs_denom), self._state, ptr(self.uniforms), ptr(self.lr_table),
            ptr(self.spent), ptr(self.adam_step), ptr(self.status), ptr(self.b_obs), ptr(self.b_act),
            ptr(self.b_logp), ptr(self.b_value), ptr(self.b_reward), cfg.tau, cfg.clip_eps, cfg.value_coef,
            cfg.entropy_coef, 0.9, 0.999, 1e-8, cfg.epochs_per_update)

    def _stream_ptr(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    # -- one round (graph-capturable: no host syncs, static shapes) ----------

    def _engine_round(self, n: int) -> None:
        """n samples (each: sample, env step, elite offer), the updates and the
        confidence check: ls_ppo_round, a fixed sequence of fused kernels."""
        _native.check(self._lib.ls_ppo_round(self.ev._ctx, ctypes.byref(self.plan), n, self._stream_ptr()))

    def _engine_start_chunk(self) -> None:
        """Fresh optimizer state; sample slot 0 <- forward of the current observation."""
        self.adam_m.zero_()
        self.adam_v.zero_()
        self.adam_step.zero_()
        _native.check(self._lib.ls_ppo_prime(self.ev._ctx, ctypes.byref(self.plan), self._stream_ptr()))

    def _run_round(self, n: int) -> int:
        """One round (replayed graph once warm); returns the status word."""
        g = self._graphs.get(n)
        ev = None
        if self.round_events is not None:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
        if g is not None:
            g.replay()
        elif self.use_graphs and self._eager_rounds.get(n, 0) >= self.capture_warmup:
            # the fused kernels need no warm-up: captured at once, then replayed
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.stream):
                self._engine_round(n)
            self._graphs[n] = g
            g.replay()
        else:
            self._engine_round(n)
            self._eager_rounds[n] = self._eager_rounds.get(n, 0) + 1
        self.rounds += 1
        if ev is not None:
            ev[1].record()
            self.round_events.append(ev)
        self.status_host.copy_(self.status, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        return int(self.status_host[0])

    # -- chunk protocol (reference run_chunk :330-359, run_search :466-528) ---

    def _start_chunk(self, allowance: int) -> None:
        self.policy.reset_parameters(self.rng)  # the reference's PolicyNetwork(rng=rng)
        self._rng_mark = self.rng.bit_generator.state
        draws = self.rng.random(allowance * self.H)
        self.uniforms[: draws.size].copy_(torch.from_numpy(draws))
        lrs = np.array([cosine_decay(self.cfg.lr_initial, s / allowance) for s in range(allowance)])
        self.lr_table[:allowance].copy_(torch.from_numpy(lrs))
        self.spent.zero_()
        self._engine_start_chunk()

    def _end_chunk(self, spent: int) -> None:
        self.rng.bit_generator.state = self._rng_mark
        self.rng.random(spent * self.H)  # leave the generator where the reference's would be

    def run_chunk(self, allowance: int) -> ChunkOutcome:
        if allowance < 1:
            raise ValueError("chunk allowance must be >= 1")
        self._start_chunk(allowance)
        spent = 0
        outcome = ChunkExit.EXHAUSTED
        while spent < allowance:
            n = min(self.cfg.n_steps, allowance - spent)
            status = self._run_round(n)
            spent += n
            if status & _NONFINITE:
                raise NumericsError("non-finite loss or parameters in a PPO update")
            if status & _CONFIDENT:
                outcome = ChunkExit.EARLY_EXIT
                break
        self._end_chunk(spent)
        return ChunkOutcome(outcome, spent)

    def run(self) -> tuple[list[int], int]:
        cfg = self.cfg
        restarts, evals_done, carry = [], 0, 0
        with torch.cuda.stream(self.stream):
            for base in [cfg.budget // cfg.chunks] * cfg.chunks:
                allowance = base + carry
                restarts.append(evals_done)
                out = self.run_chunk(allowance)
                evals_done += out.evals_used
                carry = allowance - out.evals_used
            while carry > 0:  # early exit in the last chunk: extra restarts spend the rest
                allowance = carry
                restarts.append(evals_done)
                out = self.run_chunk(allowance)
                evals_done += out.evals_used
                carry = allowance - out.evals_used
        self.stream.synchronize()
        return restarts, evals_done

    def records(self, first_index: int, count: int) -> list[EvalRecord]:
        vec = self.log_vec[:count].cpu().numpy()
        raw = self.log_raw[:count].cpu().numpy()
        rew = self.log_reward[:count].cpu().numpy()
        why = self.log_reason[:count].cpu().numpy()
        if (why == 255).any():
            raise DecodingError(f"sampled vector {vec[int(np.argmax(why == 255))].tolist()} failed to decode")
        return [EvalRecord(first_index + i, tuple(int(x) for x in vec[i]), float(raw[i]), float(rew[i]),
                           bool(why[i] == 0), REASON_NAMES[int(why[i])]) for i in range(count)]


def run_search(env: SearchEnv, cfg: PpoConfig, seed: int, *, use_graphs: bool = True,
               stats: dict | None = None, search_cls=None) -> SearchReport:
    """Full chunked-restart PPO search on the GPU; consumes exactly ``cfg.budget`` evals.

    Appends the eval records to ``env`` (and its NDJSON sink) when the search
    ends and leaves ``env.best_raw`` where the reference's would be.
    """
    start = time.perf_counter()
    search = (search_cls or GpuSearch)(env, cfg, seed, use_graphs=use_graphs)
    if stats is not None:
        search.round_events = []
    restarts, evals_done = search.run()
    if stats is not None:
        gpu = [a.elapsed_time(b) for a, b in search.round_events]
        stats.update(rounds=search.rounds, round_gpu_ms_total=sum(gpu),
                     round_gpu_us_median=1e3 * sorted(gpu)[len(gpu) // 2] if gpu else 0.0)
    first = env.evals_used
    records = search.records(first, evals_done)
    for r in records:
        env._append(r)
    env.best_raw = float(search.best.item())
    return build_report("ppo", seed, records, restarts, cfg.budget, time.perf_counter() - start)
