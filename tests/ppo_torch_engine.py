"""The autograd / cuBLAS PPO engine — a TEST REFERENCE for the fused kernels.

Round 1 shipped two PPO engines in the product (``engine="torch"`` beside
the fused kernels); the product now runs the fused float64 kernels only
(paper_2509_00217_b200/ppo.py, csrc/ls_policy.cu). This module keeps the
autograd engine for the tests: the same ``GpuSearch`` protocol (chunked
restarts, PCG64 draws, the device env step), with the policy forward in
torch ops, the loss of the reference's loss_and_grads (ppo.py:203-294)
differentiated by autograd and torch's Adam. Its float64 rounding follows
cuBLAS, so it tracks the reference for the opening stretch only.
"""

from __future__ import annotations

import ctypes

import torch

from paper_2509_00217_b200 import _native
from paper_2509_00217_b200.knobs import PpoConfig
from paper_2509_00217_b200.policy import TorchPolicy, sample_actions
from paper_2509_00217_b200.ppo import _CONFIDENT, _NONFINITE, GpuSearch, run_search

__all__ = ["ppo_loss", "TorchEngineSearch", "run_search_torch"]


def ppo_loss(pol: TorchPolicy, obs, act, logp_old, value_old, reward, cfg: PpoConfig) -> torch.Tensor:
    """Clipped-surrogate PPO loss over a rollout batch (reference loss_and_grads,
    ppo.py:203-294): per sample -min(rho*A, clip(rho)*A) + value_coef*(v - r)^2
    - entropy_coef*H, averaged; A = reward - value_old. Its autograd gradient is
    the reference's hand-written one (the unclipped branch carries the
    gradient on ties, the clamped branch is constant outside the band)."""
    n = obs.shape[0]
    log_probs, probs, value = pol(obs)
    logp_new = log_probs.gather(2, act.unsqueeze(2)).sum(dim=(1, 2))
    entropy = pol.entropy(log_probs, probs)
    ratio = torch.exp(logp_new - logp_old)
    advantage = reward - value_old
    unclipped = ratio * advantage
    clamped = ratio.clamp(1.0 - cfg.clip_eps, 1.0 + cfg.clip_eps) * advantage
    surrogate = torch.where(unclipped <= clamped, unclipped, clamped)
    err = value - reward
    return (-surrogate / n).sum() + (cfg.value_coef * err * err / n).sum() - cfg.entropy_coef * (entropy / n).sum()



class TorchEngineSearch(GpuSearch):
    """GpuSearch with the autograd engine (rounds warm up eagerly, then graph capture)."""

    capture_warmup = 3

    def _init_engine(self) -> None:
        self.opt = torch.optim.Adam(self.policy.parameters(), lr=self.lr, betas=(0.9, 0.999), eps=1e-8,
                                    capturable=True, foreach=True)

    def _engine_start_chunk(self) -> None:  # fresh optimizer
        for st in self.opt.state.values():
            for v in st.values():
                v.zero_()

    def _engine_round(self, n: int) -> None:
        self._round(n)

    def _sample_and_step(self, j: int) -> None:
        pol, H = self.policy, self.H
        obs = pol.observation(self.elite_vec, self.elite_reward)
        with torch.no_grad():
            log_probs, probs, value = pol(obs)
            u = self.uniforms.index_select(0, self.spent * H + self.head_offsets)
            act = sample_actions(probs, u, self.size_cap)
            self.b_obs[j].copy_(obs)
            self.b_act[j].copy_(act)
            self.action.copy_(act)
            self.b_logp[j:j + 1].copy_(log_probs.gather(1, act.unsqueeze(1)).sum().reshape(1))
            self.b_value[j:j + 1].copy_(value.reshape(1))
        _native.check(self._lib.ls_env_step(self.ev._ctx, ctypes.byref(self._state), ctypes.c_void_p(self.action.data_ptr()),
                                            ctypes.c_void_p(self.b_reward.data_ptr() + 8 * j),
                                            ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)))
        self.spent.add_(1)

    def _update(self, n: int) -> torch.Tensor:
        cfg, pol = self.cfg, self.policy
        obs, act = self.b_obs[:n], self.b_act[:n]
        logp_old, value_old, reward = self.b_logp[:n], self.b_value[:n], self.b_reward[:n]
        bad = ~(torch.isfinite(reward) & torch.isfinite(value_old) & torch.isfinite(logp_old)).all()
        for _ in range(cfg.epochs_per_update):
            loss = ppo_loss(pol, obs, act, logp_old, value_old, reward, cfg)
            loss.backward()
            self.opt.step()
            self.opt.zero_grad(set_to_none=False)
            bad = bad | ~torch.isfinite(loss)
        norms = torch._foreach_norm(list(pol.parameters()), float("inf"))
        return bad | ~torch.isfinite(torch.stack(norms)).all()

    def _round(self, n: int) -> None:
        self.lr.copy_(self.lr_table.index_select(0, self.spent).reshape(()))
        for j in range(n):
            self._sample_and_step(j)
        bad = self._update(n)
        with torch.no_grad():
            _, probs, _ = self.policy(self.policy.observation(self.elite_vec, self.elite_reward))
            confident = (self.policy.confidence(probs) >= self.cfg.tau).all()
        self.status.copy_((confident.int() * _CONFIDENT + bad.int() * _NONFINITE).reshape(1))



def run_search_torch(env, cfg: PpoConfig, seed: int, *, use_graphs: bool = True):
    return run_search(env, cfg, seed, use_graphs=use_graphs, search_cls=TorchEngineSearch)
