"""Hyper-parameter records of the searches that drive the evaluator.

Same fields, defaults and validation as the reference's ``PpoConfig``
(pkg/src/shardsearch/ppo.py:42-84) and ``SaConfig`` (baselines.py:35-47), so
YAML files written for the reference load unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["PpoConfig", "SaConfig"]


@dataclass(frozen=True)
class PpoConfig:
    budget: int = 4000
    chunks: int = 5
    n_steps: int = 2
    epochs_per_update: int = 2
    lr_initial: float = 1e-3
    clip_eps: float = 0.2
    value_coef: float = 0.5
    entropy_coef: float = 0.01
    tau: float = 0.95
    history_len: int = 3
    width: int = 256
    ffn_width: int = 256

    def __post_init__(self) -> None:
        for name in ("budget", "chunks", "n_steps", "epochs_per_update", "lr_initial", "clip_eps", "tau",
                     "history_len", "width", "ffn_width"):
            value = getattr(self, name)
            if value <= 0:
                raise ValueError(f"ppo.{name} must be positive, got {value}")
        for name in ("value_coef", "entropy_coef"):
            value = getattr(self, name)
            if value < 0:
                raise ValueError(f"ppo.{name} must be non-negative, got {value}")
        if self.budget % self.chunks:
            raise ValueError(f"ppo.chunks ({self.chunks}) must divide ppo.budget ({self.budget})")


@dataclass(frozen=True)
class SaConfig:
    t_initial: float = 100.0
    neighbor_moves: int = 1

    def __post_init__(self) -> None:
        if self.t_initial <= 0:
            raise ValueError(f"sa.t_initial must be positive, got {self.t_initial}")
        if self.neighbor_moves < 1:
            raise ValueError(f"sa.neighbor_moves must be >= 1, got {self.neighbor_moves}")
