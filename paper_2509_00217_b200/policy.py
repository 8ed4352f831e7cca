"""Elite-conditioned policy in PyTorch (reference policy.py), for the GPU search.

Same architecture, parameter names, shapes and initialisation as the
reference's numpy ``PolicyNetwork`` (policy.py:213-499): one post-norm
self-attention block over the ``history_len`` elite rows, mean-pooled, one
masked categorical head per sub-action (inadmissible axes at logit -1e30,
policy.py:36, :120-146) and a value head. Gradients come from autograd
instead of the reference's hand-written backward. The host ``EliteBuffer`` and
``build_observation`` keep the reference's exact semantics; the GPU search
(ppo.py) runs the same rules on device tensors.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import Iterable, Mapping, Sequence

import numpy as np
import torch

from .strategy import ActionSpaceSpec, AxisChoice, FusedOpDescriptor

__all__ = ["MASKED_LOGIT", "NumericsError", "Elite", "EliteBuffer", "build_observation", "head_masks", "TorchPolicy",
           "sample_actions", "policy_shapes", "policy_layout",
           "CheckpointError", "save_checkpoint", "load_checkpoint"]

MASKED_LOGIT = -1e30
_LN_EPS = 1e-5


class NumericsError(FloatingPointError):
    """A forward pass or update produced non-finite values."""


@dataclass(frozen=True)
class Elite:
    vector: tuple[int, ...]
    reward: float


class EliteBuffer:
    """Top-``capacity`` valid strategies by reward (reference policy.py:57-102)."""

    def __init__(self, capacity: int = 3) -> None:
        if capacity < 1:
            raise ValueError("elite buffer capacity must be >= 1")
        self.capacity = int(capacity)
        self._entries: list[Elite] = []

    def __len__(self) -> int:
        return len(self._entries)

    @property
    def entries(self) -> tuple[Elite, ...]:
        return tuple(self._entries)

    @property
    def min_reward(self) -> float:
        return float("-inf") if len(self._entries) < self.capacity else self._entries[-1].reward

    def offer(self, vector: Sequence[int], reward: float) -> bool:
        vec = tuple(int(v) for v in vector)
        if any(e.vector == vec for e in self._entries):
            return False
        if len(self._entries) >= self.capacity:
            if reward <= self._entries[-1].reward:
                return False
            self._entries.pop()
        self._entries.append(Elite(vec, float(reward)))
        self._entries.sort(key=lambda e: -e.reward)  # stable: older first among equals
        return True


def build_observation(buf: EliteBuffer, space: ActionSpaceSpec) -> np.ndarray:
    """capacity x vector_length rows, best first, each index / max(k-1, 1), zero padded."""
    denom = np.maximum(np.asarray(space.head_sizes, dtype=np.float64) - 1.0, 1.0)
    obs = np.zeros((buf.capacity, space.vector_length), dtype=np.float64)
    for row, elite in enumerate(buf.entries):
        obs[row] = np.asarray(elite.vector, dtype=np.float64) / denom
    return obs


def head_masks(space: ActionSpaceSpec, ops: Iterable[FusedOpDescriptor]) -> tuple[np.ndarray, ...]:
    """Allowed choices per head: coarse heads all; axis heads UNSHARDED + admitted axes."""
    by_name = {op.name: op for op in ops}
    masks = [np.ones(len(d), dtype=bool) for d in (space.tp_domain, space.ep_domain, space.pp_domain,
                                                     space.batch_domain)]
    for name in space.op_names:
        if name not in by_name:
            raise ValueError(f"action space controls unknown operator {name!r}")
        op = by_name[name]
        masks.append(np.array([True, op.admits(AxisChoice.DIM0), op.admits(AxisChoice.DIM1)]))
    return tuple(masks)


def policy_shapes(a: int, d: int, f: int, hk: int) -> list[tuple[str, tuple[int, ...]]]:
    """Packed parameter tensors in arena order (include/ls_eval.h LS_PSEG_*)."""
    return [("embed_w", (a, d)), ("embed_b", (d,)), ("wqkv", (d, 3 * d)), ("bqkv", (3 * d,)), ("wo", (d, d)),
            ("bo", (d,)), ("ln1_g", (d,)), ("ln1_b", (d,)), ("ffn_w1", (d, f)), ("ffn_b1", (f,)),
            ("ffn_w2", (f, d)), ("ffn_b2", (d,)), ("ln2_g", (d,)), ("ln2_b", (d,)), ("head_w", (d, hk)),
            ("head_b", (hk,)), ("value_w1", (d, d)), ("value_b1", (d,)), ("value_w2", (d, 1)), ("value_b2", (1,))]


def policy_layout(shapes) -> tuple[list[int], int]:
    """Element offsets of each tensor in the arena, 32-element aligned."""
    offsets, off = [], 0
    for _, shape in shapes:
        offsets.append(off)
        off = (off + int(np.prod(shape)) + 31) & ~31
    return offsets, off


class TorchPolicy(torch.nn.Module):
    """The reference network with packed parameters.

    Storage is packed for few, larger kernels: q/k/v share one [d, 3d]
    matrix and all heads one [d, heads*Kmax] matrix whose padding columns
    never receive gradient (their logits are overwritten by the mask). The
    reference's per-tensor names ("attn.wq", "head.3.w", ...) are views into
    the packed storage, so ``state``/``load_state`` and checkpoints are
    interchangeable with the reference's.
    """

    def __init__(self, space: ActionSpaceSpec, ops: Iterable[FusedOpDescriptor], *, history_len: int = 3,
                 width: int = 256, ffn_width: int = 256, device=None, dtype=torch.float64) -> None:
        super().__init__()
        if history_len < 1 or width < 1 or ffn_width < 1:
            raise ValueError("history_len, width and ffn_width must be >= 1")
        self.space = space
        self.history_len, self.width, self.ffn_width = int(history_len), int(width), int(ffn_width)
        self.head_sizes = space.head_sizes
        self.num_heads = nh = len(self.head_sizes)
        self.kmax = kmax = max(self.head_sizes)
        masks = head_masks(space, ops)
        blocked = np.ones((nh, kmax), dtype=bool)  # inadmissible or padding: logit MASKED_LOGIT, probability 0
        for i, m in enumerate(masks):
            blocked[i, : len(m)] = ~m
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self.register_buffer("blocked", torch.tensor(blocked, device=dev))
        self.register_buffer("sizes", torch.tensor(self.head_sizes, dtype=torch.int64, device=dev))
        denom = np.maximum(np.asarray(self.head_sizes, dtype=np.float64) - 1.0, 1.0)
        self.register_buffer("obs_denom", torch.tensor(denom, dtype=dtype, device=dev))
        d, f, a = self.width, self.ffn_width, space.vector_length
        shapes = policy_shapes(a, d, f, nh * kmax)
        offsets, total = policy_layout(shapes)
        self.offsets = offsets
        # one float64 arena in the C ABI's layout (ls_policy_layout_of); every
        # parameter is a leaf over its slice, so the fused kernels and autograd
        # see the same storage
        self.flat = torch.zeros(total, dtype=dtype, device=dev)
        for (attr, shape), off in zip(shapes, offsets):
            n = int(np.prod(shape))
            setattr(self, attr, torch.nn.Parameter(self.flat[off:off + n].view(shape)))
        with torch.no_grad():  # plain aliases: no autograd node may be created outside the search's stream
            self._views = self._name_views()
        self.names = list(self._views)

    def _name_views(self) -> dict:
        d, nh, kmax = self.width, self.num_heads, self.kmax
        hw, hb = self.head_w.view(d, nh, kmax), self.head_b.view(nh, kmax)
        v = {"embed.w": self.embed_w, "embed.b": self.embed_b,
             "attn.wq": self.wqkv[:, :d], "attn.bq": self.bqkv[:d], "attn.wk": self.wqkv[:, d:2 * d],
             "attn.bk": self.bqkv[d:2 * d], "attn.wv": self.wqkv[:, 2 * d:], "attn.bv": self.bqkv[2 * d:],
             "attn.wo": self.wo, "attn.bo": self.bo, "ln1.g": self.ln1_g, "ln1.b": self.ln1_b,
             "ffn.w1": self.ffn_w1, "ffn.b1": self.ffn_b1, "ffn.w2": self.ffn_w2, "ffn.b2": self.ffn_b2,
             "ln2.g": self.ln2_g, "ln2.b": self.ln2_b}
        for i, k in enumerate(self.head_sizes):
            v[f"head.{i}.w"] = hw[:, i, :k]
            v[f"head.{i}.b"] = hb[i, :k]
        v.update({"value.w1": self.value_w1, "value.b1": self.value_b1, "value.w2": self.value_w2,
                  "value.b2": self.value_b2})
        return v

    def p(self, name: str) -> torch.Tensor:
        """The reference-named parameter tensor (a view into packed storage)."""
        return self._views[name]

    # -- parameters ---------------------------------------------------------

    def init_state(self, rng: np.random.Generator) -> dict[str, np.ndarray]:
        """Reference initialisation (policy.py:245-281) from the shared numpy rng, in
        its draw order: fan-in uniform matrices, zero biases, unit LN gains, zero
        head and value-output layers (an untrained policy samples uniformly)."""
        d, f, a = self.width, self.ffn_width, self.space.vector_length

        def fan_in(rows, cols):
            limit = 1.0 / np.sqrt(float(rows))
            return rng.uniform(-limit, limit, size=(rows, cols))

        out = {"embed.w": fan_in(a, d), "embed.b": np.zeros(d), "attn.wq": fan_in(d, d), "attn.bq": np.zeros(d),
               "attn.wk": fan_in(d, d), "attn.bk": np.zeros(d), "attn.wv": fan_in(d, d), "attn.bv": np.zeros(d),
               "attn.wo": fan_in(d, d), "attn.bo": np.zeros(d), "ln1.g": np.ones(d), "ln1.b": np.zeros(d),
               "ffn.w1": fan_in(d, f), "ffn.b1": np.zeros(f), "ffn.w2": fan_in(f, d), "ffn.b2": np.zeros(d),
               "ln2.g": np.ones(d), "ln2.b": np.zeros(d)}
        for i, k in enumerate(self.head_sizes):
            out[f"head.{i}.w"] = np.zeros((d, k))
            out[f"head.{i}.b"] = np.zeros(k)
        out.update({"value.w1": fan_in(d, d), "value.b1": np.zeros(d), "value.w2": np.zeros((d, 1)),
                    "value.b2": np.zeros(1)})
        return out

    def reset_parameters(self, rng: np.random.Generator) -> None:
        self.load_state(self.init_state(rng))

    def state(self) -> dict[str, np.ndarray]:
        return {n: self.p(n).detach().cpu().numpy().copy() for n in self.names}

    def load_state(self, tensors: Mapping[str, np.ndarray]) -> None:
        """Replace all parameters; names and shapes must match exactly (padding stays 0)."""
        if set(tensors) != set(self.names):
            raise ValueError(f"state mismatch: missing={sorted(set(self.names) - set(tensors))} "
                             f"extra={sorted(set(tensors) - set(self.names))}")
        for n in self.names:
            if tuple(np.shape(tensors[n])) != tuple(self.p(n).shape):
                raise ValueError(f"shape mismatch for {n}: expected {tuple(self.p(n).shape)}, "
                                 f"got {tuple(np.shape(tensors[n]))}")
        with torch.no_grad():
            self.head_w.zero_()
            self.head_b.zero_()
            for n in self.names:
                self.p(n).copy_(torch.as_tensor(np.asarray(tensors[n], dtype=np.float64)))

    @property
    def num_parameters(self) -> int:
        return sum(self.p(n).numel() for n in self.names)

    def check_finite(self) -> None:
        for n in self.names:
            if not bool(torch.isfinite(self.p(n)).all()):
                raise NumericsError(f"non-finite values in {n}")

    # -- forward ------------------------------------------------------------

    @staticmethod
    def _ln(x, g, b):
        mean = x.mean(dim=-1, keepdim=True)
        c = x - mean
        var = (c * c).mean(dim=-1, keepdim=True)
        inv_std = 1.0 / torch.sqrt(var + _LN_EPS)
        return g * (c * inv_std) + b

    def observation(self, elite_vec: torch.Tensor, elite_reward: torch.Tensor) -> torch.Tensor:
        """build_observation on device tensors: rows best first, empty slots (reward -inf) zero."""
        full = torch.isfinite(elite_reward).unsqueeze(-1)
        return torch.where(full, elite_vec.to(self.obs_denom.dtype) / self.obs_denom, 0.0)

    def forward(self, obs: torch.Tensor):
        """obs [..., T, A] -> (log_probs [..., heads, Kmax], probs, value [...])."""
        d = self.width
        emb = obs @ self.embed_w + self.embed_b
        qkv = emb @ self.wqkv + self.bqkv
        q, k, v = qkv[..., :d], qkv[..., d:2 * d], qkv[..., 2 * d:]
        scores = (q @ k.transpose(-1, -2)) * (1.0 / float(np.sqrt(float(d))))
        weights = torch.softmax(scores, dim=-1)
        h1 = self._ln(emb + ((weights @ v) @ self.wo + self.bo), self.ln1_g, self.ln1_b)
        ffn = torch.relu(h1 @ self.ffn_w1 + self.ffn_b1) @ self.ffn_w2 + self.ffn_b2
        h2 = self._ln(h1 + ffn, self.ln2_g, self.ln2_b)
        pooled = h2.mean(dim=-2)
        raw = (pooled @ self.head_w + self.head_b).unflatten(-1, (self.num_heads, self.kmax))
        logits = torch.where(self.blocked, MASKED_LOGIT, raw)
        shifted = logits - logits.amax(dim=-1, keepdim=True)
        ex = torch.exp(shifted)
        total = ex.sum(dim=-1, keepdim=True)
        log_probs = shifted - torch.log(total)
        probs = ex / total
        value = (torch.relu(pooled @ self.value_w1 + self.value_b1) @ self.value_w2 + self.value_b2).squeeze(-1)
        return log_probs, probs, value

    @staticmethod
    def entropy(log_probs: torch.Tensor, probs: torch.Tensor) -> torch.Tensor:
        """Total head entropy (blocked entries have probability 0 and contribute 0)."""
        return -(probs * log_probs).sum(dim=(-1, -2))

    def confidence(self, probs: torch.Tensor) -> torch.Tensor:
        """Max probability per head (reference policy.py:502-504)."""
        return probs.amax(dim=-1)


def sample_actions(probs: torch.Tensor, u: torch.Tensor, size_cap: torch.Tensor) -> torch.Tensor:
    """Inverse-CDF draw per head (reference sample_categorical, policy.py:205-210):
    idx = searchsorted(cumsum(p), u * cumsum[-1], right), clamped to k - 1.
    probs [heads, Kmax] (zero past each head's size), u [heads] uniforms."""
    cdf = probs.cumsum(dim=-1)
    draw = u.unsqueeze(-1) * cdf[..., -1:]
    return torch.minimum(torch.searchsorted(cdf, draw, right=True).squeeze(-1), size_cap)


# ---------------------------------------------------------------------------
# Checkpoints: the reference's "SSPL" v1 little-endian layout (policy.py:507-566)

CHECKPOINT_MAGIC = b"SSPL"
CHECKPOINT_VERSION = 1


class CheckpointError(ValueError):
    """Checkpoint bytes do not match the documented layout."""


def save_checkpoint(path: str, tensors: Mapping[str, np.ndarray]) -> None:
    chunks = [CHECKPOINT_MAGIC, struct.pack("<II", CHECKPOINT_VERSION, len(tensors))]
    for name, tensor in tensors.items():
        raw = name.encode("utf-8")
        arr = np.ascontiguousarray(tensor, dtype=np.float64)
        chunks += [struct.pack("<H", len(raw)), raw, struct.pack("<B", arr.ndim), struct.pack(f"<{arr.ndim}I", *arr.shape),
                   arr.tobytes(order="C")]
    with open(path, "wb") as sink:
        sink.write(b"".join(chunks))


def load_checkpoint(path: str) -> dict[str, np.ndarray]:
    with open(path, "rb") as source:
        data = source.read()
    try:
        return _parse_checkpoint(data)
    except (struct.error, UnicodeDecodeError) as exc:
        raise CheckpointError(f"malformed checkpoint: {exc}") from exc


def _parse_checkpoint(data: bytes) -> dict[str, np.ndarray]:
    if data[:4] != CHECKPOINT_MAGIC:
        raise CheckpointError("bad magic: not a policy checkpoint")
    version, count = struct.unpack_from("<II", data, 4)
    if version != CHECKPOINT_VERSION:
        raise CheckpointError(f"unsupported checkpoint version {version}")
    off, out = 12, {}
    for _ in range(count):
        (nl,) = struct.unpack_from("<H", data, off)
        off += 2
        name = data[off:off + nl].decode("utf-8")
        off += nl
        (ndim,) = struct.unpack_from("<B", data, off)
        off += 1
        shape = struct.unpack_from(f"<{ndim}I", data, off)
        off += 4 * ndim
        size = int(np.prod(shape, dtype=np.int64)) if ndim else 1
        end = off + 8 * size
        if end > len(data):
            raise CheckpointError(f"truncated tensor data for {name!r}")
        out[name] = np.frombuffer(data[off:end], dtype="<f8").reshape(shape).astype(np.float64)
        off = end
    if off != len(data):
        raise CheckpointError("trailing bytes after final tensor")
    return out
