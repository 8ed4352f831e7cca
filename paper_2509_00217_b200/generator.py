"""Candidate streams: the on-device generators of ``ls_sweep`` / ``ls_generate``.

Three streams map a stream position ``i`` to an index vector:

* ``GEN_UNIFORM`` — i.i.d. uniform over every head, the random-walk proposal
  ``uniform_vector`` (reference baselines.py:50-54), as a counter-based
  function of (seed, i): two splitmix64 draws pick a uniform coarse rank
  (tp, ep, pp, batch) and a uniform axis rank.
* ``GEN_ENUM`` — the i-th vector of ``itertools.product`` over the head
  domains, head 0 most significant: the order of the reference's exhaustive
  sweeps (``megatron_exhaustive`` baselines.py:172-179, the acceptance oracle
  test_acceptance.py:86), so "earliest index wins ties" carries over.
* ``GEN_ENUM_ADMISSIBLE`` — the same over admissible axes only
  (``FusedOpDescriptor.admits``, strategy.py:57-59).

This module is the host twin used to verify the device streams and to decode
stream positions back into vectors; it is not on the evaluation path.
"""

from __future__ import annotations

import numpy as np

from .strategy import AxisChoice, canonical_fused_ops

__all__ = ["GEN_UNIFORM", "GEN_ENUM", "GEN_ENUM_ADMISSIBLE", "axis_radices", "stream_size", "stream_vectors"]

GEN_UNIFORM = 1
GEN_ENUM = 2
GEN_ENUM_ADMISSIBLE = 3

_M64 = (1 << 64) - 1


def axis_radices(model, space, mode: int) -> list[list[int]]:
    """Per axis head (heads 4..), the axis values the stream draws from, in order."""
    ops = {op.name: op for op in canonical_fused_ops(model)}
    out = []
    for name in space.op_names:
        op = ops.get(name)
        if mode == GEN_ENUM_ADMISSIBLE and op is not None:
            out.append([a for a in (0, 1, 2) if op.admits(AxisChoice(a))])
        else:
            out.append([0, 1, 2])
    return out


def stream_size(model, space, mode: int) -> int:
    n = 1
    for k in space.head_sizes[:4]:
        n *= k
    for vals in axis_radices(model, space, mode):
        n *= len(vals)
    return n


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = (x + np.uint64(0x9E3779B97F4A7C15)).astype(np.uint64)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def _mulhi64_vec(a: np.ndarray, b: int) -> np.ndarray:
    """High 64 bits of a * b (the device's __umul64hi) for uint64 arrays a."""
    mask = np.uint64(0xFFFFFFFF)
    a_lo, a_hi = a & mask, a >> np.uint64(32)
    b_lo, b_hi = np.uint64(b & 0xFFFFFFFF), np.uint64(b >> 32)
    with np.errstate(over="ignore"):
        lo_lo = a_lo * b_lo
        lo_hi = a_lo * b_hi
        hi_lo = a_hi * b_lo
        hi_hi = a_hi * b_hi
        cross = (lo_lo >> np.uint64(32)) + (hi_lo & mask) + (lo_hi & mask)
        return hi_hi + (hi_lo >> np.uint64(32)) + (lo_hi >> np.uint64(32)) + (cross >> np.uint64(32))


def stream_vectors(model, space, mode: int, start: int, n: int, seed: int = 0) -> np.ndarray:
    """[n, A] index vectors of stream positions [start, start + n)."""
    sizes = list(space.head_sizes[:4])
    axes = axis_radices(model, space, mode)
    coarse_size = int(np.prod(sizes))
    axis_size = int(np.prod([len(v) for v in axes])) if axes else 1
    idx = np.arange(start, start + n, dtype=np.uint64)
    if mode == GEN_UNIFORM:
        s = np.uint64(seed & _M64)
        with np.errstate(over="ignore"):
            r1 = _splitmix64(s ^ (np.uint64(2) * idx))
            r2 = _splitmix64(s ^ (np.uint64(2) * idx + np.uint64(1)))
        coarse = _mulhi64_vec(r1, coarse_size)
        axis = _mulhi64_vec(r2, axis_size)
    else:
        coarse = idx // np.uint64(axis_size)
        axis = idx % np.uint64(axis_size)
    out = np.zeros((n, 4 + len(axes)), dtype=np.int64)
    rem = coarse.copy()
    for h in (3, 2, 1, 0):
        out[:, h] = (rem % np.uint64(sizes[h])).astype(np.int64)
        rem //= np.uint64(sizes[h])
    rem = axis.copy()
    for j in range(len(axes) - 1, -1, -1):
        r = len(axes[j])
        digit = (rem % np.uint64(r)).astype(np.int64)
        out[:, 4 + j] = np.asarray(axes[j])[digit]
        rem //= np.uint64(r)
    return out
