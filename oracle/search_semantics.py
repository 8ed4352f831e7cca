"""Sequential reference semantics of reward shaping and the elite buffer.

Pure-Python restatement of
    SearchEnv.step reward/best update   pkg/src/shardsearch/env.py:152-180
    EliteBuffer.offer                   pkg/src/shardsearch/policy.py:86-102
    build_report winner selection       pkg/src/shardsearch/ppo.py:424-463
used to check the batched device scan / top-k. Small inputs only.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

from __future__ import annotations


def rewards_sequential(reason, throughput, b0=0.0, alpha=1.0, beta=1.0, penalty=-10.0):
    """Per-candidate reward and the final best_raw, one step at a time."""
    best = b0
    rewards = []
    for r, thr in zip(reason, throughput):
        valid = int(r) == 0
        if valid:
            raw = float(thr)
            rewards.append(alpha * raw + beta * (raw - best))
            if raw > best:
                best = raw
        else:
            rewards.append(penalty)
    return rewards, best


def elite_offers(vectors, rewards, valid, capacity):
    """Offer every valid (vector, reward) in order to an initially empty buffer.

    Returns the final entries best first as (vector, reward, first_index).
    """
    entries = []  # (vector, reward, index)
    for i, (vec, rew, ok) in enumerate(zip(vectors, rewards, valid)):
        if not ok:
            continue
        vec = tuple(int(v) for v in vec)
        if any(e[0] == vec for e in entries):
            continue
        if len(entries) >= capacity:
            if rew <= entries[-1][1]:
                continue
            entries.pop()
        entries.append((vec, float(rew), i))
        entries.sort(key=lambda e: -e[1])  # stable: older first among equals
    return entries


def best_by_raw(reason, throughput):
    """Index of the best valid record by raw, earliest on ties (by_raw=True)."""
    best = None
    for i, (r, thr) in enumerate(zip(reason, throughput)):
        if int(r) != 0:
            continue
        if best is None or thr > throughput[best]:
            best = i
    return best
