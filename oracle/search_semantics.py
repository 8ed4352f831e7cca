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


def elite_merge(lists, capacity):
    """Merge elite lists [(vector, key, index), ...] with the device merge rule:
    a duplicate vector is replaced only by a better occurrence (key desc,
    index asc), the worst entry is evicted when full. Exact for any order."""
    out = []  # sorted best first
    def better(a, b):
        return a[1] > b[1] or (a[1] == b[1] and a[2] < b[2])
    for lst in lists:
        for rec in lst:
            dup = next((i for i, e in enumerate(out) if e[0] == rec[0]), None)
            if dup is not None:
                if not better(rec, out[dup]):
                    continue
                out.pop(dup)
            elif len(out) >= capacity:
                if not better(rec, out[-1]):
                    continue
                out.pop()
            pos = sum(1 for e in out if better(e, rec))
            out.insert(pos, rec)
    return out
