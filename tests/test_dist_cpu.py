"""Multi-rank host logic on CPU (gloo, world size 2): index-range sharding,
the cross-rank exclusive running best of SearchEnv.step (env.py:159-164,
:178-179) and the exactness of merging per-rank elites (policy.py:86-102,
SURVEY.md §8e / A.5) — the protocol bench.py runs over NCCL on B200s."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from golden_io import load_search
from oracle.search_semantics import elite_merge, elite_offers, rewards_sequential
from paper_2509_00217_b200.dist import exclusive_prefix_best, shard_range


def test_shard_range_partitions():
    for n in (0, 1, 7, 1000, 10**9 + 7):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl, meta, data = load_search(name)
        r = meta["reward"]
        reasons = np.where(data["valid"], 0, 2).astype(np.uint8)
        raws = data["raws"]
        n = len(raws)
        lo, hi = shard_range(n, rank, world)
        # this rank's best valid raw, then its exclusive baseline
        local = raws[lo:hi][data["valid"][lo:hi]]
        local_best = float(local.max()) if local.size else float("-inf")
        base, best_all = exclusive_prefix_best(local_best, meta["b0"])
        rewards, _ = rewards_sequential(reasons[lo:hi], raws[lo:hi], base, r["alpha"], r["beta"],
                                        r["invalid_penalty"])
        # per-rank elites over this slice (global indices), keyed by reward and by raw
        vecs = [tuple(int(x) for x in v) for v in data["vectors"][lo:hi]]
        valid = data["valid"][lo:hi]
        elites = {}
        for cap in (3, 8):
            by_rew = elite_offers(vecs, rewards, valid, cap)
            by_raw = elite_offers(vecs, list(raws[lo:hi]), valid, cap)
            elites[cap] = ([(v, k, i + lo) for v, k, i in by_rew], [(v, k, i + lo) for v, k, i in by_raw])
        gathered = [None] * world
        dist.all_gather_object(gathered, {"rewards": rewards, "elites": elites, "best": best_all})
        if rank == 0:
            out_q.put(gathered)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["moe_1p2t_stream", "moe_1p2t_stream_b0", "tiny_stream"])
def test_two_rank_rewards_and_elites_match_sequential(name):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    wl, meta, data = load_search(name)
    # rewards: concatenation of per-rank rewards == reference sequential stream
    rewards = np.concatenate([np.asarray(g["rewards"]) for g in gathered])
    assert np.array_equal(rewards.view(np.uint64), data["rewards"].view(np.uint64))
    assert gathered[0]["best"] == meta["best_raw_final"]
    vecs_all = [tuple(int(x) for x in v) for v in data["vectors"]]
    for cap in (3, 8):
        merged_rew = elite_merge([g["elites"][cap][0] for g in gathered], cap)
        want = data[f"elite{cap}_vectors"]
        assert [m[0] for m in merged_rew] == [tuple(int(x) for x in v) for v in want]
        assert [m[1] for m in merged_rew] == list(data[f"elite{cap}_rewards"])
        merged_raw = elite_merge([g["elites"][cap][1] for g in gathered], cap)
        want_raw = elite_offers(vecs_all, list(data["raws"]), data["valid"], cap)
        assert [(m[0], m[2]) for m in merged_raw] == [(w[0], w[2]) for w in want_raw]
