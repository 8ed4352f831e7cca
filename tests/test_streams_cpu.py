"""Host twin of the on-device candidate streams (generator.py): enumeration
order is itertools.product order (the reference's exhaustive sweeps,
baselines.py:172-179, test_acceptance.py:86) and the uniform stream covers
every head's domain uniformly."""

import itertools

import numpy as np

from golden_io import load_eval
from paper_2509_00217_b200.generator import GEN_ENUM, GEN_ENUM_ADMISSIBLE, GEN_UNIFORM, stream_size, stream_vectors
from paper_2509_00217_b200.strategy import AxisChoice, canonical_fused_ops


def test_enum_is_itertools_product_order():
    wl, _, _ = load_eval("tiny")
    want = np.asarray(list(itertools.product(*(range(k) for k in wl.space.head_sizes))))
    got = stream_vectors(wl.model, wl.space, GEN_ENUM, 0, len(want))
    assert np.array_equal(got, want)
    assert stream_size(wl.model, wl.space, GEN_ENUM) == len(want) == 6561
    mid = stream_vectors(wl.model, wl.space, GEN_ENUM, 1234, 77)
    assert np.array_equal(mid, want[1234:1311])


def test_admissible_enum_matches_filtered_product():
    wl, _, _ = load_eval("unit_small")
    ops = {op.name: op for op in canonical_fused_ops(wl.model)}
    choices = [range(k) for k in wl.space.head_sizes[:4]]
    choices += [[a for a in (0, 1, 2) if ops[n].admits(AxisChoice(a))] for n in wl.space.op_names]
    size = stream_size(wl.model, wl.space, GEN_ENUM_ADMISSIBLE)
    assert size == int(np.prod([len(c) for c in choices]))
    want = np.asarray(list(itertools.islice(itertools.product(*choices), 5000)))
    assert np.array_equal(stream_vectors(wl.model, wl.space, GEN_ENUM_ADMISSIBLE, 0, 5000), want)
    # the 1.2T admissible subspace of SURVEY.md §0: 49,509,306 points of 2,005,126,893
    big, _, _ = load_eval("moe_1p2t")
    assert stream_size(big.model, big.space, GEN_ENUM) == 2_005_126_893
    assert stream_size(big.model, big.space, GEN_ENUM_ADMISSIBLE) == 3773 * 13122


def test_uniform_stream_covers_domains_uniformly():
    wl, _, _ = load_eval("moe_1p2t")
    v = stream_vectors(wl.model, wl.space, GEN_UNIFORM, 0, 200_000, seed=7)
    for h, k in enumerate(wl.space.head_sizes):
        counts = np.bincount(v[:, h], minlength=k)
        assert len(counts) == k and counts.min() > 0
        assert np.abs(counts / len(v) - 1 / k).max() < 0.01
    # counter based: any window equals the same positions of a longer draw
    w = stream_vectors(wl.model, wl.space, GEN_UNIFORM, 123, 1000, seed=7)
    assert np.array_equal(w, v[123:1123])
    assert not np.array_equal(stream_vectors(wl.model, wl.space, GEN_UNIFORM, 0, 1000, seed=8), v[:1000])


def test_oracle_uniform_stream_matches_generator():
    """oracle/streams.c (the host twin bench.py's parity block uses) regenerates
    the same vectors as generator.py, which the GPU tests pin to the device."""
    from oracle.cost_model import uniform_planes

    for name in ("moe_1p6t_2048", "llama3_70b_h100x64", "tiny"):
        wl, _, _ = load_eval(name)
        for seed, start, n in ((0, 0, 5000), (2**64 - 3, 1 << 33, 777), (1000, 12345, 4096)):
            want = stream_vectors(wl.model, wl.space, GEN_UNIFORM, start, n, seed=seed)
            got = uniform_planes(wl.desc(), seed, start, n, threads=3)
            assert np.array_equal(got.T.astype(np.int64), want), (name, seed, start)
