"""Packed candidate words (ls_evaluate_packed / ls_evaluate_packed_topk /
ls_evaluate_host_packed / ls_pack): the same verdicts as the planes path and
the reference's golden values, bit for bit; malformed words are decode errors."""

import numpy as np
import pytest

from golden_io import eval_sets, load_eval, mismatches

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2509_00217_b200.strategy import pack_vectors, packed_layout, unpack_words  # noqa: E402


@pytest.fixture(scope="module")
def ev_factory():
    from paper_2509_00217_b200.evaluator import Evaluator

    made = []

    def make(workload):
        e = Evaluator(workload, device=0)
        made.append(e)
        return e

    yield make
    for e in made:
        e.close()


def _words(vecs, space):
    return torch.from_numpy(pack_vectors(vecs, space).view(np.int64)).cuda()


@pytest.mark.parametrize("name", eval_sets())
def test_packed_golden_bit_exact(name, ev_factory):
    wl, meta, data = load_eval(name)
    if wl.space.vector_length > 16:
        pytest.skip("packed words cover vectors of <= 16 heads")
    ev = ev_factory(wl)
    assert ev.packed_layout() == packed_layout(wl.space)
    got = ev.evaluate_packed(_words(data["vectors"], wl.space), fields="all").numpy()
    bad = mismatches(got, data)
    assert not bad.any(), f"{int(bad.sum())} mismatches, first at {np.nonzero(bad)[0][:5]}"
    host = ev.evaluate_host_packed(pack_vectors(data["vectors"], wl.space), fields="all")
    assert not mismatches(host, data).any()


@pytest.mark.parametrize("name", ["moe_1p2t", "edge_odd", "tiny"])
def test_device_pack_equals_host_pack_and_round_trips(name, ev_factory):
    wl, meta, data = load_eval(name)
    ev = ev_factory(wl)
    rng = np.random.default_rng(1)
    vecs = np.concatenate([data["vectors"], rng.integers(0, 5, size=(5000, wl.space.vector_length))])
    planes = torch.from_numpy(np.ascontiguousarray(vecs.T.astype(np.uint8))).cuda()
    dev = ev.pack(planes).cpu().numpy().view(np.uint64)
    np.testing.assert_array_equal(dev, pack_vectors(vecs, wl.space))
    ok = dev != np.uint64(0xFFFFFFFFFFFFFFFF)
    np.testing.assert_array_equal(unpack_words(dev[ok], wl.space), vecs[ok])
    # every vector verdict equals the planes path, including decode errors
    a = ev.evaluate(planes, fields="all").numpy()
    b = ev.evaluate_packed(ev.pack(planes), fields="all").numpy()
    assert not mismatches(b, a).any()


def test_malformed_words_are_decode_errors(ev_factory):
    wl, meta, data = load_eval("moe_1p2t")
    ev = ev_factory(wl)
    shift, size = packed_layout(wl.space)
    good = pack_vectors(data["vectors"][:5], wl.space)
    low24 = np.uint64((1 << 24) - 1)
    bad = [good[0] | np.uint64(1 << 63), good[1] | np.uint64(1 << 48),  # bits past the rank field
           good[2] | np.uint64(3 << 4),  # an axis field holding 3
           (good[3] & low24) | np.uint64(size << shift),  # rank past the coarse space
           good[4] | np.uint64(1 << 23)]  # axis bits past head A (A = 16 uses all 24: use a 14-head set below)
    words = torch.from_numpy(np.asarray(bad[:4], dtype=np.uint64).view(np.int64)).cuda()
    got = ev.evaluate_packed(words).numpy()
    assert (got["reason"] == 255).all() and (got["throughput"] == 0).all()
    wl14, _, data14 = load_eval("llama3_8b_h100x8")  # A = 14: axis bits 20..23 must be zero
    ev14 = ev_factory(wl14)
    w14 = pack_vectors(data14["vectors"][:2], wl14.space)
    w14[1] |= np.uint64(1 << 21)
    got = ev14.evaluate_packed(torch.from_numpy(w14.view(np.int64)).cuda()).numpy()
    assert got["reason"][1] == 255 and got["reason"][0] != 255


@pytest.mark.parametrize("n", [0, 1, 5, 1023, 1024, 1025, 4097, 300_001])
def test_ragged_sizes_match_planes(n, ev_factory):
    wl, meta, data = load_eval("moe_1p6t_2048")
    ev = ev_factory(wl)
    rng = np.random.default_rng(n)
    vecs = np.stack([rng.integers(0, k, size=n) for k in wl.space.head_sizes], axis=1) if n else \
        np.zeros((0, wl.space.vector_length), dtype=np.int64)
    planes = torch.from_numpy(np.ascontiguousarray(vecs.T.astype(np.uint8))).cuda()
    words = _words(vecs, wl.space)
    a = ev.evaluate(planes, fields="all").numpy() if n else None
    b = ev.evaluate_packed(words, fields="all").numpy()
    if n:
        assert not mismatches(b, a).any()
    _, r1, c1 = ev.evaluate_topk(planes, k=8, index_base=7)
    _, r2, c2 = ev.evaluate_packed_topk(words, k=8, index_base=7)
    got, want = ev.decode_records(r2, c2), ev.decode_records(r1, c1)
    assert [(e.vector, e.index, e.raw) for e in got] == [(e.vector, e.index, e.raw) for e in want]
    _, r3, c3 = ev.evaluate_packed_topk(words, k=8, index_base=7, verdicts=False)
    assert [e.index for e in ev.decode_records(r3, c3)] == [e.index for e in want]


@pytest.mark.parametrize("n", [4, 4096, 4098, 100_003])
def test_pack_vectorised_path_and_tail(n, ev_factory):
    """ls_pack's 4-per-thread path (4-byte aligned planes, stride % 4 == 0)
    plus the per-candidate tail equal the host packing, malformed heads
    included."""
    wl, meta, data = load_eval("moe_1p2t")
    ev = ev_factory(wl)
    rng = np.random.default_rng(n)
    vecs = rng.integers(0, 4, size=(n, wl.space.vector_length))
    vecs[:, :4] = np.stack([rng.integers(0, k + 1, size=n) for k in wl.space.head_sizes[:4]], axis=1)
    width = (n + 3) // 4 * 4 + 4  # stride % 4 == 0 with n % 4 != 0 for the odd sizes
    big = np.zeros((wl.space.vector_length, width), dtype=np.uint8)
    big[:, :n] = vecs.T
    planes = torch.from_numpy(big).cuda()[:, :n]
    dev = ev.pack(planes).cpu().numpy().view(np.uint64)
    np.testing.assert_array_equal(dev, pack_vectors(vecs, wl.space))


@pytest.mark.parametrize("fields", ["all", ("throughput",)])
def test_fused_back_to_back_verdicts_and_elites(fields):
    """Consecutive fused launches on one stream (programmatic dependent launch,
    dynamic tile claims, the ragged tail tile claimed by any CTA) over planes and
    packed words, with one or all six verdict fields: every verdict bit equals
    the oracle's and every elite equals the standalone top-k of the batch."""
    from oracle.cost_model import simulate_planes
    from paper_2509_00217_b200.evaluator import Evaluator

    wl, _, _ = load_eval("moe_1p6t_2048")
    ev = Evaluator(wl, device=0)
    rng = np.random.default_rng(41)
    for n in (2047, 2049, 5 * 2048 + 77, 1 << 20, (1 << 22) + 4093):
        planes_np = np.stack([rng.integers(0, k, size=n, dtype=np.uint8) for k in ev.head_sizes])
        want = simulate_planes(wl.desc(), planes_np)
        planes = torch.from_numpy(planes_np).cuda()
        words = ev.pack(planes)
        runs = []
        for _ in range(3):  # back to back, no sync in between
            runs.append(ev.evaluate_topk(planes, k=8, index_base=11, fields=fields))
            runs.append(ev.evaluate_packed_topk(words, k=8, index_base=11, fields=fields))
        torch.cuda.synchronize()
        _, r0, c0 = ev.evaluate_topk(planes, k=8, index_base=11, verdicts=False)
        ref_elite = ev.decode_records(r0, c0)
        for out, recs, count in runs:
            got = out.numpy()
            assert np.array_equal(got["reason"], want["reason"]), n
            for f in got:
                if f != "reason":
                    assert np.array_equal(np.asarray(got[f]).view(np.uint64), want[f].view(np.uint64)), (n, f)
            assert ev.decode_records(recs, count) == ref_elite, n
