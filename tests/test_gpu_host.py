"""Host-buffer entry points: compact host results (ls_evaluate_host_compact —
reason bytes + the valid candidates' raws, from host planes packed on host
threads or from packed words) must equal the full host path
(ls_evaluate_host) and the oracle, for ragged sizes, several pipeline
chunks, decode errors and an undersized result buffer."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from golden_io import load_eval  # noqa: E402


def _planes(ev, n, seed, bad=0):
    rng = np.random.default_rng(seed)
    p = np.stack([rng.integers(0, k, size=n, dtype=np.uint8) for k in ev.head_sizes])
    if bad:
        idx = rng.choice(n, size=bad, replace=False)
        p[rng.integers(0, p.shape[0], size=bad), idx] = 250  # decode errors
    return p


@pytest.mark.parametrize("name", ["moe_1p6t_2048", "llama3_70b_h100x64", "tiny"])
@pytest.mark.parametrize("n", [1, 4097, (1 << 22) * 2 + 12345])
def test_compact_equals_full_host_path(name, n):
    from oracle.cost_model import simulate_planes
    from paper_2509_00217_b200.evaluator import Evaluator

    wl, _, _ = load_eval(name)
    ev = Evaluator(wl, device=0)
    planes = _planes(ev, n, 3, bad=min(n, 50))
    want = simulate_planes(wl.desc(), planes, fields=("throughput",))
    reason, vraw = ev.evaluate_host_compact(planes)
    assert np.array_equal(reason, want["reason"])
    dense = Evaluator.scatter_raw(reason, vraw)
    assert np.array_equal(dense.view(np.uint64), want["throughput"].view(np.uint64))
    full = ev.evaluate_host(planes)
    assert np.array_equal(full["reason"], reason)
    # packed words from the host
    words = ev.pack(torch.from_numpy(planes).cuda()).cpu().numpy()
    r2, v2 = ev.evaluate_host_compact(words)
    assert np.array_equal(r2, reason) and np.array_equal(v2.view(np.uint64), vraw.view(np.uint64))


def test_compact_host_packing_equals_raw_planes(monkeypatch):
    """LS_HOST_PACK=1: planes packed on host worker threads (SWAR packer) give the
    same results as copying the planes (ragged sizes, decode errors)."""
    from paper_2509_00217_b200.evaluator import Evaluator

    wl, _, _ = load_eval("moe_1p6t_2048")
    raw = Evaluator(wl, device=0)
    monkeypatch.setenv("LS_HOST_PACK", "1")
    packed = Evaluator(wl, device=0)
    for n in (7, 8, 4099, (1 << 22) + 13):
        planes = _planes(raw, n, n, bad=min(n, 40))
        r1, v1 = raw.evaluate_host_compact(planes)
        r2, v2 = packed.evaluate_host_compact(planes)
        assert np.array_equal(r1, r2) and np.array_equal(v1.view(np.uint64), v2.view(np.uint64)), n


def test_compact_strided_planes_and_capacity():
    from paper_2509_00217_b200._native import NativeError
    from paper_2509_00217_b200.evaluator import Evaluator

    wl, _, _ = load_eval("moe_1p2t")
    ev = Evaluator(wl, device=0)
    big = _planes(ev, 300_000, 9)
    view = big[:, 1000:251_000]  # plane stride 300000, not contiguous across heads
    reason, vraw = ev.evaluate_host_compact(view)
    r_ref, v_ref = ev.evaluate_host_compact(np.ascontiguousarray(view))
    assert np.array_equal(reason, r_ref) and np.array_equal(vraw, v_ref)
    nvalid = int((reason == 0).sum())
    assert nvalid == len(vraw) > 10
    with pytest.raises(NativeError, match="capacity"):
        ev.evaluate_host_compact(view, valid_raw=np.empty(nvalid - 1))
    r3, v3 = ev.evaluate_host_compact(view)  # the context recovers
    assert np.array_equal(r3, reason)
