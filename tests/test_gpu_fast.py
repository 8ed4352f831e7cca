"""The fp32 fast mode of the on-device sweeps (ls_set_precision LS_PREC_FP32,
north_star: "1e-5 in the fp32 fast mode"): every elite record is a valid
candidate per the oracle with raw within 1e-5 relative of the reference's
value, and the elite equals the fp64 (bit-exact) elite up to reorderings
among candidates whose raws agree to 1e-5."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from golden_io import load_eval  # noqa: E402

REL = 1e-5


def _oracle_raw(wl, vectors):
    from oracle.cost_model import simulate_planes

    planes = np.ascontiguousarray(np.asarray(vectors, dtype=np.uint8).T)
    return simulate_planes(wl.desc(), planes, fields=("throughput",))


@pytest.mark.parametrize("name", ["moe_1p2t", "moe_1p6t_2048", "llama3_70b_h100x64", "edge_odd"])
@pytest.mark.parametrize("mode", [1, 3])
def test_fp32_sweep_elite_within_1e5(name, mode):
    from paper_2509_00217_b200.evaluator import Evaluator

    wl, _, _ = load_eval(name)
    ev = Evaluator(wl, device=0)
    n = min(ev.stream_size(mode), 1 << 22) if mode != 1 else 1 << 22
    k = 16
    exact = ev.decode_records(*ev.sweep(mode, n, k=k, seed=5))
    ev.set_precision("fp32")
    fast = ev.decode_records(*ev.sweep(mode, n, k=k, seed=5))
    ev.set_precision("fp64")
    assert len(fast) == len(exact)
    want = _oracle_raw(wl, [e.vector for e in fast])
    assert (want["reason"] == 0).all()
    rel = np.abs(np.asarray([e.raw for e in fast]) - want["throughput"]) / want["throughput"]
    assert rel.max() <= REL, rel.max()
    # membership: an exact record clearly above the k-th is in the fast elite
    kth = exact[-1].raw
    fast_idx = {e.index for e in fast}
    for e in exact:
        if e.raw > kth * (1 + 2 * REL):
            assert e.index in fast_idx or any(abs(f.raw - e.raw) <= 2 * REL * e.raw for f in fast), e
    assert ev.decode_records(*ev.sweep(mode, n, k=k, seed=5)) == exact  # back to bit-exact
