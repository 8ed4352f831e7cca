"""Policy network parity against the reference's numpy PolicyNetwork
(golden fixture tests/golden/policy_reference.npz, made by
tests/golden/make_golden_ppo.py from the reference itself).

Runs the TorchPolicy on the CPU in float64: same initialisation draws (bit
exact), forward within 1e-12, autograd gradients of the PPO loss against the
reference's hand-written backward within 1e-10, and one ppo_update (two Adam
epochs) within 1e-9.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2509_00217_b200.config import load_workload
from paper_2509_00217_b200.knobs import PpoConfig
from paper_2509_00217_b200.policy import (CheckpointError, EliteBuffer, TorchPolicy, build_observation, head_masks,
                                          load_checkpoint, sample_actions, save_checkpoint)
from ppo_torch_engine import ppo_loss
from paper_2509_00217_b200.strategy import canonical_fused_ops

GOLD = np.load(Path(__file__).parent / "golden" / "policy_reference.npz")


@pytest.fixture(scope="module")
def wl():
    return load_workload("moe_1p2t_h100")


def make_policy(wl, width=16, ffn=8):
    return TorchPolicy(wl.space, canonical_fused_ops(wl.model), history_len=3, width=width, ffn_width=ffn,
                       device="cpu")


def test_init_draws_match_reference_bit_exactly(wl):
    pol = make_policy(wl)
    state = pol.init_state(np.random.default_rng(11))
    for name, ref in ((k[6:], GOLD[k]) for k in GOLD.files if k.startswith("param.")):
        np.testing.assert_array_equal(state[name], ref, err_msg=name)
    assert set(state) == {k[6:] for k in GOLD.files if k.startswith("param.")}


def loaded(wl):
    pol = make_policy(wl)
    pol.load_state({k[6:]: GOLD[k] for k in GOLD.files if k.startswith("param.")})
    return pol


def test_forward_matches_reference(wl):
    pol = loaded(wl)
    for i in (0, 1):
        obs = torch.from_numpy(GOLD[f"obs{i}"])
        with torch.no_grad():
            log_probs, probs, value = pol(obs)
        ref_p = GOLD[f"probs{i}"]
        ok = ~np.isnan(ref_p)
        np.testing.assert_allclose(probs.numpy()[ok], ref_p[ok], rtol=0, atol=1e-13)
        assert (probs.numpy()[~ok] == 0).all()
        np.testing.assert_allclose(float(value), float(GOLD[f"value{i}"]), rtol=1e-12, atol=1e-14)
        ent = float(pol.entropy(log_probs, probs))
        np.testing.assert_allclose(ent, float(GOLD[f"entropy{i}"]), rtol=1e-12)


def test_sampling_consumes_the_reference_stream(wl):
    """Same generator positions as the reference fixture: init, two integer
    vectors for the elite offers, then one random() per head per sample."""
    pol = loaded(wl)
    rng = np.random.default_rng(11)
    pol.init_state(rng)
    for _ in range(2):
        for k in wl.space.head_sizes:
            rng.integers(k)
    cap = pol.sizes - 1
    for i in (0, 1):
        with torch.no_grad():
            _, probs, _ = pol(torch.from_numpy(GOLD[f"obs{i}"]))
        act = sample_actions(probs, torch.from_numpy(rng.random(wl.space.vector_length)), cap)
        np.testing.assert_array_equal(act.numpy(), GOLD[f"action{i}"])


def rollout(pol):
    obs = torch.from_numpy(np.stack([GOLD["obs0"], GOLD["obs1"]]))
    act = torch.from_numpy(np.stack([GOLD["action0"], GOLD["action1"]]).astype(np.int64))
    logp = torch.tensor([float(GOLD["logprob0"]), float(GOLD["logprob1"])], dtype=torch.float64)
    val = torch.tensor([float(GOLD["value0"]), float(GOLD["value1"])], dtype=torch.float64)
    rew = torch.tensor([3.0, -10.0], dtype=torch.float64)
    return obs, act, logp, val, rew


def test_autograd_gradients_match_reference_backward(wl):
    pol = loaded(wl)
    loss = ppo_loss(pol, *rollout(pol), PpoConfig())
    np.testing.assert_allclose(float(loss.detach()), float(GOLD["loss"][3]), rtol=1e-12)
    loss.backward()
    for name in pol.names:
        ref = GOLD["grad." + name]
        np.testing.assert_allclose(_grad_of(pol, name), ref, rtol=1e-10, atol=1e-13 * max(1.0, np.abs(ref).max()),
                                   err_msg=name)


def _grad_of(pol, name):
    """Gradient of a reference-named parameter, read out of the packed .grad tensors."""
    views = {}
    d, nh, kmax = pol.width, pol.num_heads, pol.kmax
    gw, gb = pol.head_w.grad.view(d, nh, kmax), pol.head_b.grad.view(nh, kmax)
    views.update({"attn.wq": pol.wqkv.grad[:, :d], "attn.wk": pol.wqkv.grad[:, d:2 * d], "attn.wv": pol.wqkv.grad[:, 2 * d:],
                  "attn.bq": pol.bqkv.grad[:d], "attn.bk": pol.bqkv.grad[d:2 * d], "attn.bv": pol.bqkv.grad[2 * d:]})
    for i, k in enumerate(pol.head_sizes):
        views[f"head.{i}.w"] = gw[:, i, :k]
        views[f"head.{i}.b"] = gb[i, :k]
    if name in views:
        return views[name].numpy()
    return pol.p(name).grad.numpy()


def test_padding_columns_never_move(wl):
    pol = loaded(wl)
    ppo_loss(pol, *rollout(pol), PpoConfig()).backward()
    d, nh, kmax = pol.width, pol.num_heads, pol.kmax
    masks = head_masks(wl.space, canonical_fused_ops(wl.model))
    gw = pol.head_w.grad.view(d, nh, kmax).numpy()
    for i, m in enumerate(masks):
        blocked = np.ones(kmax, dtype=bool)
        blocked[: len(m)] = ~m
        assert (gw[:, i, blocked] == 0).all()


def test_two_adam_epochs_match_reference_update(wl):
    pol = loaded(wl)
    opt = torch.optim.Adam(pol.parameters(), lr=1e-3, betas=(0.9, 0.999), eps=1e-8, foreach=True)
    batch = rollout(pol)
    for _ in range(2):
        opt.zero_grad()
        ppo_loss(pol, *batch, PpoConfig()).backward()
        opt.step()
    state = pol.state()
    for name in pol.names:
        ref = GOLD["updated." + name]
        np.testing.assert_allclose(state[name], ref, rtol=1e-9, atol=1e-12, err_msg=name)


def test_fresh_policy_is_uniform_over_admissible_choices(wl):
    pol = make_policy(wl, width=32, ffn=32)
    pol.reset_parameters(np.random.default_rng(0))
    masks = head_masks(wl.space, canonical_fused_ops(wl.model))
    with torch.no_grad():
        _, probs, value = pol(torch.zeros(3, wl.space.vector_length, dtype=torch.float64))
    assert float(value) == 0.0
    for i, m in enumerate(masks):
        row = probs[i, : len(m)].numpy()
        np.testing.assert_allclose(row[m], 1.0 / m.sum(), rtol=1e-15)
        assert (row[~m] == 0).all()


def test_elite_buffer_and_observation_rules(wl):
    buf = EliteBuffer(3)
    v = [tuple([i] + [0] * (wl.space.vector_length - 1)) for i in range(4)]
    assert buf.offer(v[0], 5.0) and buf.offer(v[1], 5.0) and buf.offer(v[2], 7.0)
    assert not buf.offer(v[0], 9.0)  # duplicate vector
    assert not buf.offer(v[3], 5.0)  # full, not better than the minimum
    assert [e.vector for e in buf.entries] == [v[2], v[0], v[1]]  # stable among equal rewards
    assert buf.offer(v[3], 6.0)
    assert [e.reward for e in buf.entries] == [7.0, 6.0, 5.0]
    obs = build_observation(buf, wl.space)
    pol = make_policy(wl)
    ev = torch.tensor([list(e.vector) for e in buf.entries], dtype=torch.int64)
    er = torch.tensor([e.reward for e in buf.entries], dtype=torch.float64)
    np.testing.assert_array_equal(pol.observation(ev, er).numpy(), obs)
    er[2] = float("-inf")  # empty slot renders as zeros
    assert (pol.observation(ev, er).numpy()[2] == 0).all()


def test_checkpoint_round_trip_and_errors(wl, tmp_path):
    pol = loaded(wl)
    path = tmp_path / "p.sspl"
    save_checkpoint(str(path), pol.state())
    back = load_checkpoint(str(path))
    other = make_policy(wl)
    other.load_state(back)
    for n in pol.names:
        np.testing.assert_array_equal(other.state()[n], pol.state()[n])
    raw = path.read_bytes()
    (tmp_path / "bad").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(CheckpointError):
        load_checkpoint(str(tmp_path / "bad"))
    (tmp_path / "short").write_bytes(raw[:-9])
    with pytest.raises(CheckpointError):
        load_checkpoint(str(tmp_path / "short"))
    with pytest.raises(ValueError):
        other.load_state({k: v for k, v in back.items() if k != "ln1.g"})


def test_arena_layout_matches_the_c_abi(wl):
    """TorchPolicy's flat parameter arena is the layout ls_policy_layout_of
    documents, so the fused kernels and autograd share storage."""
    import ctypes

    from paper_2509_00217_b200 import _native

    lib = _native.lib()
    for width, ffn, hist, steps in ((16, 8, 3, 2), (256, 256, 3, 2), (64, 64, 4, 4)):
        pol = make_policy(wl, width=width, ffn=ffn)
        dims = _native.PolicyDims(wl.space.vector_length, width, ffn, hist, pol.num_heads, pol.kmax, steps)
        lay = _native.PolicyLayout()
        assert lib.ls_policy_layout_of(ctypes.byref(dims), ctypes.byref(lay)) == 0
        assert list(lay.off) == pol.offsets
        assert lay.total == pol.flat.numel()
        assert lib.ls_ppo_workspace_bytes(ctypes.byref(dims)) > 0
    too_many_rows = _native.PolicyDims(wl.space.vector_length, 16, 8, 9, 16, 11, 2)
    assert lib.ls_ppo_workspace_bytes(ctypes.byref(too_many_rows)) == 0
    bad = _native.PolicyDims(0, 16, 8, 3, 16, 11, 2)
    assert lib.ls_policy_layout_of(ctypes.byref(bad), ctypes.byref(_native.PolicyLayout())) != 0


def test_search_structs_have_the_header_layout():
    import ctypes

    from paper_2509_00217_b200 import _native

    assert ctypes.sizeof(_native.SearchState) == 104
    assert ctypes.sizeof(_native.PolicyDims) == 28
    assert ctypes.sizeof(_native.PolicyLayout) == 8 * 21
    # dims (28, padded to 32) + 8 pointers + state + 10 pointers + 7 doubles + int (padded)
    assert ctypes.sizeof(_native.PpoPlan) == 32 + 64 + 104 + 80 + 56 + 8
