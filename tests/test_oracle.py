"""Pins for the fp64 attention oracle (oracle/oracle_attn.c) -- CPU only.

Each test checks the oracle against something other than itself, chosen so
that a plausible mistake (dropped scale, wrong max, transposed operand,
wrong GQA index, off-by-one causal mask, j/i swap) fails at least one:

  closed form   two-key softmax worked by hand                  (eq:fa)
  library       torch float64 softmax(QK^T*scale + mask) @ V
  invariants    rows sum to 1; constant V -> V; joint K/V key
                permutation; causal row i ignores keys j > i;
                scale = 0 -> (prefix) mean; hard-attention limit
  reduction     GQA == MHA with K/V repeat_interleave
  widening      bf16 bit patterns widen exactly
"""
import math

import numpy as np
import pytest
import torch

from oracle import attn as oa

pytestmark = pytest.mark.filterwarnings("ignore::UserWarning")


def _rand(shape, seed, dtype=torch.float64):
    g = torch.Generator().manual_seed(seed)
    return torch.randn(shape, generator=g, dtype=torch.float64).to(dtype)


def torch_reference(q, k, v, causal, scale):
    """Library-routine pin: torch fp64 softmax with repeat_interleave for GQA."""
    q, k, v = (t.to(torch.float64) for t in (q, k, v))
    G = q.shape[1] // k.shape[1]
    k = k.repeat_interleave(G, dim=1)
    v = v.repeat_interleave(G, dim=1)
    s = torch.einsum("bhid,bhjd->bhij", q, k) * scale
    if causal:
        N = q.shape[2]
        mask = torch.triu(torch.ones(N, N, dtype=torch.bool), diagonal=1)
        s = s.masked_fill(mask, float("-inf"))
    return torch.einsum("bhij,bhjd->bhid", torch.softmax(s, dim=-1), v).numpy()


def test_two_key_closed_form():
    # B=H=1, N=2, d=1, scale=1: q=[1,2], k=[0,1], v=[1,3]
    q = np.array([1.0, 2.0]).reshape(1, 1, 2, 1)
    k = np.array([0.0, 1.0]).reshape(1, 1, 2, 1)
    v = np.array([1.0, 3.0]).reshape(1, 1, 2, 1)
    e = math.e
    o = oa.attention(q, k, v, causal=False, scale=1.0)
    assert o[0, 0, 0, 0] == pytest.approx((1 + 3 * e) / (1 + e), rel=1e-15)
    assert o[0, 0, 1, 0] == pytest.approx((1 + 3 * e**2) / (1 + e**2), rel=1e-15)
    oc = oa.attention(q, k, v, causal=True, scale=1.0)
    assert oc[0, 0, 0, 0] == 1.0  # row 0 sees key 0 only
    assert oc[0, 0, 1, 0] == pytest.approx((1 + 3 * e**2) / (1 + e**2), rel=1e-15)


def test_default_scale_is_inv_sqrt_d():
    q, k, v = (_rand((1, 1, 5, 4), s) for s in (1, 2, 3))
    a = oa.attention(q, k, v)
    b = oa.attention(q, k, v, scale=0.5)  # 1/sqrt(4)
    np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("B,Hq,Hkv,N,d,causal", [
    (1, 2, 2, 17, 16, False), (2, 4, 2, 33, 64, True), (1, 4, 1, 64, 128, True),
    (2, 3, 3, 128, 16, False), (1, 2, 2, 256, 64, True),
])
def test_matches_torch_fp64(B, Hq, Hkv, N, d, causal):
    q = _rand((B, Hq, N, d), 10)
    k = _rand((B, Hkv, N, d), 11)
    v = _rand((B, Hkv, N, d), 12)
    scale = 1.0 / math.sqrt(d)
    np.testing.assert_allclose(oa.attention(q, k, v, causal, scale),
                               torch_reference(q, k, v, causal, scale), rtol=0, atol=1e-12)


def test_float32_and_bf16_inputs_widen_exactly():
    qf = _rand((1, 2, 31, 16), 20, torch.float32)
    kf = _rand((1, 2, 31, 16), 21, torch.float32)
    vf = _rand((1, 2, 31, 16), 22, torch.float32)
    ref = torch_reference(qf, kf, vf, True, 0.25)
    np.testing.assert_allclose(oa.attention(qf, kf, vf, True, 0.25), ref, atol=1e-12, rtol=0)
    qb, kb, vb = (t.to(torch.bfloat16) for t in (qf, kf, vf))
    # bf16 widened exactly == the same values passed as float64
    np.testing.assert_array_equal(
        oa.attention(qb, kb, vb, True, 0.25),
        oa.attention(qb.double(), kb.double(), vb.double(), True, 0.25))
    # and a few known bit patterns: 0x3F80 = 1.0, 0xC000 = -2.0, 0x3E00 = 0.125
    bits = np.array([0x3F80, 0xC000, 0x3E00, 0x0000], dtype=np.uint16).reshape(1, 1, 1, 4)
    one = np.zeros((1, 1, 1, 4), dtype=np.uint16)
    w, o = oa.attention_weights(one, one, bits, 0, 0, 0, scale=1.0)
    np.testing.assert_array_equal(o, [1.0, -2.0, 0.125, 0.0])


def test_weights_sum_to_one_and_match_softmax():
    q, k, v = (_rand((1, 2, 40, 8), s) for s in (30, 31, 32))
    for causal in (False, True):
        for i in (0, 7, 39):
            w, o = oa.attention_weights(q, k, v, 0, 1, i, causal=causal, scale=0.3)
            assert w.sum() == pytest.approx(1.0, abs=1e-14)
            if causal:
                assert np.all(w[i + 1:] == 0.0)
            np.testing.assert_allclose(o, w @ v[0, 1].numpy(), atol=1e-13, rtol=0)


def test_constant_v_returns_v():
    q, k = _rand((2, 2, 50, 16), 40), _rand((2, 2, 50, 16), 41)
    v = torch.full((2, 2, 50, 16), 0.0, dtype=torch.float64)
    v += torch.arange(16, dtype=torch.float64) * 0.5 - 3.0
    for causal in (False, True):
        o = oa.attention(q, k, v, causal, 0.7)
        np.testing.assert_allclose(o, np.broadcast_to(v.numpy(), o.shape), atol=1e-13, rtol=0)


def test_joint_key_permutation_invariance():
    q, k, v = (_rand((1, 2, 64, 32), s) for s in (50, 51, 52))
    perm = torch.randperm(64, generator=torch.Generator().manual_seed(5))
    a = oa.attention(q, k, v, False, 0.2)
    b = oa.attention(q, k[:, :, perm], v[:, :, perm], False, 0.2)
    np.testing.assert_allclose(a, b, atol=1e-13, rtol=0)
    # permuting K alone does change the answer (R12)
    c = oa.attention(q, k[:, :, perm], v, False, 0.2)
    assert np.abs(a - c).max() > 1e-3


def test_causal_row_ignores_future_keys():
    q, k, v = (_rand((1, 1, 48, 16), s) for s in (60, 61, 62))
    a = oa.attention(q, k, v, True, 0.25)
    for i in (0, 10, 47):
        k2, v2 = k.clone(), v.clone()
        k2[:, :, i + 1:] = 100.0 * _rand(k2[:, :, i + 1:].shape, 63)
        v2[:, :, i + 1:] = -50.0
        b = oa.attention(q, k2, v2, True, 0.25)
        np.testing.assert_array_equal(a[:, :, : i + 1], b[:, :, : i + 1])
    # row 0 is v_0 exactly
    np.testing.assert_array_equal(a[0, 0, 0], v[0, 0, 0].numpy())


def test_scale_zero_is_mean():
    q, k, v = (_rand((1, 2, 20, 8), s) for s in (70, 71, 72))
    o = oa.attention(q, k, v, False, 0.0)
    np.testing.assert_allclose(o, np.broadcast_to(v.numpy().mean(axis=2, keepdims=True), o.shape),
                               atol=1e-14, rtol=0)
    oc = oa.attention(q, k, v, True, 0.0)
    prefix = np.cumsum(v.numpy(), axis=2) / np.arange(1, 21).reshape(1, 1, 20, 1)
    np.testing.assert_allclose(oc, prefix, atol=1e-14, rtol=0)


def test_hard_attention_limit():
    # distinct orthogonal keys; q_i = alpha * k_t(i) -> o_i -> v_t(i)
    N, d = 8, 8
    k = torch.eye(N, d, dtype=torch.float64).reshape(1, 1, N, d)
    v = _rand((1, 1, N, d), 80)
    tgt = [3, 0, 7, 5, 1, 6, 2, 4]
    q = torch.stack([60.0 * k[0, 0, t] for t in tgt]).reshape(1, 1, N, d)
    o = oa.attention(q, k, v, False, 1.0)
    np.testing.assert_allclose(o[0, 0], v[0, 0, tgt].numpy(), atol=1e-20, rtol=1e-20)


def test_gqa_equals_mha_with_repeated_kv():
    q = _rand((2, 8, 24, 16), 90)
    k, v = _rand((2, 2, 24, 16), 91), _rand((2, 2, 24, 16), 92)
    a = oa.attention(q, k, v, True, 0.25)
    b = oa.attention(q, k.repeat_interleave(4, 1), v.repeat_interleave(4, 1), True, 0.25)
    np.testing.assert_array_equal(a, b)


def test_rows_equal_full():
    q, k, v = (_rand(s, t) for s, t in (((2, 4, 40, 16), 100), ((2, 2, 40, 16), 101),
                                        ((2, 2, 40, 16), 102)))
    full = oa.attention(q, k, v, True, 0.3)
    rows = np.array([[0, 0, 0], [1, 3, 39], [0, 2, 17], [1, 1, 5]])
    r = oa.attention_rows(q, k, v, rows, True, 0.3)
    for n, (b, h, i) in enumerate(rows):
        np.testing.assert_array_equal(r[n], full[b, h, i])


def test_independent_slices():
    """Head / batch slices computed alone equal slices of the full result."""
    q = _rand((2, 4, 32, 16), 110)
    k, v = _rand((2, 2, 32, 16), 111), _rand((2, 2, 32, 16), 112)
    full = oa.attention(q, k, v, True, 0.3)
    part = oa.attention(q[1:, 2:], k[1:, 1:], v[1:, 1:], True, 0.3)
    np.testing.assert_array_equal(part, full[1:, 2:])


def test_rejects_bad_shapes():
    q = np.zeros((1, 3, 4, 4))
    k = np.zeros((1, 2, 4, 4))
    with pytest.raises(ValueError):
        oa.attention(q, k, k)
