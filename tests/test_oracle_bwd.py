"""Pins for the fp64 backward oracle (eq:ba) -- CPU only.

  finite differences  d/dx sum(dO * attention(x)) from the FORWARD oracle,
                      independent of the backward code
  library routine     torch float64 autograd of softmax(QK^T*scale+mask) V
  reduction           GQA gradients == MHA gradients of repeat_interleaved K/V,
                      summed over each group's heads
  closed form         LSE of a row with identical scores = log(n_visible)
"""
import math

import numpy as np
import pytest
import torch

from oracle import attn as oa


def _rand(shape, seed):
    return torch.randn(shape, generator=torch.Generator().manual_seed(seed), dtype=torch.float64)


@pytest.mark.parametrize("causal", [False, True])
def test_finite_differences(causal):
    B, Hq, Hkv, N, d = 1, 2, 1, 6, 4
    q, k, v, do = _rand((B, Hq, N, d), 1), _rand((B, Hkv, N, d), 2), _rand((B, Hkv, N, d), 3), _rand((B, Hq, N, d), 4)
    dq, dk, dv, _ = oa.attention_bwd(q, k, v, do, causal=causal, scale=0.7)
    L = lambda q_, k_, v_: float((oa.attention(q_, k_, v_, causal=causal, scale=0.7) * do.numpy()).sum())
    eps = 1e-6
    for name, x, grad in (("q", q, dq), ("k", k, dk), ("v", v, dv)):
        for idx in [(0, 0, 0, 0), (0, x.shape[1] - 1, N - 1, d - 1), (0, 0, N // 2, 1)]:
            xp, xm = x.clone(), x.clone()
            xp[idx] += eps
            xm[idx] -= eps
            args_p = {"q": (xp, k, v), "k": (q, xp, v), "v": (q, k, xp)}[name]
            args_m = {"q": (xm, k, v), "k": (q, xm, v), "v": (q, k, xm)}[name]
            fd = (L(*args_p) - L(*args_m)) / (2 * eps)
            assert grad[idx] == pytest.approx(fd, abs=1e-6, rel=1e-6), (name, idx)


@pytest.mark.parametrize("B,Hq,Hkv,N,d,causal", [(1, 2, 2, 17, 8, False), (2, 4, 2, 33, 16, True),
                                                 (1, 4, 1, 64, 32, True)])
def test_matches_torch_autograd(B, Hq, Hkv, N, d, causal):
    q, k, v, do = _rand((B, Hq, N, d), 5), _rand((B, Hkv, N, d), 6), _rand((B, Hkv, N, d), 7), _rand((B, Hq, N, d), 8)
    scale = 1 / math.sqrt(d)
    qt, kt, vt = (t.clone().requires_grad_(True) for t in (q, k, v))
    G = Hq // Hkv
    s = torch.einsum("bhid,bhjd->bhij", qt, kt.repeat_interleave(G, 1)) * scale
    if causal:
        s = s.masked_fill(torch.triu(torch.ones(N, N, dtype=torch.bool), 1), float("-inf"))
    o = torch.einsum("bhij,bhjd->bhid", torch.softmax(s, -1), vt.repeat_interleave(G, 1))
    (o * do).sum().backward()
    dq, dk, dv, lse = oa.attention_bwd(q, k, v, do, causal=causal, scale=scale)
    np.testing.assert_allclose(dq, qt.grad.numpy(), atol=1e-12, rtol=0)
    np.testing.assert_allclose(dk, kt.grad.numpy(), atol=1e-12, rtol=0)
    np.testing.assert_allclose(dv, vt.grad.numpy(), atol=1e-12, rtol=0)
    np.testing.assert_allclose(lse, torch.logsumexp(s, -1).detach().numpy(), atol=1e-12, rtol=0)


def test_gqa_equals_mha_summed():
    q, k, v, do = _rand((1, 4, 20, 8), 9), _rand((1, 2, 20, 8), 10), _rand((1, 2, 20, 8), 11), _rand((1, 4, 20, 8), 12)
    dq, dk, dv, _ = oa.attention_bwd(q, k, v, do, causal=True, scale=0.3)
    dq2, dk2, dv2, _ = oa.attention_bwd(q, k.repeat_interleave(2, 1), v.repeat_interleave(2, 1), do, causal=True,
                                        scale=0.3)
    np.testing.assert_allclose(dq, dq2, atol=1e-13, rtol=0)
    np.testing.assert_allclose(dk, dk2.reshape(1, 2, 2, 20, 8).sum(2), atol=1e-13, rtol=0)
    np.testing.assert_allclose(dv, dv2.reshape(1, 2, 2, 20, 8).sum(2), atol=1e-13, rtol=0)


def test_lse_closed_form_and_zero_dv_for_unseen_keys():
    N, d = 9, 4
    q = torch.zeros((1, 1, N, d), dtype=torch.float64)
    k, v, do = _rand((1, 1, N, d), 13), _rand((1, 1, N, d), 14), _rand((1, 1, N, d), 15)
    _, _, dv, lse = oa.attention_bwd(q, k, v, do, causal=True, scale=1.0)
    np.testing.assert_allclose(lse[0, 0], np.log(np.arange(1, N + 1)), atol=1e-15, rtol=0)  # uniform rows
    # key N-1 is seen only by query N-1 with weight 1/N: dv[N-1] = dO[N-1]/N
    np.testing.assert_allclose(dv[0, 0, N - 1], do[0, 0, N - 1].numpy() / N, atol=1e-15, rtol=0)


@pytest.mark.parametrize("causal", [False, True])
def test_rows_variant_matches_full_oracle(causal):
    """attention_bwd_rows (numpy, chunked statistics: the full-size backward
    parity test's checker) equals the pinned C oracle's gradients row by row,
    GQA group sums included, with a chunk that splits the rows unevenly."""
    from paper_2511_02132_b200 import synth

    q, k, v = synth.make_qkv(2, 4, 2, 300, 24, base=5, device="cpu")
    do = synth.make_tensor("q", 2, 4, 300, 24, base=6, device="cpu")
    rq, rk, rv, _ = oa.attention_bwd(q, k, v, do, causal=causal)
    qrows, krows = [0, 1, 127, 128, 299], [0, 5, 200, 299]
    for b, g in ((0, 0), (1, 1)):
        dq, dk, dv = oa.attention_bwd_rows(q, k, v, do, b, g, qrows, krows, causal=causal, chunk=64)
        np.testing.assert_allclose(dq, rq[b, 2 * g:2 * g + 2][:, qrows], atol=1e-12, rtol=0)
        np.testing.assert_allclose(dk, rk[b, g, krows], atol=1e-12, rtol=0)
        np.testing.assert_allclose(dv, rv[b, g, krows], atol=1e-12, rtol=0)


def test_rows_variant_column_sum_identities():
    """Closed forms of eq:ba that hold at any size (each row of P sums to 1 and
    sum_j P_ij dP_ij = D_i): sum_j dv_j = sum_i dO_i and sum_j dk_j = 0."""
    from paper_2511_02132_b200 import synth

    N = 96
    q, k, v = synth.make_qkv(1, 1, 1, N, 16, base=7, device="cpu")
    do = synth.make_tensor("q", 1, 1, N, 16, base=8, device="cpu")
    _, dk, dv = oa.attention_bwd_rows(q, k, v, do, 0, 0, [0], np.arange(N), causal=True, chunk=40)
    np.testing.assert_allclose(dv.sum(0), do[0, 0].double().numpy().sum(0), atol=1e-11, rtol=0)
    np.testing.assert_allclose(dk.sum(0), 0.0, atol=1e-11)
