"""CUDA-graph capture of the C-ABI calls (the task's "streams and graphs"
execution model): attn_fwd (plain and as CTA-pair clusters, every mapping) and
attn_bwd captured once in a torch.cuda.CUDAGraph and replayed several times
must give exactly the eager results -- the persistent grid's queue counters
re-zero themselves at the end of every launch (include/attn_numa.h,
"Concurrency"), so a replay needs no host-side reset.  Forward parity with the
fp64 oracle (eq:fa) is covered elsewhere; here the eager
call is the reference, bit for bit (forward and the deterministic backward)."""
import math

import pytest
import torch

from paper_2511_02132_b200 import attn_bwd, attn_fwd, attn_fwd_lse, synth

pytestmark = pytest.mark.gpu

MAPPINGS = ("block_first", "head_first", "swizzled_head_first", "swizzled_block_first")


def _same(a, b):
    return torch.equal(a.view(torch.int16), b.view(torch.int16))


@pytest.mark.parametrize("shape", [(1, 4, 4, 1000, 128, True), (2, 4, 2, 640, 128, False),
                                   (1, 4, 4, 777, 56, True)])
@pytest.mark.parametrize("cluster", [False, True])
def test_fwd_graph_replay_bit_identical(shape, cluster):
    B, Hq, Hkv, N, d, causal = shape
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=21, device="cuda")
    scale = 1.0 / math.sqrt(d)
    refs = [attn_fwd(q, k, v, causal=causal, scale=scale, mapping=m, cluster=cluster) for m in MAPPINGS]
    torch.cuda.synchronize()
    outs = [torch.empty_like(q) for _ in MAPPINGS]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for m, o in zip(MAPPINGS, outs):
            attn_fwd(q, k, v, o, causal=causal, scale=scale, mapping=m, cluster=cluster)
    for _ in range(3):
        for o in outs:
            o.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        for m, o, r in zip(MAPPINGS, outs, refs):
            assert _same(o, r), f"graph replay differs from eager ({m}, cluster={cluster})"
    assert all(_same(r, refs[0]) for r in refs)  # mappings agree bit for bit


@pytest.mark.parametrize("shape", [(1, 2, 2, 384, 128, True), (1, 4, 2, 300, 64, False)])
def test_bwd_graph_replay_bit_identical(shape):
    B, Hq, Hkv, N, d, causal = shape
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=22, device="cuda")
    scale = 1.0 / math.sqrt(d)
    o, lse = attn_fwd_lse(q, k, v, causal=causal, scale=scale)
    do = synth.make_tensor("q", B, Hq, N, d, base=23, device="cuda")
    ref = attn_bwd(q, k, v, o, do, lse, causal=causal, scale=scale, deterministic=True)
    torch.cuda.synchronize()
    dq, dk, dv = (torch.empty_like(t) for t in (q, k, v))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        attn_bwd(q, k, v, o, do, lse, causal=causal, scale=scale, dq=dq, dk=dk, dv=dv, deterministic=True)
    for _ in range(3):
        for t in (dq, dk, dv):
            t.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        for name, got, r in zip(("dq", "dk", "dv"), (dq, dk, dv), ref):
            assert _same(got, r), f"graph replay {name} differs from eager"


def test_bwd_single_pass_graph_replay():
    """d <= 64 single-pass backward (dq reduce-added by TMA into an fp32
    workspace allocated per call in stream order): dk / dv bit-identical to
    eager, dq equal up to the fp32 summation order (<= 1 bf16 ulp)."""
    B, Hq, Hkv, N, d, causal = 1, 4, 4, 512, 56, True
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=24, device="cuda")
    scale = 1.0 / math.sqrt(d)
    o, lse = attn_fwd_lse(q, k, v, causal=causal, scale=scale)
    do = synth.make_tensor("q", B, Hq, N, d, base=25, device="cuda")
    ref = attn_bwd(q, k, v, o, do, lse, causal=causal, scale=scale)
    torch.cuda.synchronize()
    dq, dk, dv = (torch.empty_like(t) for t in (q, k, v))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        attn_bwd(q, k, v, o, do, lse, causal=causal, scale=scale, dq=dq, dk=dk, dv=dv)
    for _ in range(3):
        for t in (dq, dk, dv):
            t.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        assert _same(dk, ref[1]) and _same(dv, ref[2])
        diff = (dq.float() - ref[0].float()).abs()
        assert bool(torch.isfinite(dq.float()).all())
        assert bool((diff <= 2.0 ** -7 * ref[0].float().abs() + 1e-6).all())
