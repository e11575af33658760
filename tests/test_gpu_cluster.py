"""NEXT-4: CTA-pair clusters with TMA multicast of K/V (ATTN_CLUSTER_MULTICAST).

The pair streams one K/V sequence for two work units of the same head, so the
result must be exactly the plain path's: parity against the fp64 oracle on
small shapes, bit-identity with the non-cluster kernel at full size, and the
on-device trace shows every unit once with both units of a cluster unit on the
same die (a cluster is two SMs of one GPC).
"""
import collections
import math

import numpy as np
import pytest
import torch

from oracle import attn as oa
from paper_2511_02132_b200 import (attn_fwd, attn_fwd_lse, attn_set_schedule_trace, attn_topology, decode_trace,
                                   synth, trace_buffer)

from test_gpu_parity import MAPS, SMALL, _check

pytestmark = pytest.mark.gpu


def _run(q, k, v, causal, mapping, cluster):
    o = torch.full_like(q, float("nan"))
    attn_fwd(q, k, v, o, causal=causal, mapping=mapping, cluster=cluster)
    torch.cuda.synchronize()
    return o


def _same(a, b):
    return torch.equal(a.view(torch.int16), b.view(torch.int16))


@pytest.mark.parametrize("B,Hq,Hkv,N,d,causal", SMALL)
def test_cluster_small_parity_all_mappings(B, Hq, Hkv, N, d, causal):
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=1, device="cuda")
    ref = oa.attention(q.cpu(), k.cpu(), v.cpu(), causal=causal, scale=1.0 / math.sqrt(d))
    plain = _run(q, k, v, causal, "swizzled_head_first", False)
    for m in MAPS:
        o = _run(q, k, v, causal, m, True)
        _check(o, ref, f"cluster {m} {B}x{Hq}/{Hkv}x{N}x{d} causal={causal}")
        assert _same(o, plain), f"cluster {m} differs bitwise from the plain path"


@pytest.mark.parametrize("B,Hq,Hkv,N,d,causal", [
    (1, 32, 32, 8192, 128, False),    # C2
    (1, 16, 16, 32768, 128, True),    # C3 sequence length, fewer heads
    (2, 64, 8, 16384, 128, True),     # C4
    (1, 8, 8, 8000, 56, True),        # d = 56, ragged N
])
def test_cluster_full_size_bitexact(B, Hq, Hkv, N, d, causal):
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=5, device="cuda")
    plain = _run(q, k, v, causal, "block_first", False)
    for m in ("block_first", "swizzled_head_first"):
        o = _run(q, k, v, causal, m, True)
        assert not torch.isnan(o.float()).any(), "unwritten output elements"
        assert _same(o, plain)


def test_cluster_lse_bitexact():
    q, k, v = synth.make_qkv(1, 4, 2, 1000, 128, base=6, device="cuda")
    o0, l0 = attn_fwd_lse(q, k, v, causal=True)
    o1, l1 = attn_fwd_lse(q, k, v, causal=True, cluster=True)
    torch.cuda.synchronize()
    assert _same(o0, o1) and torch.equal(l0, l1)


@pytest.mark.parametrize("Hkv", [16, 4])   # MHA: adjacent-unit pairs; GQA 4: head pairs
@pytest.mark.parametrize("mapping", ["block_first", "swizzled_head_first"])
def test_cluster_trace_pairs_share_a_die(mapping, Hkv):
    B, Hq, N, d = 2, 16, 2304, 128   # U = 9 units per head: MHA's last cluster unit has one unit
    U = (N + 255) // 256
    buf = trace_buffer(B * Hq * U)
    attn_set_schedule_trace(0, buf)
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=3, device="cuda")
    attn_fwd(q, k, v, causal=True, mapping=mapping, cluster=True)
    torch.cuda.synchronize()
    attn_set_schedule_trace(0, None)
    tr = decode_trace(buf)
    ids = tr[:, 0] * Hq * U + tr[:, 1] * U + tr[:, 2]
    assert torch.equal(ids, torch.arange(B * Hq * U, dtype=ids.dtype))  # every unit exactly once
    t = attn_topology(0)
    pair_heads = (Hq // Hkv) % 2 == 0
    by_cu = collections.defaultdict(list)
    for b, h, u, sm, dom, qi, st, seq in tr.tolist():
        assert dom == t["domain_of_smid"][sm]
        key = (b, h // 2, u) if pair_heads else (b, h, u // 2)
        by_cu[key].append((h if pair_heads else u, sm, dom, seq))
    peer = {}
    for key, recs in by_cu.items():
        if len(recs) == 1:
            assert not pair_heads and recs[0][0] == U - 1   # only MHA's odd last unit runs alone
            continue
        (r0, sm0, d0, s0), (r1, sm1, d1, s1) = sorted(recs)
        assert (r0 % 2, r1 % 2) == (0, 1) and sm0 != sm1 and d0 == d1
        assert s0 == s1                  # both CTAs consumed the same scheduler entry
        # a cluster keeps its two SMs for the whole launch
        assert peer.setdefault(sm0, sm1) == sm1
