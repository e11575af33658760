"""The analytic L2 model (scripts/l2model.py, NEXT-4) pinned on cases whose
traffic is known in closed form, independent of any measurement."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "scripts"))
import l2model  # noqa: E402

BIG = 1 << 40   # an L2 that never evicts


def _compulsory(B, Hq, Hkv, N, d):
    """Q read, K and V read once, O written once (bytes)."""
    return 2 * B * N * d * (2 * Hq + 2 * Hkv)


@pytest.mark.parametrize("mapping", ["block_first", "head_first", "swizzled_head_first", "swizzled_block_first"])
@pytest.mark.parametrize("causal", [False, True])
def test_infinite_cache_is_compulsory_traffic(mapping, causal):
    B, Hq, Hkv, N, d = 2, 8, 4, 1024, 128
    r = l2model.simulate(B, Hq, Hkv, N, d, causal, mapping, (3, 2), l2_bytes=BIG)
    assert r["dram_gb"] * 1e9 == pytest.approx(_compulsory(B, Hq, Hkv, N, d))
    assert r["q_gb"] * 1e9 == B * Hq * N * d * 2 and r["o_gb"] * 1e9 == B * Hq * N * d * 2


def test_kv_requests_count_every_unit_block():
    # non-causal: every unit streams all nblk blocks; causal: unit u streams 2u+2
    B, Hq, Hkv, N, d = 1, 4, 4, 1024, 64
    nblk, U = N // 128, N // 256
    blk = 2 * 128 * d * 2
    r = l2model.simulate(B, Hq, Hkv, N, d, False, "head_first", (2,), l2_bytes=BIG)
    assert r["kv_l2_gb"] * 1e9 == B * Hq * U * nblk * blk
    r = l2model.simulate(B, Hq, Hkv, N, d, True, "head_first", (2,), l2_bytes=BIG)
    assert r["kv_l2_gb"] * 1e9 == B * Hq * sum(2 * u + 2 for u in range(U)) * blk


def test_single_worker_reuse_by_hand():
    # one worker, one head, 4 blocks: unit 0 misses its 4 blocks, unit 1 hits them
    r = l2model.simulate(1, 1, 1, 512, 64, False, "head_first", (1,), l2_bytes=BIG)
    assert r["kv_hit_rate_pct"] == pytest.approx(50.0)


def test_cache_too_small_for_one_block_never_hits():
    # capacity of one entry and O lines in between: no K/V reuse survives
    r = l2model.simulate(1, 2, 2, 1024, 64, False, "block_first", (1,), l2_bytes=1)
    assert r["kv_hit_rate_pct"] == 0.0


def test_head_first_beats_block_first_when_heads_exceed_l2():
    # 256 heads (more than the 148 CTAs, so block-first runs one CTA per head)
    # x 1 MB of K/V >> an 8 MB L2: block-first's order finds no reuse
    B, Hq, Hkv, N, d = 1, 256, 256, 2048, 128
    bf = l2model.simulate(B, Hq, Hkv, N, d, False, "block_first", (74, 74), l2_bytes=8 << 20)
    hf = l2model.simulate(B, Hq, Hkv, N, d, False, "head_first", (74, 74), l2_bytes=8 << 20)
    # head-first: a head's 8 units run side by side, one miss per block -> 7/8
    assert hf["kv_hit_rate_pct"] == pytest.approx(87.5, abs=1.0)
    assert bf["kv_hit_rate_pct"] == 0.0
    assert bf["dram_gb"] > 4 * hf["dram_gb"]


def test_cluster_pairs_halve_kv_requests():
    # MHA non-causal, even unit count: each pair streams a block once for two units
    B, Hq, Hkv, N, d = 1, 8, 8, 2048, 128
    plain = l2model.simulate(B, Hq, Hkv, N, d, False, "head_first", (8, 8), l2_bytes=BIG)
    pairs = l2model.simulate(B, Hq, Hkv, N, d, False, "head_first", (8, 8), l2_bytes=BIG, cluster=True)
    assert pairs["kv_l2_gb"] == pytest.approx(plain["kv_l2_gb"] / 2)
    assert pairs["dram_gb"] == pytest.approx(plain["dram_gb"])
    # GQA head pairs likewise
    plain = l2model.simulate(B, 8, 2, N, d, True, "block_first", (8, 8), l2_bytes=BIG)
    pairs = l2model.simulate(B, 8, 2, N, d, True, "block_first", (8, 8), l2_bytes=BIG, cluster=True)
    assert pairs["kv_l2_gb"] == pytest.approx(plain["kv_l2_gb"] / 2)


def test_random_policy_matches_lru_when_everything_fits():
    r1 = l2model.simulate(1, 4, 2, 1024, 64, True, "swizzled_head_first", (2, 2), l2_bytes=BIG, policy="random")
    r2 = l2model.simulate(1, 4, 2, 1024, 64, True, "swizzled_head_first", (2, 2), l2_bytes=BIG)
    assert r1["dram_gb"] == r2["dram_gb"]
