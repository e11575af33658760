"""Pins for the mapping reference (oracle/mapping.py) -- CPU only.

Pinned against SPEC.md's printed worked examples (tests/golden/
spec_mapping_pins.json, each with its citation), brute-force bijectivity,
the co-location invariants of P:259-270 / S:202-206, and the derived B200
per-die examples of DESIGN.md R8.
"""
import json
import os
import random

import pytest

from oracle import mapping as om

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_mapping_pins.json")))


@pytest.mark.parametrize("ex", GOLD["grid_size"])
def test_grid_size(ex):
    assert om.grid_size(ex["B"], ex["Hq"], ex["N"], ex["block_m"]) == ex["expect"]


@pytest.mark.parametrize("ex", GOLD["acc_of"])
def test_acc_of(ex):
    assert list(om.acc_of(ex["Hq"], ex["Hkv"], ex["b"], ex["h"])) == ex["expect"]


@pytest.mark.parametrize("ex", GOLD["validate"])
def test_validate(ex):
    args = (ex["B"], ex["Hq"], ex["Hkv"], ex["N"], ex["block_m"])
    if ex["expect"] == "error":
        with pytest.raises(ValueError):
            om.validate(*args)
    else:
        got = om.validate(*args)
        for key, val in ex["expect"].items():
            assert got[key] == val


@pytest.mark.parametrize("ex", GOLD["hardware_dispatch"])
def test_hardware_dispatch(ex):
    assert om.hardware_dispatch(ex["wgid"], ex["num_xcd"], ex["chunk"]) == ex["expect"]


@pytest.mark.parametrize("ex", GOLD["swizzle_chiplet"])
def test_swizzle_chiplet(ex):
    assert om.swizzle_chiplet(ex["wgid"], ex["grid"], ex["num_xcd"]) == ex["expect"]


def test_swizzle_chiplet_is_permutation():
    for grid, X in ((16, 4), (64, 8), (1024, 8)):
        assert sorted(om.swizzle_chiplet(w, grid, X) for w in range(grid)) == list(range(grid))


@pytest.mark.parametrize("ex", GOLD["map_tile"])
def test_map_tile(ex):
    t = om.map_tile_mi300(ex["strategy"], ex["wid"], ex["B"], ex["H"], ex["nblk"], ex["X"])
    assert list(t) == ex["expect_tile"]
    if "expect_xcd" in ex:
        assert om.hardware_dispatch(ex["wid"], ex["X"]) == ex["expect_xcd"]


@pytest.mark.parametrize("BATCH,H,nblk,X", [(1, 8, 128, 4), (2, 8, 16, 4), (4, 16, 8, 8), (3, 8, 5, 2)])
def test_fig7_reconstruction_equals_closed_form(BATCH, H, nblk, X):
    grid = BATCH * H * nblk
    a = [om.fig7_swizzled_head_first(w, BATCH, H, nblk, X) for w in range(grid)]
    b = [om.map_tile_mi300("swizzled_head_first", w, BATCH, H, nblk, X) for w in range(grid)]
    assert a == b
    assert len(set(a)) == grid  # bijection
    # co-location: every (b, h) lands on exactly one XCD under chunk-1 dispatch
    where = {}
    for w, (bb, h, _k) in enumerate(a):
        where.setdefault((bb, h), set()).add(om.hardware_dispatch(w, X))
    assert all(len(s) == 1 for s in where.values())


def test_literal_fig7_wid_div_batch_is_not_bijective():
    """R6: P:290's literal wid_per_batch = wid // BATCH misses tiles for BATCH > 1."""
    BATCH, H, nblk, X = 2, 8, 4, 4
    hpx = H // X
    seen = set()
    for wid in range(BATCH * H * nblk):
        w = wid // BATCH
        head = (w % X) * hpx + (w // (X * nblk)) % hpx
        blk = (w % (X * nblk)) // X
        b = (wid // (nblk * H)) % BATCH
        seen.add((b, head, blk))
    assert len(seen) < BATCH * H * nblk


def test_attention_flops_and_footprint_pins():
    for ex in GOLD["attention_flops"]:
        assert 4 * ex["B"] * ex["Hq"] * ex["N"] ** 2 * ex["d"] == ex["expect"]
    for ex in GOLD["kv_footprint_bytes"]:
        assert 2 * ex["N"] * ex["d"] * ex["elem_bytes"] == ex["expect"]


# ---------------------------------------------------------- B200 queues
def test_worked_examples_two_equal_dies():
    # MHA Z=1, H=4, nblk=3 (R8 worked example)
    bf = om.build_queues("block_first", 1, 4, 4, 3, [74, 74])
    assert bf == [[(0, 0, 0), (0, 1, 0), (0, 2, 0), (0, 3, 0), (0, 0, 1), (0, 1, 1), (0, 2, 1),
                   (0, 3, 1), (0, 0, 2), (0, 1, 2), (0, 2, 2), (0, 3, 2)]]
    hf = om.build_queues("head_first", 1, 4, 4, 3, [74, 74])
    assert hf[0][:4] == [(0, 0, 0), (0, 0, 1), (0, 0, 2), (0, 1, 0)]
    shf = om.build_queues("swizzled_head_first", 1, 4, 4, 3, [74, 74])
    assert shf[0] == [(0, h, k) for h in (0, 1) for k in range(3)]
    assert shf[1] == [(0, h, k) for h in (2, 3) for k in range(3)]
    # GQA Z=2, Hq=4, Hkv=2: per batch item, group 0 -> die 0, group 1 -> die 1 (Fig. 7: batch outermost)
    g = om.build_queues("swizzled_head_first", 2, 4, 2, 2, [74, 74])
    assert g[0] == [(b, h, k) for b in (0, 1) for h in (0, 1) for k in range(2)]
    assert g[1] == [(b, h, k) for b in (0, 1) for h in (2, 3) for k in range(2)]
    # odd ACC count: 3 heads on 2 dies -> 2 + 1 (rounded proportional cut)
    o = om.build_queues("swizzled_head_first", 1, 3, 3, 4, [74, 74])
    assert [len(q) for q in o] == [8, 4]
    # fewer ACCs per batch than dies but enough overall: Hkv=1, B=2 -> one batch per die
    m = om.build_queues("swizzled_head_first", 2, 2, 1, 2, [74, 74])
    assert m[0] == [(0, h, k) for h in (0, 1) for k in range(2)]
    # fewer ACCs than dies: MQA Hkv=1, B=1 -> tile-granular split
    t = om.build_queues("swizzled_head_first", 1, 2, 1, 3, [74, 74])
    assert [len(q) for q in t] == [3, 3]


def test_shf_equal_dies_matches_fig7_assignment():
    """With X equal dies the per-die queues are exactly the XCD queues Fig. 7 +
    chunk-1 dispatch produce (S:181-189 build_assignment)."""
    for BATCH, H, nblk, X in ((1, 8, 16, 4), (2, 8, 4, 2), (3, 16, 5, 8)):
        q = om.build_queues("swizzled_head_first", BATCH, H, H, nblk, [10] * X)
        ref = [[] for _ in range(X)]
        for w in range(BATCH * H * nblk):
            ref[om.hardware_dispatch(w, X)].append(om.fig7_swizzled_head_first(w, BATCH, H, nblk, X))
        assert q == ref


def test_random_configs_bijective_and_colocated():
    rng = random.Random(1234)
    for _ in range(250):
        Hkv = rng.choice([1, 2, 3, 4, 8, 16])
        Hq = Hkv * rng.choice([1, 2, 4])
        B = rng.randint(1, 4)
        nblk = rng.randint(1, 9)
        D = rng.randint(1, 4)
        sizes = [rng.randint(60, 80) for _ in range(D)]
        for m in om.MAPPINGS:
            qs = om.build_queues(m, B, Hq, Hkv, nblk, sizes)
            assert om.is_bijection(qs, B, Hq, nblk), (m, B, Hq, Hkv, nblk, sizes)
        qs = om.build_queues("swizzled_head_first", B, Hq, Hkv, nblk, sizes)
        doms = om.acc_domains(qs, Hq, Hkv)
        if B * Hkv >= D:
            assert all(len(s) == 1 for s in doms.values())  # 100% co-location
        else:
            assert sum(len(s) > 1 for s in doms.values()) <= D - 1
        # each queue is head-major ordered (one ACC at a time)
        for q in qs:
            key = [(b, h, k) for (b, h, k) in q]
            assert key == sorted(key)


def test_swizzled_block_first_examples():
    """groups with g mod X == x on XCD x, block-major inside; with
    #groups == #dies every ACC sits on one die."""
    q = om.build_queues("swizzled_block_first", 1, 8, 2, 3, [74, 74])   # GQA, 2 groups of 4
    assert q[0] == [(0, h, k) for k in range(3) for h in range(4)]
    assert q[1] == [(0, h, k) for k in range(3) for h in range(4, 8)]
    mha = om.build_queues("swizzled_block_first", 1, 4, 4, 2, [74, 74])
    assert mha[0] == [(0, 0, 0), (0, 2, 0), (0, 0, 1), (0, 2, 1)]
    assert mha[1] == [(0, 1, 0), (0, 3, 0), (0, 1, 1), (0, 3, 1)]
    for Hkv in (2, 8):
        qs = om.build_queues("swizzled_block_first", 2, 64, Hkv, 4, [74, 74])
        assert all(len(s) == 1 for s in om.acc_domains(qs, 64, Hkv).values())
    assert (om.build_queues("swizzled_block_first", 2, 8, 2, 3, [148])
            == om.build_queues("block_first", 2, 8, 2, 3, [148]))


def test_single_domain_degenerates_to_head_first():
    """S:189 / S:206: with one die SHF == HF."""
    for B, Hq, Hkv, nblk in ((1, 4, 4, 3), (2, 8, 2, 5)):
        assert (om.build_queues("swizzled_head_first", B, Hq, Hkv, nblk, [148])
                == om.build_queues("head_first", B, Hq, Hkv, nblk, [148]))


def test_descending_worked_example():
    """DESIGN.md R19 written out by hand (not recomputed): Z=1, Hq=Hkv=4, three
    query blocks, two equal dies.  Descending visits each head's blocks
    last-first and changes nothing else -- same queues, same heads per die."""
    shf = om.build_queues(om.SWIZZLED_HEAD_FIRST, 1, 4, 4, 3, [74, 74])
    assert om.descending(shf, 3) == [
        [(0, 0, 2), (0, 0, 1), (0, 0, 0), (0, 1, 2), (0, 1, 1), (0, 1, 0)],
        [(0, 2, 2), (0, 2, 1), (0, 2, 0), (0, 3, 2), (0, 3, 1), (0, 3, 0)],
    ]
    bf = om.build_queues(om.BLOCK_FIRST, 1, 2, 2, 3, [74, 74])
    assert om.descending(bf, 3) == [[(0, 0, 2), (0, 1, 2), (0, 0, 1), (0, 1, 1), (0, 0, 0), (0, 1, 0)]]
    # GQA (Hq=4, Hkv=2), two batch items, two blocks: die 1 keeps group 1 (heads 2, 3) of every batch item
    g = om.build_queues(om.SWIZZLED_HEAD_FIRST, 2, 4, 2, 2, [74, 74])
    assert om.descending(g, 2)[1] == [(0, 2, 1), (0, 2, 0), (0, 3, 1), (0, 3, 0),
                                      (1, 2, 1), (1, 2, 0), (1, 3, 1), (1, 3, 0)]


def test_alternate_worked_example():
    """DESIGN.md R22 by hand: queue 0 ascending, queue 1 descending; a single
    queue (head-first) is unchanged."""
    shf = om.build_queues(om.SWIZZLED_HEAD_FIRST, 1, 4, 4, 3, [74, 74])
    assert om.alternate(shf, 3) == [
        [(0, 0, 0), (0, 0, 1), (0, 0, 2), (0, 1, 0), (0, 1, 1), (0, 1, 2)],
        [(0, 2, 2), (0, 2, 1), (0, 2, 0), (0, 3, 2), (0, 3, 1), (0, 3, 0)],
    ]
    hf = om.build_queues(om.HEAD_FIRST, 1, 2, 2, 2, [74, 74])
    assert om.alternate(hf, 2) == [[(0, 0, 0), (0, 0, 1), (0, 1, 0), (0, 1, 1)]]


def test_shared_acc_worked_example():
    """DESIGN.md R23 written out by hand: with its ACCs shared, swizzled
    head-first runs over ONE capacity domain, which S:189 / S:206 define to be
    head-first -- Z=1, Hq=Hkv=2, three blocks, dies of 2 and 1 SMs: one queue
    (0,0,0) (0,0,1) (0,0,2) (0,1,0) (0,1,1) (0,1,2)."""
    q = om.build_queues(om.SWIZZLED_HEAD_FIRST, 1, 2, 2, 3, [2, 1], shared_acc=True)
    assert q == [[(0, 0, 0), (0, 0, 1), (0, 0, 2), (0, 1, 0), (0, 1, 1), (0, 1, 2)]]
    # GQA: heads of a group stay together in the one queue
    q = om.build_queues(om.SWIZZLED_HEAD_FIRST, 1, 4, 2, 2, [74, 74], shared_acc=True)
    assert q == [[(0, 0, 0), (0, 0, 1), (0, 1, 0), (0, 1, 1), (0, 2, 0), (0, 2, 1), (0, 3, 0), (0, 3, 1)]]
    assert q == om.build_queues(om.HEAD_FIRST, 1, 4, 2, 2, [74, 74])
    # the flag is an SHF grain only: the other mappings ignore it
    assert (om.build_queues(om.BLOCK_FIRST, 1, 2, 2, 3, [2, 1], shared_acc=True)
            == om.build_queues(om.BLOCK_FIRST, 1, 2, 2, 3, [2, 1]))


def test_shf_acc_rule_closed_form():
    """R23's threshold by hand on B200's 126 MiB L2 (132,120,576 bytes), two
    dies, d = 128: K+V of one head = 512*N bytes; shared iff 2*512*N > 66,060,288
    i.e. N > 64,512 -> 32K and 64,512 per-die, 64K and 128K shared."""
    l2 = 132120576
    assert not om.shf_acc_shared(2, 32768, 128, l2)
    assert not om.shf_acc_shared(2, 64512, 128, l2)
    assert om.shf_acc_shared(2, 64513, 128, l2)
    assert om.shf_acc_shared(2, 65536, 128, l2) and om.shf_acc_shared(2, 131072, 128, l2)
    assert not om.shf_acc_shared(1, 131072, 128, l2)  # one die: nothing to share
    assert not om.shf_acc_shared(2, 131072, 128, 0)   # unknown L2: the paper's grain
