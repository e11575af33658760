"""Multi-rank head sharding on CPU (gloo, world_size 2): the shard arithmetic,
the per-head seeded inputs of each rank, the optional O all-gather and the
max-over-ranks timing reduction.  The per-shard attention here is the CPU
oracle (test infrastructure) standing in for the GPU kernel, which is covered
by the -m gpu head-shard test."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2511_02132_b200 import dist as pdist


def test_shard_heads_partition():
    for Hq, Hkv, G in ((128, 128, 8), (64, 8, 4), (64, 8, 8), (32, 32, 2)):
        shards = [pdist.shard_heads(Hq, Hkv, r, G) for r in range(G)]
        assert [s.q_lo for s in shards] == [r * Hq // G for r in range(G)]
        assert shards[-1].q_hi == Hq and shards[-1].kv_hi == Hkv
        for s in shards:  # whole GQA groups stay together
            assert s.q_lo == s.kv_lo * (Hq // Hkv) and s.q_hi == s.kv_hi * (Hq // Hkv)
    with pytest.raises(ValueError):
        pdist.shard_heads(64, 8, 0, 3)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    try:
        from oracle import attn as oa
        from paper_2511_02132_b200 import synth

        r, w, _ = pdist.init(backend="gloo")
        B, Hq, Hkv, N, d = 2, 8, 4, 64, 16
        sh = pdist.shard_heads(Hq, Hkv, r, w)
        qs, ks, vs = synth.make_qkv(B, sh.hq, sh.hkv, N, d, base=5, q_head_offset=sh.q_lo, kv_head_offset=sh.kv_lo)
        o_local = torch.from_numpy(oa.attention(qs, ks, vs, causal=True, scale=0.25)).float()
        full = pdist.all_gather_heads(o_local, w)
        t = pdist.max_over_ranks(float(r + 1))
        if r == 0:
            qf, kf, vf = synth.make_qkv(B, Hq, Hkv, N, d, base=5)
            ref = torch.from_numpy(oa.attention(qf, kf, vf, causal=True, scale=0.25)).float()
            q.put((torch.equal(full, ref), t))
        torch.distributed.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put(repr(e))


def test_two_rank_gloo_shard_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=240)
    assert res == (True, 2.0), res
