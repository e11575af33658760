"""Replicated output stored by the forward's epilogue (C-ABI attn_fwd_replicated,
SURVEY.md §8(e) fused alternative to the all-gather of O; heads are
independent).

CPU (gloo, world 2): the PeerOutput / replicated_fwd plumbing with a fake
binding (handle exchange order, own buffer first, head offsets, peer unmaps).
GPU: one process with several local destinations (bit-identical to attn_fwd
on the shard, other heads untouched, validation), and two processes sharing
cuda:0 whose kernels write into each other's buffers through CUDA IPC."""
import os
import socket
import struct

import pytest
import torch
import torch.multiprocessing as mp

from paper_2511_02132_b200 import dist as pdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _FakeApi:
    """Stands in for the C-ABI: a handle is (rank, address) packed in 72 bytes."""

    def __init__(self, rank):
        self.rank, self.opened, self.closed, self.calls = rank, [], [], []

    def ipc_get_handle(self, t):
        return struct.pack("<qq", self.rank, t.data_ptr()) + bytes(56)

    def ipc_open(self, rec):
        r, addr = struct.unpack("<qq", rec[:16])
        assert r != self.rank, "a rank must not open its own handle"
        self.opened.append(r)
        return 1_000_000 * (r + 1)  # fake mapped address of rank r's buffer

    def ipc_close(self, p):
        self.closed.append(p)

    def attn_fwd_replicated(self, q, k, v, dsts, Hq_out, head_offset, **kw):
        self.calls.append((list(dsts), Hq_out, head_offset))


def _plumbing_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    try:
        r, w, _ = pdist.init(backend="gloo")
        fake = _FakeApi(r)
        B, Hq, Hkv, N, d = 1, 8, 4, 16, 8
        sh = pdist.shard_heads(Hq, Hkv, r, w)
        po = pdist.PeerOutput((B, Hq, N, d), r, w, "cpu", api=fake)
        q = torch.zeros(B, sh.hq, N, d)
        pdist.replicated_fwd(q, q, q, sh, po, api=fake, sync=False)
        dsts, Hq_out, off = fake.calls[0]
        own = po.local.data_ptr()
        ok = (po.ptrs[r] == own and dsts[0] == own and Hq_out == Hq and off == r * (Hq // w)
              and sorted(fake.opened) == [x for x in range(w) if x != r]
              and all(po.ptrs[x] == 1_000_000 * (x + 1) for x in range(w) if x != r)
              and sorted(dsts[1:]) == sorted(po.ptrs[x] for x in range(w) if x != r))
        po.close()
        ok = ok and sorted(fake.closed) == sorted(1_000_000 * (x + 1) for x in range(w) if x != r)
        out.put((r, ok))
        torch.distributed.destroy_process_group()
    except Exception as e:  # pragma: no cover
        out.put((rank, repr(e)))


def test_peer_output_plumbing_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_plumbing_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(2))
    for p in procs:
        p.join(timeout=240)
    assert res == {0: True, 1: True}, res


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("causal,d,N", [(False, 128, 512), (True, 128, 1000), (True, 56, 384)])
def test_replicated_local_destinations(causal, d, N):
    from paper_2511_02132_b200 import attn_fwd, attn_fwd_replicated, synth

    B, Hq_full, Hkv_full = 2, 8, 4
    sh = pdist.shard_heads(Hq_full, Hkv_full, 1, 2)  # second half of the heads
    q, k, v = synth.make_qkv(B, sh.hq, sh.hkv, N, d, base=21, q_head_offset=sh.q_lo, kv_head_offset=sh.kv_lo,
                             device="cuda")
    ref = attn_fwd(q, k, v, causal=causal)
    dsts = [torch.full((B, Hq_full, N, d), float("nan"), dtype=torch.bfloat16, device="cuda") for _ in range(3)]
    attn_fwd_replicated(q, k, v, dsts, Hq_full, sh.q_lo, causal=causal)
    torch.cuda.synchronize()
    for o in dsts:
        assert torch.equal(o[:, sh.q_lo:sh.q_hi].view(torch.int16), ref.view(torch.int16))
        assert torch.isnan(o[:, :sh.q_lo].float()).all()  # heads of the other rank untouched


@pytest.mark.gpu
def test_replicated_validation():
    from paper_2511_02132_b200 import AttnError, attn_fwd_replicated, synth

    q, k, v = synth.make_qkv(1, 2, 2, 256, 64, base=1, device="cuda")
    full = torch.empty((1, 4, 256, 64), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(AttnError):  # shard does not fit at this offset
        attn_fwd_replicated(q, k, v, [full], 4, 3)
    with pytest.raises(AttnError):  # destinations overlap
        attn_fwd_replicated(q, k, v, [full.data_ptr(), full.data_ptr() + 16], 4, 0)
    with pytest.raises(AttnError):  # destination overlaps an input
        attn_fwd_replicated(q, k, v, [q.data_ptr()], 4, 0)
    with pytest.raises(ValueError):
        attn_fwd_replicated(q, k, v, [], 4, 0)


def _ipc_worker(rank, world, port, causal, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK="0", ATTN_BENCH_SHARE_GPU="1")
    try:
        from paper_2511_02132_b200 import attn_fwd, synth

        r, w, local = pdist.init()
        torch.cuda.set_device(local)
        B, Hq, Hkv, N, d = 1, 8, 8, 768, 128
        sh = pdist.shard_heads(Hq, Hkv, r, w)
        q, k, v = synth.make_qkv(B, sh.hq, sh.hkv, N, d, base=33, q_head_offset=sh.q_lo, kv_head_offset=sh.kv_lo,
                                 device="cuda")
        po = pdist.PeerOutput((B, Hq, N, d), r, w, "cuda")
        po.local.fill_(float("nan"))
        torch.cuda.synchronize()
        torch.distributed.barrier()
        full = pdist.replicated_fwd(q, k, v, sh, po, causal=causal)
        qf, kf, vf = synth.make_qkv(B, Hq, Hkv, N, d, base=33, device="cuda")
        ref = attn_fwd(qf, kf, vf, causal=causal)
        torch.cuda.synchronize()
        ok = torch.equal(full.view(torch.int16), ref.view(torch.int16))
        po.close()
        out.put((r, ok))
        torch.distributed.destroy_process_group()
    except Exception as e:  # pragma: no cover
        out.put((rank, repr(e)))


@pytest.mark.gpu
@pytest.mark.parametrize("causal", [False, True])
def test_replicated_two_processes_ipc(causal):
    """Two ranks on cuda:0 (gloo plumbing): each kernel stores its heads into
    both ranks' buffers through CUDA IPC; both end with the full output,
    bit-identical to the one-process forward over all heads."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, causal, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=300)
    assert res == {0: True, 1: True}, res
