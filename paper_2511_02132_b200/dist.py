"""Head sharding across the GPUs of one node.

PAPER.md:167: "Each grid cell operates independently with no data reuse
between heads or batch items."  Rank r of G therefore owns KV heads
[r*Hkv/G, (r+1)*Hkv/G) and their query heads [r*Hq/G, (r+1)*Hq/G) for every
batch item, and runs attn_fwd on that shard with NO communication.  Inside
each GPU the paper's mapping logic is unchanged (swizzled head-first splits
the rank's ACCs across its two dies).

The only collectives are optional: an all-gather of O when the caller asks
for replicated output, and the max-over-ranks of timings.  torch.distributed
(NCCL on GPUs, gloo in the CPU tests) is plumbing only.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class HeadShard:
    rank: int
    world: int
    q_lo: int
    q_hi: int
    kv_lo: int
    kv_hi: int

    @property
    def hq(self) -> int:
        return self.q_hi - self.q_lo

    @property
    def hkv(self) -> int:
        return self.kv_hi - self.kv_lo


def shard_heads(Hq: int, Hkv: int, rank: int, world: int) -> HeadShard:
    """Contiguous KV-head ranges (whole GQA groups) per rank; needs Hkv % world == 0."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    if Hq % Hkv != 0:
        raise ValueError("Hq % Hkv != 0")
    if Hkv % world != 0:
        raise ValueError(f"Hkv={Hkv} is not divisible by world={world}: heads cannot be sharded evenly")
    G = Hq // Hkv
    per = Hkv // world
    kv_lo, kv_hi = rank * per, (rank + 1) * per
    return HeadShard(rank, world, kv_lo * G, kv_hi * G, kv_lo, kv_hi)


def env_rank_world():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def init(backend: Optional[str] = None, nccl_debug_init: bool = False, force: bool = False) -> tuple:
    """Initialise the default process group from torchrun's env (127.0.0.1 rendezvous).

    Only for world > 1, or with force=True under torchrun (a process group of
    one rank, so the NCCL collective path itself can be exercised on one GPU).
    nccl_debug_init: NCCL_DEBUG=INFO scoped to the INIT subsystem unless the
    caller set NCCL_DEBUG, so communicator creation (ranks, transports, NVLS)
    is visible in the log.  ATTN_BENCH_SHARE_GPU=1 (tests only): every rank
    uses cuda:0 and gloo, so the multi-rank code path runs on a one-GPU box."""
    rank, world, local = env_rank_world()
    if os.environ.get("ATTN_BENCH_SHARE_GPU") == "1":
        local = 0
        backend = "gloo"
    under_torchrun = "RANK" in os.environ and "MASTER_PORT" in os.environ
    if (world > 1 or (force and under_torchrun)) and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            if nccl_debug_init and "NCCL_DEBUG" not in os.environ:
                os.environ["NCCL_DEBUG"] = "INFO"
                os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            torch.cuda.set_device(local)
            dist.init_process_group(backend=backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend=backend)
    return rank, world, local


def all_gather_heads(o_local: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """Replicated O from per-rank head shards [B, Hq/G, N, d] -> [B, Hq, N, d]."""
    B, hq, N, d = o_local.shape
    if not (dist.is_available() and dist.is_initialized()):
        if world != 1:
            raise RuntimeError("all_gather_heads: no process group for world > 1")
        return o_local
    buf = torch.empty((world, B, hq, N, d), dtype=o_local.dtype, device=o_local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(buf, o_local.contiguous(), group=group)  # NVLink / NVSwitch
    else:
        dist.all_gather(list(buf.unbind(0)), o_local.contiguous(), group=group)
    return buf.permute(1, 0, 2, 3, 4).reshape(B, world * hq, N, d)


def max_over_ranks(x: float, device=None) -> float:
    """Max of a scalar over all ranks (timing aggregation)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    if dist.get_backend() != "nccl":
        device = "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class PeerOutput:
    """A full-size output [B, Hq, N, d] on every rank, mapped into every other
    rank's address space (CUDA IPC; NVLink P2P between GPUs of one node), so
    the forward's epilogue can store each finished O tile straight into all
    ranks' copies (C-ABI attn_fwd_replicated) instead of an all-gather after
    the kernel (fused alternative).

    ptrs[r] is rank r's buffer as seen from this process (this rank's own
    tensor for r == rank).  Collective: every rank of `group` must construct
    it with the same shape.  close() unmaps the peers (also collective)."""

    def __init__(self, shape, rank: int, world: int, device, group=None, api=None):
        if api is None:
            from . import api as api_mod
            api = api_mod
        self._api = api
        self.rank, self.world, self.group = rank, world, group
        self.local = torch.empty(tuple(shape), dtype=torch.bfloat16, device=device)
        rec = api.ipc_get_handle(self.local) if world > 1 else b""
        recs = [None] * world
        if world > 1:
            dist.all_gather_object(recs, rec, group=group)
        self.ptrs = [self.local.data_ptr() if r == rank else api.ipc_open(recs[r]) for r in range(world)]

    def close(self) -> None:
        for r, p in enumerate(self.ptrs):
            if r != self.rank:
                self._api.ipc_close(p)
        self.ptrs = [self.local.data_ptr() if r == self.rank else 0 for r in range(self.world)]
        if self.world > 1:
            dist.barrier(group=self.group)  # no rank frees its buffer while a peer still maps it


def replicated_fwd(q, k, v, shard: HeadShard, out: PeerOutput, *, causal: bool = False, scale=None,
                   mapping="swizzled_head_first", sync: bool = True, api=None, **kw) -> torch.Tensor:
    """This rank's head shard forward, its O tiles stored into every rank's
    PeerOutput buffer by the kernel epilogue (own buffer first).  With sync,
    waits for the stream and then for all ranks, after which out.local holds
    the whole output.  Shard heads land at shard.q_lo."""
    if api is None:
        from . import api as api_mod
        api = api_mod
    dsts = [out.ptrs[out.rank]] + [p for r, p in enumerate(out.ptrs) if r != out.rank]
    Hq_out = out.local.shape[1]
    api.attn_fwd_replicated(q, k, v, dsts, Hq_out, shard.q_lo, causal=causal, scale=scale, mapping=mapping, **kw)
    if sync:
        # the stream the epilogue's peer stores were enqueued on, not merely
        # the current one: the barrier below must not pass before they land
        (kw.get("stream") or torch.cuda.current_stream()).synchronize()
        if out.world > 1:
            dist.barrier(group=out.group)
    return out.local
