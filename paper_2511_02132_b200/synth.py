"""Seeded synthetic inputs shared by tests, bench and smoke.

Holds none of the method's arithmetic: it only draws i.i.d. N(0, 1) values
(unit variance, as the north star states) and rounds them to bf16 (RNE via
torch's ``.to``).  Each (tensor, batch, head) slice has its own generator
seeded by

    seed = 1_000_003 * base + 65_537 * tensor + 4_099 * b + head
    tensor: q = 0, k = 1, v = 2

so a head shard generated alone on one GPU is bit-identical to the same
slice of the full tensor generated on another.
"""
from __future__ import annotations

import torch

TENSOR_ID = {"q": 0, "k": 1, "v": 2}


def slice_seed(base: int, tensor: str, b: int, head: int) -> int:
    return 1_000_003 * base + 65_537 * TENSOR_ID[tensor] + 4_099 * b + head


def make_tensor(tensor: str, B: int, H: int, N: int, d: int, *, base: int = 0,
                head_offset: int = 0, batch_offset: int = 0, device="cpu", dtype=torch.bfloat16) -> torch.Tensor:
    """[B, H, N, d] tensor whose (b, h) slice is drawn from
    slice_seed(.., batch_offset + b, head_offset + h): any sub-block of heads
    and batch items is bit-identical to that slice of the full tensor."""
    out = torch.empty((B, H, N, d), dtype=dtype, device=device)
    gen = torch.Generator(device=device)
    for b in range(B):
        for h in range(H):
            gen.manual_seed(slice_seed(base, tensor, batch_offset + b, head_offset + h))
            x = torch.randn((N, d), generator=gen, device=device, dtype=torch.float32)
            out[b, h].copy_(x.to(dtype))
    return out


def make_qkv(B: int, Hq: int, Hkv: int, N: int, d: int, *, base: int = 0,
             q_head_offset: int = 0, kv_head_offset: int = 0, batch_offset: int = 0, device="cpu",
             dtype=torch.bfloat16):
    kw = dict(base=base, batch_offset=batch_offset, device=device, dtype=dtype)
    q = make_tensor("q", B, Hq, N, d, head_offset=q_head_offset, **kw)
    k = make_tensor("k", B, Hkv, N, d, head_offset=kv_head_offset, **kw)
    v = make_tensor("v", B, Hkv, N, d, head_offset=kv_head_offset, **kw)
    return q, k, v
