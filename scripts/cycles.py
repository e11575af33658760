"""Cycle account of the softmax warps (build with -D ATTN_CYCLES): per 128-key
block, the average cycles each softmax warp spends waiting for S, loading S,
in the row max, in the exps + P stores (excluding the p_free wait), waiting
for p_free, plus the per-unit epilogue.  Averaged over the 8 softmax warps of
the first 64 CTAs.

    python scripts/cycles.py [B Hq Hkv N d causal]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2511_02132_b200 import attn_fwd, attn_set_schedule_trace, synth

a = sys.argv[1:]
B, Hq, Hkv, N, d = (int(x) for x in a[:5]) if a else (1, 32, 32, 8192, 64)
causal = bool(int(a[5])) if len(a) > 5 else False
q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=0, device="cuda")
attn_fwd(q, k, v, causal=causal)
buf = torch.zeros(8192 * 2, dtype=torch.int32, device="cuda")
attn_set_schedule_trace(0, buf)
attn_fwd(q, k, v, causal=causal, mapping="swizzled_head_first")
torch.cuda.synchronize()
attn_set_schedule_trace(0, None)
c = buf.view(torch.int64).cpu().numpy()[:4096].reshape(64, 8, 8).astype(np.float64)
blocks = c[:, :, 7].sum()
per = c[:, :, :7].sum(axis=(0, 1)) / blocks
names = ["S wait", "ld S", "row max", "exps+stores", "p_free wait", "epilogue (per block)", "o_ready wait (per block)"]
print(f"shape B{B} H{Hq}/{Hkv} N{N} d{d} causal={causal}: {blocks / (64 * 8):.0f} blocks per warp")
for n_, x in zip(names, per):
    print(f"  {n_:26s} {x:8.0f} cycles per block")
print(f"  {'total per block':26s} {per[:6].sum():8.0f}")
