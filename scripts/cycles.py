"""Cycle account of the softmax warps (build with -D ATTN_CYCLES): per 128-key
block, the average cycles each softmax warp spends waiting for S, loading S,
in the row max, in the exps, the P stores, the O fix-up, waiting
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
buf = torch.zeros(8192 * 4, dtype=torch.int32, device="cuda")
attn_set_schedule_trace(0, buf)
attn_fwd(q, k, v, causal=causal, mapping="swizzled_head_first")
torch.cuda.synchronize()
attn_set_schedule_trace(0, None)
c = buf.view(torch.int64).cpu().numpy()[:8192].reshape(64, 8, 16).astype(np.float64)
blocks = c[:, :, 7].sum()
per = c[:, :, [0, 1, 2, 3, 8, 9, 4, 5, 6, 10, 11]].sum(axis=(0, 1)) / blocks
names = ["S wait", "ld S", "row max", "exps (+ row sum)", "P stores + publish", "O fix-up", "p_free (+ token) wait",
         "epilogue (per block)", "o_ready wait (per block)", "P_h1 SMEM stores", "P_h1 proxy fence"]
print(f"shape B{B} H{Hq}/{Hkv} N{N} d{d} causal={causal}: {blocks / (64 * 8):.0f} blocks per warp")
for n_, x in zip(names, per):
    print(f"  {n_:26s} {x:8.0f} cycles per block")
print(f"  {'total per block':26s} {per[:8].sum() + per[9:].sum():8.0f}")
