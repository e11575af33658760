"""Cycle account of the backward's dK/dV elementwise warps (the fused kernel for
d <= 64, the two-pass dK/dV kernel for d > 64) (library built with
-D ATTN_CYCLES, loaded via ATTN_NUMA_LIB): per (key block, query block) pair,
the average cycles each elementwise warp spends in each step.  Averaged over
the 8 elementwise warps of the first 64 CTAs.

    python -m paper_2511_02132_b200.build -D ATTN_CYCLES --out paper_2511_02132_b200/lib/libattnnuma_cycles.so
    ATTN_NUMA_LIB=paper_2511_02132_b200/lib/libattnnuma_cycles.so python scripts/bwd_cycles.py [B Hq Hkv N d causal]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2511_02132_b200 import attn_bwd, attn_fwd_lse, attn_set_schedule_trace, synth

a = sys.argv[1:]
B, Hq, Hkv, N, d = (int(x) for x in a[:5]) if a else (1, 128, 128, 32768, 56)
causal = bool(int(a[5])) if len(a) > 5 else True
q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=0, device="cuda")
do = synth.make_tensor("q", B, Hq, N, d, base=1, device="cuda")
o, lse = attn_fwd_lse(q, k, v, causal=causal)
attn_bwd(q, k, v, o, do, lse, causal=causal)
buf = torch.zeros(8192 * 2, dtype=torch.int32, device="cuda")
attn_set_schedule_trace(0, buf)
attn_bwd(q, k, v, o, do, lse, causal=causal)
torch.cuda.synchronize()
attn_set_schedule_trace(0, None)
c = buf.view(torch.int64).cpu().numpy()[:4096].reshape(64, 8, 8).astype(np.float64)
blocks = c[:, :, 7].sum()
per = c[:, :, :7].sum(axis=(0, 1)) / blocks
names = ["ring wait + setup", "S wait", "ld S + exps + mask", "dv_done wait + P^T pack/st/arrive",
         "dP wait", "ld dP + dS math + dS^T tmem st", "dk_done wait + dS^T STS + fence + arrive"]
if d > 64:  # two-pass dK/dV kernel (attn_bwd_sm100.cuh)
    names = ["ring (vector) wait + setup", "S^T wait", "ld S^T + exps + mask", "P^T pack + STS + fence + arrive",
             "dP^T wait", "ld dP^T + dS^T math + tmem st", "dv_done wait (P^T buffer free)"]
print(f"shape B{B} H{Hq}/{Hkv} N{N} d{d} causal={causal}: {blocks / (64 * 8):.0f} blocks per warp")
for n_, x in zip(names, per):
    print(f"  {n_:32s} {x:8.0f} cycles per block")
print(f"  {'total per block':32s} {per.sum():8.0f}")
