"""One C5-style launch per unit order for ncu (DRAM bytes / L2 hit rate by
order): python scripts/order_ncu.py [workload] [mapping] [cluster 0|1]; the
launches are ascending (2 warm-ups + 1), then descending (2 + 1)."""
import math
import sys

import torch

sys.path.insert(0, ".")
from bench import WORKLOADS
from paper_2511_02132_b200 import attn_fwd, attn_init, synth

W = sys.argv[1] if len(sys.argv) > 1 else "C5"
m = sys.argv[2] if len(sys.argv) > 2 else "swizzled_head_first"
cl = bool(int(sys.argv[3])) if len(sys.argv) > 3 else True
B, Hq, Hkv, N, d, causal, _ = WORKLOADS[W]
attn_init(0)
q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=0, device="cuda")
o = torch.empty_like(q)
for od in ("ascending", "descending"):
    for _ in range(3):
        attn_fwd(q, k, v, o, causal=causal, scale=1 / math.sqrt(d), mapping=m, order=od, cluster=cl)
    torch.cuda.synchronize()
