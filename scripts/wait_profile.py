"""Per-CTA MMA-warp wait attribution (build with -D ATTN_PROFILE_WAITS)."""
import math
import sys

import torch

sys.path.insert(0, ".")
from bench import WORKLOADS
from paper_2511_02132_b200 import attn_fwd, attn_set_schedule_trace, synth

for name in sys.argv[1].split(","):
    B, Hq, Hkv, N, d, causal, _ = WORKLOADS[name]
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=0, device="cuda")
    for m in ("block_first", "swizzled_head_first"):
        buf = torch.zeros(148 * 8 * 2, dtype=torch.int32, device="cuda")  # 148 x 8 int64
        attn_fwd(q, k, v, causal=causal, mapping=m)
        attn_set_schedule_trace(0, buf)
        attn_fwd(q, k, v, causal=causal, mapping=m)
        torch.cuda.synchronize()
        attn_set_schedule_trace(0, None)
        w = buf.view(torch.int64).view(148, 8).double()
        tot = w[:, 0].mean().item()
        names = ["q_full", "kv_full", "p_ready0", "p_ready1", "sched"]
        parts = "  ".join(f"{nm} {w[:, i + 1].mean().item() / tot * 100:5.1f}%" for i, nm in enumerate(names))
        print(f"{name} {m:20s} total {tot / 1e6:7.2f} Mcyc  {parts}")
