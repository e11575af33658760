"""Backward timing per mapping (CUDA events, L2 flushed between reps).
FLOPs: 10*B*Hq*N^2*d (five matmuls), causal x0.5."""
import argparse
import math
import sys

import torch

sys.path.insert(0, ".")
from bench import WORKLOADS
from paper_2511_02132_b200 import attn_bwd, attn_fwd_lse, attn_topology, synth

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="C2,C3")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--maps", default="block_first,head_first,swizzled_head_first")
a = ap.parse_args()
topo = attn_topology(0)
flush = torch.empty(2 * topo["l2_bytes"], dtype=torch.uint8, device="cuda")
for name in a.configs.split(","):
    B, Hq, Hkv, N, d, causal, _ = WORKLOADS[name]
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=0, device="cuda")
    do = synth.make_tensor("q", B, Hq, N, d, base=1, device="cuda")
    o, lse = attn_fwd_lse(q, k, v, causal=causal)
    flops = 10 * B * Hq * N * N * d * (0.5 if causal else 1.0)
    for m in a.maps.split(","):
        for _ in range(2):
            attn_bwd(q, k, v, o, do, lse, causal=causal, mapping=m)
        ts = []
        for _ in range(a.reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            attn_bwd(q, k, v, o, do, lse, causal=causal, mapping=m)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        med = ts[len(ts) // 2]
        print(f"bwd {name} {m:22s} {med:8.3f} ms  {flops / med / 1e9:7.1f} TFLOP/s ({flops / med / 1e9 / 1668 * 100:4.1f}% of 1668)",
              flush=True)
