"""Quick per-mapping timing (CUDA events, L2 flushed between reps)."""
import argparse
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2511_02132_b200 import attn_fwd, attn_topology, synth

CFG = {"C2": (1, 32, 32, 8192, 128, False), "C3": (1, 128, 128, 32768, 128, True),
       "C4": (2, 64, 8, 16384, 128, True), "C5": (1, 128, 128, 131072, 128, True),
       "C6": (1, 128, 128, 32768, 56, True)}
ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="C2,C3,C4")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--order", default="ascending")
ap.add_argument("--maps", default="block_first,head_first,swizzled_head_first")
a = ap.parse_args()
topo = attn_topology(0)
print({k: v for k, v in topo.items() if k != "domain_of_smid"})
flush = torch.empty(2 * topo["l2_bytes"], dtype=torch.uint8, device="cuda")
for name in a.configs.split(","):
    B, Hq, Hkv, N, d, causal = CFG[name]
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=0, device="cuda")
    o = torch.empty_like(q)
    flops = 4 * B * Hq * N * N * d * (0.5 if causal else 1.0)
    for m in a.maps.split(","):
        for _ in range(3):
            attn_fwd(q, k, v, o, causal=causal, mapping=m, order=a.order)
        times = []
        for _ in range(a.reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            attn_fwd(q, k, v, o, causal=causal, mapping=m, order=a.order)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        times.sort()
        med = times[len(times) // 2]
        print(f"{name} {a.order[:4]} {m:22s} median {med:8.3f} ms  min {times[0]:8.3f} ms  "
              f"{flops / med / 1e9:8.1f} TFLOP/s ({flops / med / 1e9 / 1668 * 100:5.1f}% of 1668)", flush=True)
    del q, k, v, o
    torch.cuda.empty_cache()
