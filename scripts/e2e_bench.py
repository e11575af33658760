"""End-to-end timing of attn_fwd_host (pinned host q/k/v/o; H2D + kernel +
D2H + sync per call) for chunking experiments."""
import argparse
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import WORKLOADS
from paper_2511_02132_b200 import api, synth

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="C2,C3")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
for name in a.configs.split(","):
    B, Hq, Hkv, N, d, causal, _ = WORKLOADS[name]
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=0, device="cpu")
    qh, kh, vh = (t.pin_memory() for t in (q, k, v))
    oh = torch.empty_like(qh).pin_memory()
    flops = 4 * B * Hq * N * N * d * (0.5 if causal else 1.0)
    for _ in range(2):
        api.attn_fwd_host(qh, kh, vh, oh, causal=causal, mapping="swizzled_head_first")
    ts = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        api.attn_fwd_host(qh, kh, vh, oh, causal=causal, mapping="swizzled_head_first")
        ts.append(time.perf_counter() - t0)
    ts.sort()
    med = ts[len(ts) // 2]
    moved = (qh.numel() * 2 + kh.numel() * 2 * 2 + oh.numel() * 2)
    print(f"{name} e2e median {med * 1e3:8.3f} ms  {flops / med / 1e12:7.1f} TFLOP/s  "
          f"{moved / med / 1e9:6.1f} GB/s moved  chunks {api.attn_last_launch_info()['kernel_launches']}", flush=True)
