"""Context only: library attention (torch SDPA: cuDNN and flash backends) on
the same box and shapes, event-timed with an L2 flush between reps.  Not on
the product path; it tells how far our kernel sits from NVIDIA's own."""
import sys

import torch
from torch.nn.attention import SDPBackend, sdpa_kernel
import torch.nn.functional as F

CFG = {"C2": (1, 32, 8192, 128, False), "C3": (1, 128, 32768, 128, True), "C6": (1, 128, 32768, 64, True)}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name in (sys.argv[1] if len(sys.argv) > 1 else "C2,C3").split(","):
    B, H, N, d, causal = CFG[name]
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn(B, H, N, d, device="cuda", generator=g).bfloat16() for _ in range(3))
    flops = 4.0 * B * H * N * N * d * (0.5 if causal else 1.0)
    for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION):
        try:
            with sdpa_kernel([be]):
                for _ in range(3):
                    F.scaled_dot_product_attention(q, k, v, is_causal=causal)
                ts = []
                for _ in range(7):
                    flush.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    F.scaled_dot_product_attention(q, k, v, is_causal=causal)
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1))
            ts.sort()
            print(f"{name} {be.name:16s} median {ts[3]:8.3f} ms  {flops / ts[3] / 1e9:7.1f} TFLOP/s", flush=True)
        except Exception as e:  # noqa: BLE001
            print(f"{name} {be.name} unavailable: {str(e)[:200]}", flush=True)
