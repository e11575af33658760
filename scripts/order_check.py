"""C5-style order check: event-timed TFLOP/s of SHF and block-first (plain and
CTA-pair cluster) with ascending vs descending unit order, interleaved rounds
(one launch per variant per round, median), so every variant sees the same
power-cap state.  usage: python scripts/order_check.py [workload] [rounds]"""
import sys

import torch

sys.path.insert(0, ".")
from bench import WORKLOADS
from paper_2511_02132_b200 import attn_fwd, attn_init, synth

W = sys.argv[1] if len(sys.argv) > 1 else "C5"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 6
B, Hq, Hkv, N, d, causal, _ = WORKLOADS[W]
attn_init(0)
q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=0, device="cuda")
o = torch.empty_like(q)
flops = 4 * B * Hq * N * N * d * (0.5 if causal else 1.0)
variants = [(m, od, cl) for m in ("swizzled_head_first", "block_first") for cl in (True, False)
            for od in ("ascending", "descending")]
times = {x: [] for x in variants}
for x in variants:
    attn_fwd(q, k, v, o, causal=causal, mapping=x[0], order=x[1], cluster=x[2])
torch.cuda.synchronize()
for _ in range(R):
    for x in variants:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        attn_fwd(q, k, v, o, causal=causal, mapping=x[0], order=x[1], cluster=x[2])
        e1.record()
        torch.cuda.synchronize()
        times[x].append(e0.elapsed_time(e1))
for x in variants:
    t = sorted(times[x])[len(times[x]) // 2]
    print(f"{W} {x[0]:20s} {x[1]:10s} cluster={int(x[2])}  {t:9.3f} ms  {flops / t / 1e9:7.1f} TFLOP/s", flush=True)
