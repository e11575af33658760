"""Single-pass (fused, d <= 64) backward vs the two-pass (deterministic) one and
the fp64 oracle: parity on small shapes, dk/dv bit-identity between the two
paths, dq difference, and event timing at full size (L2 flushed between reps).
FLOPs: 10*B*Hq*N^2*d (five matmuls), causal x0.5."""
import argparse
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from bench import WORKLOADS
from oracle import attn as oa
from tolerance import check_grad
from paper_2511_02132_b200 import attn_bwd, attn_fwd_lse, attn_topology, synth

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="C6")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--maps", default="head_first,swizzled_head_first")
ap.add_argument("--skip-small", action="store_true")
a = ap.parse_args()

if not a.skip_small:
    for (B, Hq, Hkv, N, d, causal) in [(1, 2, 2, 256, 64, False), (1, 2, 2, 256, 64, True), (2, 4, 2, 384, 64, True),
                                       (1, 2, 2, 200, 56, True), (1, 4, 1, 300, 32, False), (1, 2, 2, 77, 8, True)]:
        q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=31, device="cuda")
        do = synth.make_tensor("q", B, Hq, N, d, base=32, device="cuda")
        o, lse = attn_fwd_lse(q, k, v, causal=causal)
        f = attn_bwd(q, k, v, o, do, lse, causal=causal)
        r = attn_bwd(q, k, v, o, do, lse, causal=causal, deterministic=True)
        torch.cuda.synchronize()
        rq, rk, rv, _ = oa.attention_bwd(q.cpu(), k.cpu(), v.cpu(), do.cpu(), causal=causal, scale=1 / math.sqrt(d))
        same_kv = all(torch.equal(x.view(torch.int16), y.view(torch.int16)) for x, y in zip(f[1:], r[1:]))
        dqd = (f[0].float() - r[0].float()).abs().max().item()
        errs = []
        for name, g, ref in (("dq", f[0], rq), ("dk", f[1], rk), ("dv", f[2], rv)):
            gg = g.float().cpu().numpy().astype(np.float64)
            errs.append(f"{name} max {np.abs(gg - ref).max():.2e}")
            try:
                check_grad(name, g, ref)
                errs[-1] += " ok"
            except AssertionError as e:
                errs[-1] += f" FAIL({e})"
        print(f"small {(B, Hq, Hkv, N, d, causal)}: dk/dv bit-identical to two-pass: {same_kv}; "
              f"|dq fused - two-pass| max {dqd:.2e}; " + "; ".join(errs), flush=True)

topo = attn_topology(0)
flush = torch.empty(2 * topo["l2_bytes"], dtype=torch.uint8, device="cuda")
for name in a.configs.split(","):
    B, Hq, Hkv, N, d, causal, _ = WORKLOADS[name]
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=0, device="cuda")
    do = synth.make_tensor("q", B, Hq, N, d, base=1, device="cuda")
    o, lse = attn_fwd_lse(q, k, v, causal=causal)
    flops = 10 * B * Hq * N * N * d * (0.5 if causal else 1.0)
    res = {}
    for m in a.maps.split(","):
        for det in (False, True):
            for _ in range(2):
                out = attn_bwd(q, k, v, o, do, lse, causal=causal, mapping=m, deterministic=det)
            res[(m, det)] = out
            ts = []
            for _ in range(a.reps):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                attn_bwd(q, k, v, o, do, lse, causal=causal, mapping=m, deterministic=det)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ts.sort()
            med = ts[len(ts) // 2]
            print(f"bwd {name} {m:22s} {'two-pass' if det else 'fused':8s} {med:8.3f} ms  "
                  f"{flops / med / 1e9:7.1f} TFLOP/s", flush=True)
        f, r = res[(m, False)], res[(m, True)]
        same_kv = all(torch.equal(x.view(torch.int16), y.view(torch.int16)) for x, y in zip(f[1:], r[1:]))
        dqd = (f[0].float() - r[0].float()).abs()
        print(f"  {m}: dk/dv bit-identical {same_kv}; |dq fused - two-pass| max {dqd.max().item():.3e} "
              f"mean {dqd.mean().item():.3e} (|dq| mean {r[0].float().abs().mean().item():.3e})", flush=True)
