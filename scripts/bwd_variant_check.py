"""Screen a backward variant (ATTN_NUMA_LIB=...): two-pass gradients of a few
shapes (d 128 / 96 / 64, causal, GQA, ragged N) saved to VARIANT_REF if absent,
else compared bit for bit with it."""
import math
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2511_02132_b200 import attn_bwd, attn_fwd_lse, synth

ref_path = os.environ["VARIANT_REF"]
saved = torch.load(ref_path) if os.path.exists(ref_path) else None
outs, ok = [], True
for (B, Hq, Hkv, N, d, causal) in [(1, 4, 4, 1024, 128, True), (1, 4, 2, 777, 128, False), (2, 4, 4, 300, 96, True),
                                   (1, 2, 2, 640, 64, True)]:
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=41, device="cuda")
    o, lse = attn_fwd_lse(q, k, v, causal=causal, scale=1 / math.sqrt(d))
    do = synth.make_tensor("q", B, Hq, N, d, base=42, device="cuda")
    g = attn_bwd(q, k, v, o, do, lse, causal=causal, scale=1 / math.sqrt(d), deterministic=True)
    torch.cuda.synchronize()
    g = [t.cpu() for t in g]
    outs.append(g)
    if saved is not None:
        same = all(torch.equal(a.view(torch.int16), b.view(torch.int16)) for a, b in zip(g, saved[len(outs) - 1]))
        ok &= same
        print(f"  B{B} H{Hq}/{Hkv} N{N} d{d} causal={causal}: bit-identical {same}")
if saved is None:
    torch.save(outs, ref_path)
    print("  saved", ref_path)
print("  bwd variant check:", "PASS" if ok else "FAIL")
