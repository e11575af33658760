"""Screen an experiment variant (ATTN_NUMA_LIB=...) for correctness: forward
vs a torch fp32 reference on the GPU, several shapes incl. causal / GQA /
ragged N; prints one line per case.  (Screening only; the parity tests use
the fp64 oracle.)"""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2511_02132_b200 import attn_fwd, synth

ok = True
ref_path = os.environ.get("VARIANT_REF")  # bitwise reference outputs: saved if absent, compared if present
saved = torch.load(ref_path) if ref_path and os.path.exists(ref_path) else None
outs_all = []
for (B, Hq, Hkv, N, d, causal) in [(1, 4, 4, 2048, 128, False), (1, 4, 4, 2048, 128, True), (2, 8, 2, 1000, 128, True),
                                   (1, 2, 2, 1536, 64, False), (1, 2, 2, 777, 56, True)]:
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=3, device="cuda")
    kk = k.float().repeat_interleave(Hq // Hkv, 1)
    vv = v.float().repeat_interleave(Hq // Hkv, 1)
    s = q.float() @ kk.transpose(-1, -2) / d ** 0.5
    if causal:
        s = s.masked_fill(torch.ones(N, N, device="cuda", dtype=torch.bool).triu(1), float("-inf"))
    ref = torch.softmax(s, -1) @ vv
    outs = []
    for m in ("block_first", "swizzled_head_first"):
        o = torch.full_like(q, float("nan"))
        attn_fwd(q, k, v, o, causal=causal, mapping=m)
        outs.append(o)
    torch.cuda.synchronize()
    e = (outs[1].float() - ref).abs()
    good = bool(torch.isfinite(e).all()) and e.max().item() <= 2e-2 and e.mean().item() <= 2e-3 \
        and torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16))
    outs_all.append(outs[1].cpu())
    if saved is not None:
        same = torch.equal(saved[len(outs_all) - 1].view(torch.int16), outs_all[-1].view(torch.int16))
        good &= same
        print(f"  bit-identical to {ref_path}: {same}")
    ok &= good
    print(f"  check B{B} H{Hq}/{Hkv} N{N} d{d} causal={causal}: max {e.max().item():.2e} mean {e.mean().item():.2e} "
          f"{'ok' if good else 'FAIL'}")
if ref_path and saved is None:
    torch.save(outs_all, ref_path)
print("  variant check:", "PASS" if ok else "FAIL")
