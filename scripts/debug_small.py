"""Quick GPU sanity run: one tiny case per kernel variant, printing errors."""
import math
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import attn as oa
from paper_2511_02132_b200 import attn_fwd, attn_topology, synth

t0 = time.time()
topo = attn_topology(0)
print("topology:", {k: v for k, v in topo.items() if k != "domain_of_smid"}, f"{time.time()-t0:.2f}s")
print("domain_of_smid:", topo["domain_of_smid"])
for (B, Hq, Hkv, N, d, causal) in [(1, 1, 1, 128, 64, False), (1, 1, 1, 256, 128, False),
                                   (1, 2, 2, 256, 128, True), (1, 2, 2, 384, 64, True)]:
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=1, device="cuda")
    ref = oa.attention(q.cpu(), k.cpu(), v.cpu(), causal=causal, scale=1 / math.sqrt(d))
    for m in ("block_first", "head_first", "swizzled_head_first"):
        o = torch.full_like(q, float("nan"))
        attn_fwd(q, k, v, o, causal=causal, mapping=m)
        torch.cuda.synchronize()
        got = o.float().cpu().numpy()
        err = np.abs(got - ref)
        print(f"{B}x{Hq}/{Hkv}x{N}x{d} causal={causal} {m}: nan={np.isnan(got).sum()} "
              f"max={np.nanmax(err):.3e} mean={np.nanmean(err):.3e}")
        if np.nanmax(err) > 2e-2 and m == "block_first":
            r = np.unravel_index(np.nanargmax(err), err.shape)
            print("   worst at", r, "got", got[r], "ref", ref[r])
            print("   row0 got[:8]", got[0, 0, 0, :8], "\n   row0 ref[:8]", ref[0, 0, 0, :8])
