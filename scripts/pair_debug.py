"""Locate differences between two forward builds (pair kernel vs ATTN_FWD_PAIR=0).
    python scripts/pair_debug.py --save /tmp/a.pt [--shape B,Hq,Hkv,N,d,causal] [--mapping m]
    python scripts/pair_debug.py --compare /tmp/a.pt /tmp/b.pt
Analysis tooling only."""
import argparse
import math
import sys

import torch

sys.path.insert(0, ".")
ap = argparse.ArgumentParser()
ap.add_argument("--save")
ap.add_argument("--compare", nargs=2)
ap.add_argument("--shape", default="1,16,16,32768,128,1")
ap.add_argument("--mapping", default="swizzled_head_first")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
if a.compare:
    x, y = torch.load(a.compare[0]), torch.load(a.compare[1])
    for i in range(len(x)):
        o, r = x[i].float(), y[i].float()
        bad = (o != r) | torch.isnan(o)
        print(f"rep {i}: differing elements {int(bad.sum())} of {bad.numel()}")
        if bad.any():
            rows = bad.any(-1).nonzero()
            print("  first rows (b,h,i):", rows[:10].tolist())
            blocks = sorted(set((int(b_), int(h_), int(i_) // 128) for b_, h_, i_ in rows.tolist()))
            print("  (b,h,qblock) count", len(blocks), blocks[:20])
            print("  max|d|", (o - r).abs()[~torch.isnan(o)].max().item() if (~torch.isnan(o)).any() else None)
    sys.exit(0)
from paper_2511_02132_b200 import attn_fwd, synth  # noqa: E402

B, Hq, Hkv, N, d, causal = (int(t) for t in a.shape.split(","))
q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=1, device="cuda")
outs = []
for rep in range(a.reps):
    o = torch.full_like(q, float("nan"))
    attn_fwd(q, k, v, o, causal=bool(causal), scale=1 / math.sqrt(d), mapping=a.mapping)
    torch.cuda.synchronize()
    outs.append(o.cpu())
    print("rep", rep, "nan" if torch.isnan(o).any().item() else "ok", flush=True)
torch.save(outs, a.save)
