"""Bit-compare the forward of the current build across processes (e.g. the
pair kernel vs ATTN_FWD_PAIR=0) on small and medium shapes.

    python scripts/pair_check.py --save /tmp/a.pt
    ATTN_FWD_PAIR=0 python scripts/pair_check.py --save /tmp/b.pt
    python scripts/pair_check.py --compare /tmp/a.pt /tmp/b.pt
Analysis tooling only (not on the product path)."""
import argparse
import math
import sys

import torch

sys.path.insert(0, ".")

SHAPES = [(1, 2, 2, 128, 128, False), (1, 2, 2, 128, 128, True), (1, 4, 4, 300, 128, False),
          (1, 2, 2, 200, 128, True), (2, 4, 2, 1000, 96, True), (1, 8, 8, 4096, 128, True),
          (1, 8, 8, 4096, 128, False), (2, 16, 4, 2048, 128, True), (1, 3, 3, 77, 120, True),
          (1, 32, 32, 8192, 128, False)]
ap = argparse.ArgumentParser()
ap.add_argument("--save")
ap.add_argument("--compare", nargs=2)
a = ap.parse_args()
if a.compare:
    x, y = torch.load(a.compare[0]), torch.load(a.compare[1])
    bad = 0
    for key in x:
        same = torch.equal(x[key], y[key])
        diff = (x[key].float() - y[key].float()).abs().max().item()
        print(key, "bit-identical" if same else f"DIFFER max|d|={diff}")
        bad += not same
    sys.exit(1 if bad else 0)
from paper_2511_02132_b200 import attn_fwd, attn_last_launch_info, synth  # noqa: E402

out = {}
for (B, Hq, Hkv, N, d, causal) in SHAPES:
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=1, device="cuda")
    for m in ("swizzled_head_first", "block_first"):
        o = torch.full_like(q, float("nan"))
        attn_fwd(q, k, v, o, causal=causal, scale=1 / math.sqrt(d), mapping=m)
        torch.cuda.synchronize()
        info = attn_last_launch_info()
        key = f"{B}x{Hq}/{Hkv}x{N}x{d} c={int(causal)} {m}"
        out[key] = o.cpu()
        print(key, "grid", info["grid"], "smem", info["smem_bytes"], "nan" if torch.isnan(o).any().item() else "ok",
              flush=True)
torch.save(out, a.save)
