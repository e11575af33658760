"""Per-block timeline of CTA 0's first tile in the 256-key forward kernel
(build with -D ATTN_TIMELINE -D N256_TIMELINE)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2511_02132_b200 import attn_fwd, attn_set_schedule_trace, synth

q, k, v = synth.make_qkv(1, 32, 32, 8192, 128, base=0, device="cuda")
attn_fwd(q, k, v)
buf = torch.zeros(8192 * 2, dtype=torch.int32, device="cuda")
attn_set_schedule_trace(0, buf)
attn_fwd(q, k, v, mapping="swizzled_head_first")
torch.cuda.synchronize()
attn_set_schedule_trace(0, None)
t = buf.view(torch.int64).cpu().numpy().astype(np.int64)
t0 = t[1000]
mma = t[:32 * 8].reshape(32, 8)[:, :4] - t0
print(" j | top  sfree_ok  p0_ok  p1_ok |  hf0: s_wake ld max xchg exps pfree pub | hf1: same")
sm = [t[4096 + hf * 512: 4096 + hf * 512 + 32 * 8].reshape(32, 8)[:, :7] - t0 for hf in (0, 1)]
for j in range(4, 20):
    print(f"{j:2d} | " + " ".join(f"{x:7d}" for x in mma[j]) + " | " + " ".join(f"{x:6d}" for x in sm[0][j]) +
          " | " + " ".join(f"{x:6d}" for x in sm[1][j]))
print("cycles per block (median j=4..30):", int(np.median(np.diff(mma[4:31, 0]))), " ideal 2048")
for hf in (0, 1):
    d = np.median(np.diff(sm[hf][4:30], axis=1), axis=0).astype(int)
    print(f"hf{hf} phases: ld {d[0]} max {d[1]} xchg {d[2]} exps {d[3]} pfree-wait {d[4]} store+pub {d[5]}; "
          f"pub -> next s_wake {int(np.median(sm[hf][5:31, 0] - sm[hf][4:30, 6]))}")
