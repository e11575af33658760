"""Per-block timeline of the dQ kernel's CTA 0, second unit (build with
-D ATTN_BWD_TIMELINE): MMA warp [p_ready woke, S(j+1) issued, ds_ready woke,
dQ+dP issued] and, per column half, [s_ready woke, S released, exps done,
dp_ready woke, dS stored]."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2511_02132_b200 import attn_bwd, attn_fwd_lse, attn_set_schedule_trace, synth

B, Hq, Hkv, N, d = 1, 32, 32, 8192, 128
q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=0, device="cuda")
do = synth.make_tensor("q", B, Hq, N, d, base=1, device="cuda")
o, lse = attn_fwd_lse(q, k, v)
attn_bwd(q, k, v, o, do, lse)
buf = torch.zeros(64 * 16 * 2, dtype=torch.int32, device="cuda")
attn_set_schedule_trace(0, buf)
attn_bwd(q, k, v, o, do, lse)
torch.cuda.synchronize()
attn_set_schedule_trace(0, None)
t = buf.view(torch.int64).cpu().numpy().reshape(64, 16)
t = t - t[8, 0]
print(" j | mma: p_wake S_iss ds_wake dQdP_iss | h0: s_wake S_rel exp_done dp_wake ds_st | h1: same")
for j in range(8, 20):
    print(f"{j:2d} | " + " ".join(f"{x:7d}" for x in t[j, :4]) + " | " + " ".join(f"{x:7d}" for x in t[j, 4:9]) +
          " | " + " ".join(f"{x:7d}" for x in t[j, 9:14]))
per = np.median(np.diff(t[8:60, 0]))
print("cycles per block (median):", int(per), " tensor work 1536")
for h, o_ in ((0, 4), (1, 9)):
    ph = np.median(np.diff(t[8:60, o_:o_ + 5], axis=1), axis=0).astype(int)
    print(f"half {h}: ld+release {ph[0]}  exps {ph[1]}  wait dP {ph[2]}  dS {ph[3]}")
print("ds stored -> MMA ds_wake:", int(np.median(t[8:60, 2] - np.maximum(t[8:60, 8], t[8:60, 13]))),
      " dQdP issued -> next dp_wake (h0):", int(np.median(t[9:61, 7] - t[8:60, 3])))
