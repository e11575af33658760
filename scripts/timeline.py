"""Per-iteration timeline of CTA 0 (build with -D ATTN_TIMELINE)."""
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
mma = t[:64 * 8].reshape(64, 8)[:, :6] - t0
sm0 = t[600:600 + 192].reshape(64, 3) - t0
sm1 = t[800:800 + 192].reshape(64, 3) - t0
print(" j | it_start  kv_ok  p0_ok  t0_iss  p1_ok  t1_iss | sm0: s_wake  p_h0  p_h1 | sm1: s_wake  p_h0  p_h1")
for j in range(8, 24):
    print(f"{j:2d} | " + " ".join(f"{x:7d}" for x in mma[j]) + " | " + " ".join(f"{x:6d}" for x in sm0[j]) +
          " | " + " ".join(f"{x:6d}" for x in sm1[j]))
d = np.diff(mma[8:60, 0])
print("cycles per iteration (median over j=8..60):", int(np.median(d)), " ideal 2048")
print("softmax0 s_wake -> p_h1 (median):", int(np.median(sm0[8:60, 2] - sm0[8:60, 0])),
      " softmax1:", int(np.median(sm1[8:60, 2] - sm1[8:60, 0])))
print("t0 issue done -> softmax0 next s_wake (median):", int(np.median(sm0[9:61, 0] - mma[8:60, 3])))
print("softmax0 p_h1 -> MMA p0_ok (median):", int(np.median(mma[9:61, 2] - sm0[9:61, 2])))
# fine softmax stamps (tile 0 and 1): s_wake, ld done, max done, P half 0, P half 1, sum done
for tt in (0, 1):
    f = t[4096 + tt * 512: 4096 + tt * 512 + 64 * 8].reshape(64, 8) - t0
    # stamps: 0 s_wake, 1 ld done, 2 max done, 6 exps h0 done, 3 P h0 published, 7 exps h1 done, 4 P h1 published, 5 sum
    g = f[8:60][:, [0, 1, 2, 6, 3, 7, 4, 5]]
    dd = np.median(np.diff(g, axis=1), axis=0).astype(int)
    print(f"tile {tt} softmax phases (median cycles): ld {dd[0]}  max {dd[1]}  exps h0 {dd[2]}  st+publish h0 {dd[3]}  "
          f"exps h1 {dd[4]}  st+publish h1 {dd[5]}  sum {dd[6]}  total {int(np.median(f[8:60, 5] - f[8:60, 0]))}")
