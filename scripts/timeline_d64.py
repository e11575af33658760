"""Softmax timeline of CTA 0's first unit for a head-dim-64 forward (build with
-D ATTN_TIMELINE): per key block, each tile's S wake-up and P publication, to
see whether the two tiles' softmax phases overlap (de-phased) or coincide."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2511_02132_b200 import attn_fwd, attn_set_schedule_trace, synth

q, k, v = synth.make_qkv(1, 32, 32, 8192, 64, base=0, device="cuda")
attn_fwd(q, k, v)
buf = torch.zeros(8192 * 2, dtype=torch.int32, device="cuda")
attn_set_schedule_trace(0, buf)
attn_fwd(q, k, v, mapping="swizzled_head_first")
torch.cuda.synchronize()
attn_set_schedule_trace(0, None)
t = buf.view(torch.int64).cpu().numpy().astype(np.int64)
sm = [t[600 + tt * 200: 600 + tt * 200 + 192].reshape(64, 3) for tt in (0, 1)]
fine = [t[4096 + tt * 512: 4096 + tt * 512 + 64 * 8].reshape(64, 8) for tt in (0, 1)]
t0 = sm[0][0, 0]
print(" j | tile0: s_wake p_h0 p_h1 | tile1: s_wake p_h0 p_h1")
for j in range(8, 24):
    print(f"{j:2d} | " + " ".join(f"{x - t0:7d}" for x in sm[0][j]) + " | " + " ".join(f"{x - t0:7d}" for x in sm[1][j]))
for tt in (0, 1):
    print(f"tile {tt}: cycles per block {int(np.median(np.diff(sm[tt][8:60, 0])))}, "
          f"s_wake -> p_h1 {int(np.median(sm[tt][8:60, 2] - sm[tt][8:60, 0]))}, "
          f"p_h1 -> next s_wake {int(np.median(sm[tt][9:61, 0] - sm[tt][8:60, 2]))}")
    g = fine[tt][8:60][:, [0, 1, 2, 6, 3, 7, 4, 5]]
    dd = np.median(np.diff(g, axis=1), axis=0).astype(int)
    print(f"  phases: ld {dd[0]} max {dd[1]} exps h0 {dd[2]} st+pub h0 {dd[3]} exps h1 {dd[4]} st+pub h1 {dd[5]} sum {dd[6]}")
off = np.median(sm[1][8:60, 0] - sm[0][8:60, 0])
print("tile 1 s_wake - tile 0 s_wake (median):", int(off))
m = t[2048: 2048 + 64 * 8].reshape(64, 8)[:, [0, 1, 2, 3, 6, 4, 7, 5]] - t0
print(" j | MMA: top kv_ok S0_iss S1_iss p0_ok PV0_iss p1_ok PV1_iss  (relative to tile 0 s_wake of block j)")
for j in range(8, 16):
    print(f"{j:2d} | " + " ".join(f"{x - (sm[0][j, 0] - t0):7d}" for x in m[j]))
qq = t[5120: 5120 + 8 * 128].reshape(2, 4, 64, 2)
for tt in (0, 1):
    w = np.median(qq[tt, :, 8:40, 0] - qq[tt, 0:1, 8:40, 0], axis=1).astype(int)
    pub = np.median(qq[tt, :, 8:40, 1] - qq[tt, 0:1, 8:40, 1], axis=1).astype(int)
    dur = np.median(qq[tt, :, 8:40, 1] - qq[tt, :, 8:40, 0], axis=1).astype(int)
    print(f"tile {tt} per quarter (vs quarter 0): s_wake {list(w)}  p_h1 {list(pub)}  s_wake->p_h1 {list(dur)}")
sf = t[2048 + 512: 2048 + 512 + 128].reshape(64, 2)
print(" j | s_free ok (tile 0, tile 1) relative to tile 0 s_wake of block j")
for j in range(8, 16):
    print(f"{j:2d} | " + " ".join(f"{x - sm[0][j, 0]:7d}" for x in sf[j]))
done = t[3072: 3072 + 64]
print(" j | s_ready[0] phase j+1 complete (S_0(j+1) landed), relative to tile 0 s_wake of block j; next s_wake")
for j in range(8, 16):
    print(f"{j:2d} | {done[j + 1] - sm[0][j, 0]:7d}  {sm[0][j + 1, 0] - sm[0][j, 0]:7d}")
