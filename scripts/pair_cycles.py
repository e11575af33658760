"""Cycle account of the pair kernel (attn_fwd_pair.cuh; build with
-D ATTN_CYCLES, run with ATTN_NUMA_LIB pointing at that build).
    python scripts/pair_cycles.py [B Hq Hkv N d causal]
Analysis tooling only."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2511_02132_b200 import attn_fwd, attn_set_schedule_trace, synth

a = sys.argv[1:]
B, Hq, Hkv, N, d = (int(x) for x in a[:5]) if a else (1, 32, 32, 8192, 128)
causal = bool(int(a[5])) if len(a) > 5 else False
q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=0, device="cuda")
attn_fwd(q, k, v, causal=causal)
buf = torch.zeros(64 * 12 * 8 * 2 + 64, dtype=torch.int32, device="cuda")
attn_set_schedule_trace(0, buf)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
attn_fwd(q, k, v, causal=causal, mapping="swizzled_head_first")
e1.record()
torch.cuda.synchronize()
attn_set_schedule_trace(0, None)
c = buf.view(torch.int64).cpu().numpy()[:64 * 12 * 8].reshape(64, 12, 8).astype(np.float64)
ms = e0.elapsed_time(e1)
fl = 4.0 * B * Hq * N * N * d * (0.5 if causal else 1.0)
print(f"shape B{B} H{Hq}/{Hkv} N{N} d{d} causal={causal}: {ms:.3f} ms, {fl / ms / 1e9:.0f} TFLOP/s")
lead = c[0::2]
peer = c[1::2]


def show(title, rec, names):
    cnt = rec[:, 7].sum()
    print(f"{title}: {cnt / len(rec):.0f} counted events per warp")
    for i, n_ in enumerate(names):
        if n_:
            print(f"  {n_:28s} {rec[:, i].sum() / max(cnt, 1):9.0f} cycles per event")


show("producer (leader)", lead[:, 0], ["kv_empty wait", "", "q_empty wait (per event)"])
show("producer (peer)", peer[:, 0], ["kv_empty wait", "", "q_empty wait (per event)"])
show("S issuer (leader), per key block", lead[:, 1],
     ["K kv_full wait", "", "", "s_free wait", "S issue+commits", "", ""])
show("PV issuer (leader), per key block", lead[:, 3],
     ["V kv_full wait", "p_full wait", "PV issue", "", "", "o_empty wait", ""])
sm = np.concatenate([c[:, w] for w in range(4, 12)])
show("softmax warps, per own block", sm,
     ["S wait", "ld+mask+max", "m wait", "exps+P (+fixup)", "l wait", "epilogue", "o_full wait"] if len(sys.argv) < 8 else
     ["S wait", "ld+mask+max", "m wait", "exp math (+fixup)", "l wait", "P st + wait::st", "fence+arrive"])
