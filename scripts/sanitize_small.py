"""Small launches for compute-sanitizer (memcheck / synccheck): every mapping,
causal and not, ragged N, padded d, GQA; the CTA-pair cluster forward; the
backward kernels (single-pass and two-pass)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2511_02132_b200 import attn_bwd, attn_fwd, attn_fwd_lse, synth

for (B, Hq, Hkv, N, d, causal) in [(1, 2, 2, 256, 128, False), (2, 4, 2, 300, 64, True), (1, 2, 1, 77, 56, True),
                                   (1, 3, 3, 640, 96, False)]:
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=1, device="cuda")
    for m in ("block_first", "head_first", "swizzled_head_first", "swizzled_block_first",
              "swizzled_head_first:shared"):
        attn_fwd(q, k, v, causal=causal, mapping=m)
        attn_fwd(q, k, v, causal=causal, mapping=m, cluster=True)
    o, lse = attn_fwd_lse(q, k, v, causal=causal)
    do = synth.make_tensor("q", B, Hq, N, d, base=9, device="cuda")
    attn_bwd(q, k, v, o, do, lse, causal=causal)                      # single-pass for d <= 64
    attn_bwd(q, k, v, o, do, lse, causal=causal, deterministic=True)  # two-pass
torch.cuda.synchronize()
print("sanitize run done")
