"""Small launches for compute-sanitizer (memcheck): every mapping, causal and not,
ragged N, padded d, GQA."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2511_02132_b200 import attn_fwd, synth

for (B, Hq, Hkv, N, d, causal) in [(1, 2, 2, 256, 128, False), (2, 4, 2, 300, 64, True), (1, 2, 1, 77, 56, True),
                                   (1, 3, 3, 640, 96, False)]:
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=1, device="cuda")
    for m in ("block_first", "head_first", "swizzled_head_first", "swizzled_block_first"):
        attn_fwd(q, k, v, causal=causal, mapping=m)
torch.cuda.synchronize()
print("sanitize run done")
