"""One backward call at a bench workload (for ncu captures): python scripts/bwd_once.py C6 [--deterministic]."""
import sys

import torch

sys.path.insert(0, ".")
from bench import WORKLOADS
from paper_2511_02132_b200 import attn_bwd, attn_fwd_lse, synth

name = sys.argv[1] if len(sys.argv) > 1 else "C6"
det = "--deterministic" in sys.argv
mapping = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--mapping=")), "swizzled_head_first")
B, Hq, Hkv, N, d, causal, _ = WORKLOADS[name]
q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=0, device="cuda")
do = synth.make_tensor("q", B, Hq, N, d, base=1, device="cuda")
o, lse = attn_fwd_lse(q, k, v, causal=causal)
attn_bwd(q, k, v, o, do, lse, causal=causal, mapping=mapping, deterministic=det)
torch.cuda.synchronize()
print("done")
