"""Minimal process for ncu: W warm-up launches then 1 launch of one workload/mapping."""
import argparse
import math
import sys

import torch

sys.path.insert(0, ".")
from bench import WORKLOADS
from paper_2511_02132_b200 import attn_fwd, attn_init, synth

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C2")
ap.add_argument("--mapping", default="swizzled_head_first")
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--cluster", action="store_true", help="ATTN_CLUSTER_MULTICAST (CTA pairs, K/V multicast)")
a = ap.parse_args()
B, Hq, Hkv, N, d, causal, _ = WORKLOADS[a.workload]
attn_init(0)
q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=0, device="cuda")
o = torch.empty_like(q)
for _ in range(a.warmup + 1):
    attn_fwd(q, k, v, o, causal=causal, scale=1 / math.sqrt(d), mapping=a.mapping, cluster=a.cluster)
torch.cuda.synchronize()
