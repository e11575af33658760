"""Controlled L2-capacity experiment.

MHA, 128 heads, d = 128, causal, N in {32K, 64K, 96K, 128K}: one launch per
(N, variant), so that `ncu` (run around this script) records one kernel per
configuration.  Per-head K/V = 4*N*d bytes = 16 / 32 / 48 / 64 MiB: swizzled
head-first keeps one head in flight per die (two live K/V prefixes against
one shared 126 MiB L2), head-first keeps one head in flight on the whole GPU.

    python scripts/capacity_sweep.py [--time] [--ns 32768,65536] [--variants shf,hf]

--time: event-timed (3 warm-ups, --reps launches, L2 flushed in between)
instead of the single launch per configuration used under ncu.
Analysis tooling only (not on the product path).
"""
import argparse
import json
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2511_02132_b200 import attn_fwd, attn_init, attn_topology, synth  # noqa: E402

# name -> (mapping, order, cluster)
VARIANTS = {
    "hf": ("head_first", "ascending", False),
    "shf": ("swizzled_head_first", "ascending", False),
    "shf_alt": ("swizzled_head_first", "alternate", False),
    "shf_pd": ("swizzled_head_first:per_die", "ascending", False),   # the paper's grain, forced
    "shf_sh": ("swizzled_head_first:shared", "ascending", False),    # R23 grain, forced
    "shf_pd_cl": ("swizzled_head_first:per_die", "ascending", True),
    "shf_sh_cl": ("swizzled_head_first:shared", "ascending", True),
    "bf": ("block_first", "ascending", False),
    "hf_cl": ("head_first", "ascending", True),
    "shf_cl": ("swizzled_head_first", "ascending", True),
    "shf_alt_cl": ("swizzled_head_first", "alternate", True),
}

ap = argparse.ArgumentParser()
ap.add_argument("--ns", default="32768,65536,98304,131072")
ap.add_argument("--variants", default="hf,shf,shf_alt")
ap.add_argument("--heads", type=int, default=128)
ap.add_argument("--time", action="store_true")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--json", default=None)
a = ap.parse_args()
attn_init(0)
topo = attn_topology(0)
flush = torch.empty(2 * topo["l2_bytes"], dtype=torch.uint8, device="cuda") if a.time else None
rows = []
for N in [int(x) for x in a.ns.split(",")]:
    H, d = a.heads, 128
    q, k, v = synth.make_qkv(1, H, H, N, d, base=0, device="cuda")
    o = torch.empty_like(q)
    flops = 4.0 * H * N * N * d * 0.5
    for name in a.variants.split(","):
        m, order, cl = VARIANTS[name]
        if not a.time:
            attn_fwd(q, k, v, o, causal=True, scale=1 / math.sqrt(d), mapping=m, order=order, cluster=cl)
            torch.cuda.synchronize()
            print(f"N={N} {name} launched", flush=True)
            continue
        for _ in range(2):
            attn_fwd(q, k, v, o, causal=True, scale=1 / math.sqrt(d), mapping=m, order=order, cluster=cl)
        ts = []
        for _ in range(a.reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            attn_fwd(q, k, v, o, causal=True, scale=1 / math.sqrt(d), mapping=m, order=order, cluster=cl)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        r = {"N": N, "variant": name, "ms_median": ts[len(ts) // 2], "tflops": flops / ts[len(ts) // 2] / 1e9,
             "kv_mib_per_head": 4 * N * d / 2**20}
        rows.append(r)
        print(json.dumps(r), flush=True)
    del q, k, v, o
    torch.cuda.empty_cache()
if a.json and rows:
    json.dump(rows, open(a.json, "w"), indent=1)
