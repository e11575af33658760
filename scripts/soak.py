"""Soak test: many back-to-back launches over mixed shapes, mappings, unit
orders, cluster and head dims, each compared bit for bit with the first
result of its shape (rare protocol races would show up as mismatches).

    python scripts/soak.py [seconds]
"""
import random
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2511_02132_b200 import attn_bwd, attn_fwd, attn_fwd_lse, synth

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = random.Random(7)
shapes = []
for _ in range(24):
    Hkv = rng.choice([1, 2, 4, 8])
    G = rng.choice([1, 2, 4])
    shapes.append((rng.randint(1, 2), Hkv * G, Hkv, rng.choice([129, 1000, 2048, 4097]), rng.choice([56, 64, 128]),
                   rng.random() < 0.5))
data = {}
for s in shapes:
    B, Hq, Hkv, N, d, causal = s
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=hash(s) & 0xFFFF, device="cuda")
    ref = attn_fwd(q, k, v, causal=causal, mapping="block_first")
    data[s] = (q, k, v, ref)
maps = ["block_first", "head_first", "swizzled_head_first", "swizzled_block_first", "swizzled_head_first:shared",
        "swizzled_head_first:per_die"]
n = bad = 0
t0 = time.time()
outs = []
while time.time() - t0 < secs:
    s = rng.choice(shapes)
    q, k, v, ref = data[s]
    o = attn_fwd(q, k, v, causal=s[5], mapping=rng.choice(maps), order=rng.choice(["ascending", "descending"]),
                 cluster=rng.random() < 0.3)
    outs.append((s, o))
    n += 1
    if len(outs) >= 64:
        torch.cuda.synchronize()
        for s2, o2 in outs:
            if not torch.equal(o2.view(torch.int16), data[s2][3].view(torch.int16)):
                bad += 1
                print("MISMATCH", s2, flush=True)
        outs.clear()
torch.cuda.synchronize()
for s2, o2 in outs:
    if not torch.equal(o2.view(torch.int16), data[s2][3].view(torch.int16)):
        bad += 1
        print("MISMATCH", s2, flush=True)
# backward: repeated launches against the first result
s = (2, 8, 2, 2048, 128, True)
q, k, v = synth.make_qkv(*s[:5], base=5, device="cuda")
do = synth.make_tensor("q", 2, 8, 2048, 128, base=6, device="cuda")
o, lse = attn_fwd_lse(q, k, v, causal=True)
r = attn_bwd(q, k, v, o, do, lse, causal=True)
nb = 0
for i in range(200):
    g = attn_bwd(q, k, v, o, do, lse, causal=True, mapping=maps[i % 4])
    nb += 1
    if any(not torch.equal(a.view(torch.int16), b.view(torch.int16)) for a, b in zip(g, r)):
        bad += 1
        print("BWD MISMATCH", i, flush=True)
torch.cuda.synchronize()
print(f"soak: {n} forward + {nb} backward launches in {time.time() - t0:.0f} s, {bad} mismatches")
