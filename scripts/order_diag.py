"""Diagnose order/cluster launch timing at one workload: each variant timed
alone (3 launches) and right after a different variant, outputs compared bit
for bit with the plain SHF ascending result."""
import sys

import torch

sys.path.insert(0, ".")
from bench import WORKLOADS
from paper_2511_02132_b200 import attn_fwd, attn_init, attn_last_launch_info, synth

W = sys.argv[1] if len(sys.argv) > 1 else "C3"
B, Hq, Hkv, N, d, causal, _ = WORKLOADS[W]
attn_init(0)
q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=0, device="cuda")
ref = attn_fwd(q, k, v, causal=causal, mapping="swizzled_head_first")
flops = 4 * B * Hq * N * N * d * (0.5 if causal else 1.0)


def run(m, od, cl, tag):
    o = torch.full_like(q, float("nan"))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    attn_fwd(q, k, v, o, causal=causal, mapping=m, order=od, cluster=cl)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1)
    same = torch.equal(o.view(torch.int16), ref.view(torch.int16))
    print(f"{tag:28s} {m:20s} {od:10s} cl={int(cl)} {t:8.3f} ms {flops / t / 1e9:7.1f} TF/s same={same} "
          f"{ {k_: v_ for k_, v_ in attn_last_launch_info().items() if k_ in ('n_queues', 'shf_acc_shared', 'grid', 'cluster')} }",
          flush=True)


for _ in range(3):
    run("swizzled_head_first", "ascending", True, "alone")
for _ in range(3):
    run("swizzled_head_first", "ascending", False, "alone")
for _ in range(2):
    run("block_first", "descending", False, "prev")
    run("swizzled_head_first", "ascending", True, "after BF desc")
for _ in range(2):
    run("swizzled_head_first", "descending", True, "prev")
    run("swizzled_head_first", "ascending", True, "after SHF cl desc")
for _ in range(3):
    run("swizzled_head_first", "descending", True, "alone")
