"""Cluster-multicast forward (ATTN_CLUSTER_MULTICAST) vs the plain path:
bit-identical outputs on small / ragged / causal / GQA shapes, then timing."""
import sys
import torch

sys.path.insert(0, ".")
from bench import WORKLOADS
from paper_2511_02132_b200 import api, attn_fwd, synth

cases = [(1, 2, 2, 256, 128, False), (1, 2, 2, 384, 128, True), (2, 4, 2, 1000, 128, True),
         (1, 3, 1, 77, 64, False), (1, 2, 2, 640, 56, True), (2, 8, 8, 2048, 128, True), (1, 1, 1, 1, 128, True)]
for (B, Hq, Hkv, N, d, causal) in (cases if "--no-parity" not in sys.argv else []):
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=0, device="cuda")
    for m in ("block_first", "head_first", "swizzled_head_first", "swizzled_block_first"):
        o0 = attn_fwd(q, k, v, causal=causal, mapping=m)
        o1 = attn_fwd(q, k, v, causal=causal, mapping=m, cluster=True)
        torch.cuda.synchronize()
        same = torch.equal(o0.view(torch.int16), o1.view(torch.int16))
        print(f"{(B, Hq, Hkv, N, d, causal)} {m:22s} bit-identical={same} grid={api.attn_last_launch_info()['grid']}",
              flush=True)
        assert same
args = [x for x in sys.argv[1:] if not x.startswith("--")]
names = args[0].split(",") if args else ["C2", "C3", "C5"]
for name in names:
    B, Hq, Hkv, N, d, causal, _ = WORKLOADS[name]
    q, k, v = synth.make_qkv(B, Hq, Hkv, N, d, base=0, device="cuda")
    o = torch.empty_like(q)
    flops = 4 * B * Hq * N * N * d * (0.5 if causal else 1.0)
    for m in ("block_first", "head_first", "swizzled_head_first", "swizzled_block_first"):
        for cl in (False, True):
            for _ in range(2):
                attn_fwd(q, k, v, o, causal=causal, mapping=m, cluster=cl)
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                attn_fwd(q, k, v, o, causal=causal, mapping=m, cluster=cl)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ts.sort()
            g = api.attn_last_launch_info()["grid"]
            print(f"{name} {m:22s} cluster={int(cl)} grid={g:3d} {ts[2]:9.3f} ms {flops / ts[2] / 1e9:7.1f} TFLOP/s "
                  f"(min {flops / ts[0] / 1e9:7.1f}, max {flops / ts[-1] / 1e9:7.1f})", flush=True)
