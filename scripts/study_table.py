"""Print DESIGN.md's mapping-study table from the committed ncu summaries
(profiles/ncu_<cfg>_<mapping>.json)."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from bench import WORKLOADS  # noqa: E402

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles")
NAMES = {"block_first": "block-first", "head_first": "head-first", "swizzled_head_first": "**SHF**",
         "swizzled_block_first": "swizzled block-first"}
print("| cfg | mapping | ms | L2 hit % | DRAM GB/launch | cross-die GB | tensor % | SM GHz | TFLOP/s |")
print("|---|---|---|---|---|---|---|---|---|")
for cfg in ("C2", "C3", "C4", "C5", "C6"):
    B, Hq, Hkv, N, d, causal, _ = WORKLOADS[cfg]
    flops = 4 * B * Hq * N * N * d * (0.5 if causal else 1.0)
    for m, name in NAMES.items():
        path = os.path.join(ROOT, f"ncu_{cfg}_{m}.json")
        if not os.path.exists(path):
            continue
        s = json.load(open(path))
        ms = s["gpu__time_duration.sum"] * 1e3
        fabric = s.get("lts__t_sectors_srcunit_ltcfabric.sum")
        tensor = s.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")
        ghz = s["sm__cycles_elapsed.avg.per_second"]
        ghz = ghz if ghz < 100 else ghz / 1e9
        print(f"| {cfg} | {name} | {ms:.3f} | {s['lts__t_sector_hit_rate.pct']:.1f} | "
              f"{s['dram_bytes_per_launch'] / 1e9:.2f} | {fabric * 32 / 1e9:.1f} | "
              f"{tensor:.1f} | {ghz:.2f} | {flops / (ms * 1e-3) / 1e12:.0f} |" if fabric is not None and tensor is not None
              else f"| {cfg} | {name} | {ms:.3f} | {s['lts__t_sector_hit_rate.pct']:.1f} | "
                   f"{s['dram_bytes_per_launch'] / 1e9:.2f} | — | — | {ghz:.2f} | {flops / (ms * 1e-3) / 1e12:.0f} |")
