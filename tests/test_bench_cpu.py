"""bench.py host logic on CPU: the FLOP accounting against SPEC's printed
value, the workload table against BASELINE.json, the scaling shapes, the
exp-unit ceiling, the ncu CSV unit parsing, and the reference (oracle) arm
end to end (the one bench path that runs without a GPU)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "spec_mapping_pins.json")))


def test_flops_match_spec_worked_values():
    for ex in GOLD["attention_flops"]:  # S:417, printed by SPEC
        assert bench.flops_fwd(ex["B"], ex["Hq"], ex["N"], ex["d"], False) == ex["expect"]
    # causal is half (R14), the backward counts five matmuls
    assert bench.flops_fwd(1, 2, 256, 64, True) == 0.5 * bench.flops_fwd(1, 2, 256, 64, False)
    assert bench.flops_fwd(1, 2, 256, 64, False, "bwd") == 2.5 * bench.flops_fwd(1, 2, 256, 64, False)
    # C2 1.0995e12, C5 5.6295e14 flop
    assert abs(bench.flops_fwd(*bench.WORKLOADS["C2"][:2], *bench.WORKLOADS["C2"][3:6]) - 1.0995e12) < 1e8
    assert abs(bench.flops_fwd(*bench.WORKLOADS["C5"][:2], *bench.WORKLOADS["C5"][3:6]) - 5.6295e14) < 1e11


def test_workloads_are_baseline_configs():
    cfg = json.load(open(os.path.join(ROOT, "BASELINE.json")))["configs"]
    # "MHA B=1 Hq=Hkv=128 N=131072 d=128 bf16 causal, heads sharded across 2/4/8 B200"
    assert bench.WORKLOADS["C5"][:6] == (1, 128, 128, 131072, 128, True) and "N=131072" in cfg[4]
    assert bench.WORKLOADS["C2"][:6] == (1, 32, 32, 8192, 128, False) and "N=8192" in cfg[1]
    assert bench.WORKLOADS["C4"][:6] == (2, 64, 8, 16384, 128, True) and "Hkv=8" in cfg[3]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_job_shapes(world):
    # C5 scales strongly (the 128 heads are split), C2 weakly (each rank a C2)
    B, Hq, Hkv, N, d, causal, scaling = bench.job_shape("C5", world)
    assert (Hq, Hkv, scaling) == (128, 128, "strong")
    B, Hq, Hkv, N, d, causal, scaling = bench.job_shape("C2", world)
    assert (Hq, Hkv, scaling) == (32 * world, 32 * world, "weak")


def test_ncu_units():
    assert bench._ncu_value("1,024", "Kbyte") == 1024e3
    assert bench._ncu_value("2.5", "msecond") == 2.5e-3
    assert bench._ncu_value("1.42", "Ghz") == 1.42e9
    assert bench._ncu_value("n/a", "byte") is None


def test_variant_keys():
    assert bench.variant_key("swizzled_head_first", True) == "swizzled_head_first+cluster"
    assert bench.variant_key("swizzled_head_first:per_die", False) == "swizzled_head_first:per_die"
    assert "swizzled_head_first:per_die" in bench.VARIANT_MAPS


def test_reference_arm_runs_on_cpu():
    """--impl reference: the fp64 oracle on this host's cores, the contract's
    JSON line with impl/cpu_baseline/e2e (tier framing: the oracle is the
    reference arm)."""
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "C1", "--steps", "2",
                        "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-1000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "TFLOP/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert line["steps"] == 2 and line["warmup"] == 3 and line["higher_is_better"] is True


def test_mapping_rounds_protocol():
    # C5 (~463 ms per step): one timed step after one settle step, ~2 s timed
    assert bench.mapping_rounds(463.0) == (1, 1, 4)
    # C3 (~30 ms): 10-step chunks after 5 settle steps, 7 rounds
    assert bench.mapping_rounds(30.0) == (10, 5, 7)
    # C2 (~0.82 ms): ~300 ms chunks
    chunk, settle, rounds = bench.mapping_rounds(0.82)
    assert chunk == 366 and settle == 183 and rounds == 7
    for ms in (0.01, 1.0, 50.0, 5000.0):
        c, st, r = bench.mapping_rounds(ms)
        assert c >= 1 and st >= 1 and 3 <= r <= 50
