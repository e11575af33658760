"""bench.py's multi-rank path (torchrun, head sharding, barriers, max over
ranks, one JSON line from rank 0) exercised on ONE GPU: ATTN_BENCH_SHARE_GPU=1
puts both ranks on cuda:0 over gloo.  The 8-GPU NCCL run is the driver's."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("workload,scaling", [("C2", "weak"), ("C5", "strong")])
def test_bench_two_ranks_share_gpu(workload, scaling):
    env = dict(os.environ, ATTN_BENCH_SHARE_GPU="1")
    steps = "3" if workload == "C2" else "1"
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
                          "--steps", steps, "--warmup", "3", "--workload", workload, "--ncu", "off"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == scaling and d["gpu_launches"] == int(steps)
    rep = d["replicated_output"]  # fused peer-store epilogue over CUDA IPC (both ranks on cuda:0)
    assert "error" not in rep and rep["fused_peer_store_ms"] > 0, rep
    if workload == "C2":
        assert d["config"]["Hq"] == 64 and d["config"]["heads_per_gpu"] == 32  # weak: 32 heads per rank
    else:
        assert d["config"]["Hq"] == 128 and d["config"]["heads_per_gpu"] == 64  # strong: 128 heads split
    assert d["value"] > 0 and "cpu_baseline" not in d


def test_reference_arm_two_ranks():
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
                          "--steps", "2", "--warmup", "3", "--impl", "reference"],
                         cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["e2e"]["h2d_bytes_per_step"] == 0
