"""The NCCL branches of the multi-GPU path, executed on ONE GPU: torchrun with
a world of one rank and the NCCL backend (NCCL refuses two ranks on one
device, so world 1 is what a one-GPU box can run).  bench.py --replicated
times the fused peer-store epilogue (attn_fwd_replicated) against the forward
followed by dist.all_gather_heads, whose NCCL branch is
all_gather_into_tensor (heads are independent, so the gathered
output must equal the fused one bit for bit).  The 8-GPU run is the driver's."""
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


def test_nccl_world1_replicated_output_bit_identical():
    env = dict(os.environ)
    env.pop("ATTN_BENCH_SHARE_GPU", None)
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                          "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "1",
                          "--workload", "C2", "--steps", "3", "--warmup", "3", "--replicated", "--ncu", "off",
                          "--no-cpu-baseline"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    rep = d["replicated_output"]
    assert "error" not in rep, rep
    assert rep["allgather_backend"] == "nccl", rep
    assert rep["fwd_then_nccl_allgather_ms"] > 0 and rep["fused_peer_store_ms"] > 0
    assert rep["bit_identical"] is True
    # NCCL itself ran and announced itself (NCCL_DEBUG=INFO scoped to INIT by dist.init)
    assert "NCCL version" in out.stdout + out.stderr


def test_nccl_world1_all_gather_heads_direct(tmp_path):
    """dist.all_gather_heads under NCCL equals its input at world 1 (the
    collective runs; it is not short-circuited when a process group exists)."""
    code = r"""
import os, torch, torch.distributed as dist, sys
sys.path.insert(0, ROOT_DIR)
from paper_2511_02132_b200 import dist as pdist, attn_fwd, synth
r, w, local = pdist.init(force=True)
assert dist.is_initialized() and dist.get_backend() == "nccl" and w == 1
q, k, v = synth.make_qkv(1, 4, 4, 512, 128, base=3, device="cuda")
o = attn_fwd(q, k, v, causal=True)
g = pdist.all_gather_heads(o, w)
torch.cuda.synchronize()
assert g.data_ptr() != o.data_ptr() and torch.equal(g.view(torch.int16), o.view(torch.int16))
dist.destroy_process_group()
print("OK")
"""
    script = tmp_path / "nccl_gather.py"
    script.write_text(code.replace("ROOT_DIR", repr(ROOT)))
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                          "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(script)],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "OK" in out.stdout, out.stderr[-3000:]
