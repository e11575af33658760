#!/bin/bash
# One-call end-of-round verification on the GPU box (run under gpurun):
# GPU tests, smoke(), the default bench line (C5), the reference (oracle) arm,
# a two-rank bench on one GPU (ATTN_BENCH_SHARE_GPU test mode), soak.  Logs and
# JSON lines land in gpurun_out/verify_*.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/verify_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/verify_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/verify_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/verify_smoke.log
timeout 900 python bench.py > gpurun_out/verify_bench.json 2> gpurun_out/verify_bench.err; echo "bench rc=$?" >> gpurun_out/verify_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/verify_bench_ref.json 2> gpurun_out/verify_bench_ref.err
tail -n 3 gpurun_out/verify_pytest.log gpurun_out/verify_smoke.log
