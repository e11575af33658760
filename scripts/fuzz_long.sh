#!/bin/bash
# Extended seeded fuzz of the forward and backward against the fp64 oracle
# (tests/test_gpu_fuzz.py with more cases), under gpurun.
set -u
mkdir -p gpurun_out
ATTN_FUZZ_CASES=${FWD:-400} ATTN_FUZZ_BWD_CASES=${BWD:-120} ATTN_FUZZ_SEED=${SEED:-20261017} \
  timeout 3000 python -m pytest tests/test_gpu_fuzz.py -q > gpurun_out/fuzz_long.log 2>&1
echo "rc=$?" >> gpurun_out/fuzz_long.log
tail -3 gpurun_out/fuzz_long.log
