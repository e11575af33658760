set -u
mkdir -p gpurun_out
timeout 300 python scripts/quick_bench.py --configs C6 --maps swizzled_head_first,head_first,block_first > gpurun_out/r2q_qb_ones.log 2>&1
ATTN_ONES_L=0 timeout 300 python scripts/quick_bench.py --configs C6 --maps swizzled_head_first,head_first,block_first > gpurun_out/r2q_qb_fadd.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2q_pytest.log
cat gpurun_out/r2q_qb_ones.log gpurun_out/r2q_qb_fadd.log; tail -12 gpurun_out/r2q_pytest.log
