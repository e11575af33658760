set -u
mkdir -p gpurun_out
export ATTN_FWD_PAIR=1
L=paper_2511_02132_b200/lib/variants/libattnnuma_CYCX.so
ATTN_NUMA_LIB=$L timeout 120 python scripts/pair_cycles.py 1 32 32 8192 128 0 x > gpurun_out/r2n_cyc.log 2>&1
timeout 300 python scripts/quick_bench.py --configs C2,C3 --maps swizzled_head_first,head_first,block_first > gpurun_out/r2n_qb.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2n_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2n_pytest.log
cat gpurun_out/r2n_cyc.log gpurun_out/r2n_qb.log; tail -15 gpurun_out/r2n_pytest.log
