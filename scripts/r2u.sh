set -u
mkdir -p gpurun_out
for i in 1 2; do
timeout 300 python scripts/quick_bench.py --configs C2,C3,C6 --maps swizzled_head_first --reps 10 > gpurun_out/r2u_split_$i.log 2>&1
ATTN_NUMA_LIB=paper_2511_02132_b200/lib/variants/libattnnuma_NOSPLIT.so timeout 300 python scripts/quick_bench.py --configs C2,C3,C6 --maps swizzled_head_first --reps 10 > gpurun_out/r2u_nosplit_$i.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cluster.py tests/test_gpu_fuzz.py -q > gpurun_out/r2u_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_pytest.log
grep -h "C[236] " gpurun_out/r2u_*split_*.log; tail -3 gpurun_out/r2u_pytest.log
