set -u
mkdir -p gpurun_out
L=paper_2511_02132_b200/lib/variants/libattnnuma_CYC.so
ATTN_NUMA_LIB=$L timeout 120 python scripts/pair_cycles.py 1 32 32 8192 128 0 > gpurun_out/r2h_c2.log 2>&1
ATTN_NUMA_LIB=$L timeout 120 python scripts/pair_cycles.py 1 128 128 32768 128 1 > gpurun_out/r2h_c3.log 2>&1
cat gpurun_out/r2h_c2.log gpurun_out/r2h_c3.log
