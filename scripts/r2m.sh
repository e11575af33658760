set -u
mkdir -p gpurun_out
export ATTN_FWD_PAIR=1
ATTN_NUMA_LIB=paper_2511_02132_b200/lib/variants/libattnnuma_CYCX11.so timeout 120 python scripts/pair_cycles.py 1 32 32 8192 128 0 x > gpurun_out/r2m_cyc11.log 2>&1
ATTN_NUMA_LIB=paper_2511_02132_b200/lib/variants/libattnnuma_S11.so timeout 300 python scripts/quick_bench.py --configs C2,C3 --maps swizzled_head_first > gpurun_out/r2m_qb11.log 2>&1
cat gpurun_out/r2m_cyc11.log gpurun_out/r2m_qb11.log
