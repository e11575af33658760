set -u
L=paper_2511_02132_b200/lib/variants/libattnnuma_CYCX.so
ATTN_NUMA_LIB=$L timeout 120 python scripts/pair_cycles.py 1 32 32 8192 128 0 x
