set -u
mkdir -p gpurun_out
for v in cyc_base cyc_shs2; do echo "== $v"; ATTN_NUMA_LIB=paper_2511_02132_b200/lib/var5/$v.so timeout 300 python scripts/cycles.py 1 32 32 8192 128 0; done > gpurun_out/exp30_cycles.log 2>&1
