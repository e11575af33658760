set -u
mkdir -p gpurun_out
L=paper_2511_02132_b200/lib/variants/libattnnuma_CYCX.so
ATTN_NUMA_LIB=$L timeout 120 python scripts/pair_cycles.py 1 32 32 8192 128 0 x > gpurun_out/r2j_cyc.log 2>&1
timeout 120 python scripts/pair_check.py --save /tmp/o_pair.pt > gpurun_out/r2j_pair.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_pair.log
ATTN_FWD_PAIR=0 timeout 120 python scripts/pair_check.py --save /tmp/o_old.pt > /dev/null 2>&1
python scripts/pair_check.py --compare /tmp/o_old.pt /tmp/o_pair.pt > gpurun_out/r2j_cmp.log 2>&1; echo "cmp rc=$?" >> gpurun_out/r2j_cmp.log
timeout 300 python scripts/quick_bench.py --configs C2,C3 --maps swizzled_head_first,head_first,block_first > gpurun_out/r2j_qb.log 2>&1
cat gpurun_out/r2j_cyc.log; tail -2 gpurun_out/r2j_cmp.log; cat gpurun_out/r2j_qb.log
