set -u
mkdir -p gpurun_out
for r in 1 2; do for v in noph1 noph1e4 ph1 ph1e4 ph1e3 ph1e2; do echo "== $v" ; ATTN_NUMA_LIB=paper_2511_02132_b200/lib/var/$v.so timeout 300 python scripts/quick_bench.py --configs C2,C3 --reps 5 --maps swizzled_head_first 2>&1 | grep -v '^{'; done; done > gpurun_out/exp14_bench.log 2>&1
