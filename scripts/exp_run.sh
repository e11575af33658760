set -u
mkdir -p gpurun_out
rm -f /tmp/vref.pt
ATTN_NUMA_LIB=paper_2511_02132_b200/lib/var/base.so VARIANT_REF=/tmp/vref.pt timeout 300 python scripts/variant_check.py > gpurun_out/exp17_check.log 2>&1
ATTN_NUMA_LIB=paper_2511_02132_b200/lib/var2/grp128.so VARIANT_REF=/tmp/vref.pt timeout 300 python scripts/variant_check.py >> gpurun_out/exp17_check.log 2>&1
for r in 1 2 3; do for v in var/base var2/grp128; do echo "== $v" ; ATTN_NUMA_LIB=paper_2511_02132_b200/lib/$v.so timeout 300 python scripts/quick_bench.py --configs C2,C3 --reps 5 --maps swizzled_head_first 2>&1 | grep -v '^{'; done; done > gpurun_out/exp17_bench.log 2>&1
