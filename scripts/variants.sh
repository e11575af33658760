#!/bin/bash
# run quick_bench against every experimental variant library in lib/var
for so in paper_2511_02132_b200/lib/var/*.so; do
  echo "== $so"
  ATTN_NUMA_LIB=$so timeout 300 python scripts/quick_bench.py --configs ${CONFIGS:-C2,C3} --reps ${REPS:-5} 2>&1 | grep -v "^{"
done
