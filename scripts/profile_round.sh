#!/bin/bash
# ncu evidence for one round: launch list of the bench command + --set full
# captures of the attention kernel per workload x mapping.  Run under gpurun.
set -u
R=${ROUND:-r01}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$R.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches_bench_$R.log 2>&1
for W in ${WORKLOADS:-C2 C3}; do
  for M in ${MAPS:-block_first head_first swizzled_head_first swizzled_block_first}; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_sm100 -s 2 -c 1 \
      -o gpurun_out/full_${R}_${W}_${M} python scripts/one_launch.py --workload $W --mapping $M --warmup 2 \
      > gpurun_out/full_${R}_${W}_${M}.log 2>&1
    tail -1 gpurun_out/full_${R}_${W}_${M}.log
  done
done
