#!/bin/bash
# ncu evidence for one round (run under gpurun): launch list of the bench
# command + --set full captures of the attention kernel per workload x
# mapping, summarised ON THE BOX into gpurun_out/ncu_<W>_<M>.json (the raw
# reports are deleted except KEEP ones: gpurun returns at most 64 MiB).
set -u
R=${ROUND:-r01}
KEEP=${KEEP:-"C2_swizzled_head_first C3_swizzled_head_first"}
# CLUSTER=1: profile the CTA-pair multicast variant (files ncu_<W>_<M>_cluster.json)
if [ "${CLUSTER:-0}" = 1 ]; then CLF="--cluster"; SUF="_cluster"; else CLF=""; SUF=""; fi
mkdir -p gpurun_out
if [ "${SKIP_LAUNCHES:-0}" != 1 ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$R.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches_bench_$R.log 2>&1
fi
for W in ${WORKLOADS:-C2 C3}; do
  for M in ${MAPS:-block_first head_first swizzled_head_first swizzled_block_first}; do
    rep=gpurun_out/full_${R}_${W}_${M}${SUF}
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_sm100 -s 2 -c 1 \
      -o $rep python scripts/one_launch.py --workload $W --mapping $M --warmup 2 $CLF > $rep.log 2>&1
    python scripts/ncu_summarize.py $rep.ncu-rep gpurun_out/ncu_${W}_${M}${SUF}.json \
      "{\"workload\": \"$W\", \"mapping\": \"$M\", \"cluster\": ${CLUSTER:-0}, \"round\": \"$R\", \"command\": \"ncu --set full --clock-control none -k regex:attn_fwd_sm100 -s 2 -c 1 python scripts/one_launch.py --workload $W --mapping $M --warmup 2 $CLF\"}"
    case " $KEEP " in *" ${W}_${M}${SUF} "*) ;; *) rm -f $rep.ncu-rep ;; esac
  done
done
