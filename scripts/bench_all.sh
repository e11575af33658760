#!/bin/bash
# One bench.py JSON line per workload (current build), for the record under
# profiles/bench_<round>_<W>[_bwd].json.  Run under gpurun.
R=${ROUND:-r01}
mkdir -p gpurun_out
for W in C2 C3 C4 C6; do
  timeout 600 python bench.py --workload $W --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline 2> gpurun_out/bench_${R}_$W.err | tail -1 > gpurun_out/bench_${R}_$W.json
done
timeout 900 python bench.py --workload C5 --steps 3 --warmup 3 --no-cpu-baseline 2> gpurun_out/bench_${R}_C5.err | tail -1 > gpurun_out/bench_${R}_C5.json
for W in C2 C3 C4 C6; do
  timeout 600 python bench.py --workload $W --pass bwd --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline 2> gpurun_out/bench_${R}_${W}_bwd.err | tail -1 > gpurun_out/bench_${R}_${W}_bwd.json
done
