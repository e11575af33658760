#!/bin/bash
# End-of-round evidence in one gpurun call: GPU tests, smoke, the default bench
# line (C5) and the oracle arm, per-workload lines (forward C2/C3/C4/C6,
# backward C2/C3/C6), the seeded long fuzz, the ncu launch list of the default
# bench command and one `ncu --set full` capture of the C5 value variant.
# Everything lands in gpurun_out/final_*.
set -u
mkdir -p gpurun_out
R=${ROUND:-r02f}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench_C5.json 2> gpurun_out/final_bench_C5.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
for W in C2 C3 C4 C6; do
  timeout 600 python bench.py --workload $W --no-cpu-baseline > gpurun_out/final_bench_$W.json 2> gpurun_out/final_bench_$W.err
done
for W in C2 C3 C6; do
  timeout 600 python bench.py --workload $W --pass bwd --no-cpu-baseline > gpurun_out/final_bench_${W}_bwd.json 2> gpurun_out/final_bench_${W}_bwd.err
done
ATTN_FUZZ_CASES=400 ATTN_FUZZ_BWD_CASES=120 ATTN_FUZZ_SEED=20261018 \
  timeout 1800 python -m pytest tests/test_gpu_fuzz.py -q > gpurun_out/final_fuzz.log 2>&1; echo "rc=$?" >> gpurun_out/final_fuzz.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --ncu off \
  > gpurun_out/final_launches_bench.log 2>&1
rep=gpurun_out/final_full_C5_shf_cluster
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_sm100 -s 2 -c 1 \
  -o $rep python scripts/one_launch.py --workload C5 --mapping swizzled_head_first --warmup 2 --cluster > $rep.log 2>&1
python scripts/ncu_summarize.py $rep.ncu-rep gpurun_out/final_ncu_C5_swizzled_head_first_cluster.json \
  "{\"workload\": \"C5\", \"mapping\": \"swizzled_head_first\", \"cluster\": 1, \"round\": \"$R\", \"command\": \"ncu --set full --clock-control none -k regex:attn_fwd_sm100 -s 2 -c 1 python scripts/one_launch.py --workload C5 --mapping swizzled_head_first --warmup 2 --cluster\"}" \
  > gpurun_out/final_ncu_summarize.log 2>&1
rm -f $rep.ncu-rep
tail -n 2 gpurun_out/final_pytest.log gpurun_out/final_smoke.log gpurun_out/final_fuzz.log
