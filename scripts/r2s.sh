set -u
mkdir -p gpurun_out
R=r02
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${R}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${R}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${R}_smoke.log
timeout 900 python bench.py > gpurun_out/${R}_bench_C5.json 2> gpurun_out/${R}_bench_C5.err
timeout 600 python bench.py --workload C3 --steps 20 > gpurun_out/${R}_bench_C3.json 2> gpurun_out/${R}_bench_C3.err
timeout 600 python bench.py --workload C2 --steps 100 > gpurun_out/${R}_bench_C2.json 2> gpurun_out/${R}_bench_C2.err
timeout 600 python bench.py --workload C4 --steps 20 --no-cpu-baseline > gpurun_out/${R}_bench_C4.json 2> gpurun_out/${R}_bench_C4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${R}.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --ncu off --no-replicated > gpurun_out/launches_bench_${R}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_sm100 -s 2 -c 1 -o gpurun_out/full_${R}_C5_shf_cluster \
  python scripts/one_launch.py --workload C5 --mapping swizzled_head_first --warmup 2 --cluster > gpurun_out/full_${R}_C5.log 2>&1
python scripts/ncu_summarize.py gpurun_out/full_${R}_C5_shf_cluster.ncu-rep gpurun_out/ncu_C5_swizzled_head_first_cluster_${R}.json \
  "{\"workload\": \"C5\", \"mapping\": \"swizzled_head_first\", \"cluster\": 1, \"round\": \"$R\", \"command\": \"ncu --set full --clock-control none -k regex:attn_fwd_sm100 -s 2 -c 1 python scripts/one_launch.py --workload C5 --mapping swizzled_head_first --warmup 2 --cluster\"}" > /dev/null 2>&1
tail -n 3 gpurun_out/${R}_pytest.log gpurun_out/${R}_smoke.log
for w in C5 C3 C2 C4; do python -c "
import json; d=json.load(open('gpurun_out/${R}_bench_$w.json')); print('$w', d['value'], d['roofline']['frac'], d['roofline']['frac_of_burst'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
