set -u
mkdir -p gpurun_out
for e in 4 6 8 12 16; do
  if [ $e = 8 ]; then L=""; else L=paper_2511_02132_b200/lib/variants/libattnnuma_E$e.so; fi
  echo "EMU $e" >> gpurun_out/r2r_qb.log
  ATTN_NUMA_LIB=$L timeout 300 python scripts/quick_bench.py --configs C6 --maps swizzled_head_first >> gpurun_out/r2r_qb.log 2>&1
done
timeout 600 python bench.py --workload C3 --pass bwd --steps 10 --no-cpu-baseline > gpurun_out/r2r_bwd_c3.json 2> gpurun_out/r2r_bwd_c3.err
timeout 600 python bench.py --workload C6 --steps 10 --no-cpu-baseline > gpurun_out/r2r_c6.json 2> gpurun_out/r2r_c6.err
grep -v num_sms gpurun_out/r2r_qb.log; python -c "
import json
for f in ('gpurun_out/r2r_bwd_c3.json','gpurun_out/r2r_c6.json'):
    d=json.load(open(f)); print(f, d['value'], d['roofline']['frac'], d['roofline']['frac_of_burst'], d['roofline']['peak_source'][:60])
"
