set -u
mkdir -p gpurun_out
timeout 900 python bench.py --workload C3 --no-cpu-baseline > gpurun_out/exp22_C3.json 2> gpurun_out/exp22_C3.err
