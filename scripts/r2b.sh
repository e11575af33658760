set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b_pytest.log
timeout 900 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo "bench rc=$?" >> gpurun_out/r2b_bench.err
VARIANTS=hf,shf_pd,shf_sh NS=65536,98304,131072 bash scripts/capacity_sweep.sh
bash scripts/l2_capacity.sh
tail -n 3 gpurun_out/r2b_pytest.log
