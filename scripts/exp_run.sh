set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/exp16_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/exp16_pytest.log
timeout 900 python bench.py --workload C6 > gpurun_out/exp16_bench_C6.json 2> gpurun_out/exp16_bench_C6.err
