set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2p_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2p_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2p_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2p_smoke.log
timeout 900 python bench.py > gpurun_out/r2p_bench.json 2> gpurun_out/r2p_bench.err; echo "bench rc=$?" >> gpurun_out/r2p_bench.err
VARIANTS=hf,shf_pd,shf_sh NS=98304,131072 bash scripts/capacity_sweep.sh
tail -n 3 gpurun_out/r2p_pytest.log gpurun_out/r2p_smoke.log gpurun_out/r2p_bench.err
