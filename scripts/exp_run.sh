set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_large.py -q -x -k million > gpurun_out/exp24_large.log 2>&1; echo "rc=$?" >> gpurun_out/exp24_large.log
