set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_graph.py -q -x > gpurun_out/exp23_graph.log 2>&1; echo "rc=$?" >> gpurun_out/exp23_graph.log
