set -u
mkdir -p gpurun_out
timeout 600 python scripts/soak.py 300 > gpurun_out/soak_final.log 2>&1; echo "rc=$?" >> gpurun_out/soak_final.log
timeout 1200 compute-sanitizer --tool memcheck python scripts/sanitize_small.py > gpurun_out/san_mem_final.log 2>&1; echo "rc=$?" >> gpurun_out/san_mem_final.log
timeout 1200 compute-sanitizer --tool synccheck python scripts/sanitize_small.py > gpurun_out/san_sync_final.log 2>&1; echo "rc=$?" >> gpurun_out/san_sync_final.log
