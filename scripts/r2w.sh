set -u
mkdir -p gpurun_out
timeout 300 python scripts/soak.py 150 > gpurun_out/soak_r02.txt 2>&1; echo "rc=$?" >> gpurun_out/soak_r02.txt
timeout 900 compute-sanitizer --tool memcheck python scripts/sanitize_small.py > gpurun_out/sanitizer_memcheck_r02.txt 2>&1
timeout 900 compute-sanitizer --tool synccheck python scripts/sanitize_small.py > gpurun_out/sanitizer_synccheck_r02.txt 2>&1
ATTN_FWD_PAIR=1 timeout 900 compute-sanitizer --tool memcheck python scripts/sanitize_small.py > gpurun_out/sanitizer_memcheck_pair_r02.txt 2>&1
tail -3 gpurun_out/soak_r02.txt gpurun_out/sanitizer_*_r02.txt
