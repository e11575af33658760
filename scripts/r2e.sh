set -u
mkdir -p gpurun_out
for S in 1,16,16,32768,128,1 1,4,4,16384,128,1 1,2,2,8192,128,1; do
  timeout 120 python scripts/pair_debug.py --shape $S --save /tmp/a.pt > gpurun_out/r2e_a_$S.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_a_$S.log
  ATTN_FWD_PAIR=0 timeout 120 python scripts/pair_debug.py --shape $S --save /tmp/b.pt > gpurun_out/r2e_b_$S.log 2>&1
  python scripts/pair_debug.py --compare /tmp/a.pt /tmp/b.pt >> gpurun_out/r2e_a_$S.log 2>&1
done
timeout 300 compute-sanitizer --tool memcheck python scripts/pair_debug.py --shape 1,2,2,8192,128,1 --reps 1 --save /tmp/c.pt > gpurun_out/r2e_memcheck.log 2>&1
tail -n 30 gpurun_out/r2e_*.log
