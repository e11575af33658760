set -u
mkdir -p gpurun_out
S=1,4,4,16384,128,1
ATTN_FWD_PAIR=0 timeout 120 python scripts/pair_debug.py --shape $S --reps 1 --save /tmp/ref.pt > /dev/null 2>&1
python - <<'PY'
import torch; x=torch.load('/tmp/ref.pt'); torch.save([x[0]]*6,'/tmp/ref6.pt')
PY
for V in default WGS1 USYNC; do
  if [ $V = default ]; then L=""; else L=paper_2511_02132_b200/lib/variants/libattnnuma_$V.so; fi
  ATTN_NUMA_LIB=$L timeout 120 python scripts/pair_debug.py --shape $S --reps 6 --save /tmp/v.pt > gpurun_out/r2f_$V.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_$V.log
  python scripts/pair_debug.py --compare /tmp/v.pt /tmp/ref6.pt >> gpurun_out/r2f_$V.log 2>&1
  ATTN_NUMA_LIB=$L timeout 120 python scripts/quick_bench.py --configs C3 --maps block_first,swizzled_head_first --reps 5 >> gpurun_out/r2f_$V.log 2>&1; echo "qb rc=$?" >> gpurun_out/r2f_$V.log
done
tail -n 40 gpurun_out/r2f_*.log
