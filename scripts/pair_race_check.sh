set -u
mkdir -p gpurun_out
export ATTN_FWD_PAIR=1
for S in 1,4,4,16384,128,1 1,16,16,32768,128,1 2,16,4,8192,128,1 1,8,8,4096,128,0 1,32,32,2048,128,1; do
  timeout 120 python scripts/pair_debug.py --shape $S --reps 1 --save /tmp/ref.pt > /dev/null 2>&1
  python -c "import torch; x=torch.load('/tmp/ref.pt'); torch.save([x[0]]*8,'/tmp/ref8.pt')"
  ATTN_NUMA_LIB=paper_2511_02132_b200/lib/variants/libattnnuma_NOSYNC.so timeout 300 python scripts/pair_debug.py --shape $S --reps 8 --save /tmp/v.pt > gpurun_out/r2t_$S.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_$S.log
  python scripts/pair_debug.py --compare /tmp/v.pt /tmp/ref8.pt >> gpurun_out/r2t_$S.log 2>&1
done
grep -h "differing\|rc=" gpurun_out/r2t_*.log | sort | uniq -c
