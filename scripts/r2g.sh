set -u
mkdir -p gpurun_out
timeout 120 python scripts/pair_check.py --save /tmp/o_pair.pt > gpurun_out/r2g_pair.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_pair.log
ATTN_FWD_PAIR=0 timeout 120 python scripts/pair_check.py --save /tmp/o_old.pt > gpurun_out/r2g_old.log 2>&1
python scripts/pair_check.py --compare /tmp/o_old.pt /tmp/o_pair.pt > gpurun_out/r2g_cmp.log 2>&1
S=1,4,4,16384,128,1
ATTN_FWD_PAIR=0 timeout 120 python scripts/pair_debug.py --shape $S --reps 1 --save /tmp/ref.pt > /dev/null 2>&1
python -c "import torch; x=torch.load('/tmp/ref.pt'); torch.save([x[0]]*6,'/tmp/ref6.pt')"
timeout 120 python scripts/pair_debug.py --shape $S --reps 6 --save /tmp/v.pt > gpurun_out/r2g_dbg.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_dbg.log
python scripts/pair_debug.py --compare /tmp/v.pt /tmp/ref6.pt >> gpurun_out/r2g_dbg.log 2>&1
timeout 300 python scripts/quick_bench.py --configs C2,C3 --maps swizzled_head_first,head_first,block_first > gpurun_out/r2g_qb.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_qb.log
cat gpurun_out/r2g_pair.log | tail -4; cat gpurun_out/r2g_cmp.log gpurun_out/r2g_dbg.log gpurun_out/r2g_qb.log
