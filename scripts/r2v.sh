set -u
mkdir -p gpurun_out
export ATTN_FWD_PAIR=1
ATTN_NUMA_LIB=paper_2511_02132_b200/lib/variants/libattnnuma_CYCX.so timeout 120 python scripts/pair_cycles.py 1 32 32 8192 128 0 x > gpurun_out/r2v_cyc.log 2>&1
for S in 1,16,16,32768,128,1 1,8,8,4096,128,0; do
  ATTN_NUMA_LIB=paper_2511_02132_b200/lib/variants/libattnnuma_NOSPEC.so timeout 120 python scripts/pair_debug.py --shape $S --reps 1 --save /tmp/ref.pt > /dev/null 2>&1
  python -c "import torch; x=torch.load('/tmp/ref.pt'); torch.save([x[0]]*3,'/tmp/ref3.pt')"
  timeout 300 python scripts/pair_debug.py --shape $S --reps 3 --save /tmp/v.pt > gpurun_out/r2v_$S.log 2>&1
  python scripts/pair_debug.py --compare /tmp/v.pt /tmp/ref3.pt >> gpurun_out/r2v_$S.log 2>&1
done
timeout 300 python scripts/quick_bench.py --configs C2,C3 --maps swizzled_head_first > gpurun_out/r2v_qb.log 2>&1
ATTN_FWD_PAIR=0 timeout 300 python scripts/quick_bench.py --configs C2,C3 --maps swizzled_head_first > gpurun_out/r2v_qb_old.log 2>&1
timeout 600 python -m pytest tests/test_gpu_pair.py -q > gpurun_out/r2v_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2v_pytest.log
cat gpurun_out/r2v_cyc.log; grep -h "differing" gpurun_out/r2v_1*.log; grep -h "C[23] " gpurun_out/r2v_qb*.log; tail -2 gpurun_out/r2v_pytest.log
