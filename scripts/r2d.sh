set -u
mkdir -p gpurun_out
timeout 120 python scripts/pair_check.py --save /tmp/o_pair.pt > gpurun_out/r2d_pair.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_pair.log
ATTN_FWD_PAIR=0 timeout 120 python scripts/pair_check.py --save /tmp/o_old.pt > gpurun_out/r2d_old.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_old.log
python scripts/pair_check.py --compare /tmp/o_old.pt /tmp/o_pair.pt > gpurun_out/r2d_cmp.log 2>&1
timeout 300 python scripts/quick_bench.py --configs C2,C3 --maps swizzled_head_first,head_first,block_first > gpurun_out/r2d_qb_pair.log 2>&1
ATTN_FWD_PAIR=0 timeout 300 python scripts/quick_bench.py --configs C2,C3 --maps swizzled_head_first,head_first,block_first > gpurun_out/r2d_qb_old.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2d_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2d_pytest.log
tail -3 gpurun_out/r2d_pytest.log; cat gpurun_out/r2d_cmp.log gpurun_out/r2d_qb_pair.log gpurun_out/r2d_qb_old.log
