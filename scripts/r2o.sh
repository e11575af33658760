set -u
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_fwd_sm100 -s 2 -c 1 -o gpurun_out/r2o_c2_old python scripts/one_launch.py --workload C2 > gpurun_out/r2o_ncu.log 2>&1
ATTN_FWD_PAIR=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_fwd_pair -s 2 -c 1 -o gpurun_out/r2o_c2_pair python scripts/one_launch.py --workload C2 >> gpurun_out/r2o_ncu.log 2>&1
ls -la gpurun_out/*.ncu-rep; tail -5 gpurun_out/r2o_ncu.log
