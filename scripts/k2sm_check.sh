set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_parity.py -q -x > gpurun_out/k2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k2_pytest.log
for i in 1 2; do
timeout 600 python scripts/cluster_check.py C2,C3,C5 > gpurun_out/k2_cc_$i.log 2>&1
ATTN_NUMA_LIB=paper_2511_02132_b200/lib/variants/libattnnuma_MC.so timeout 600 python scripts/cluster_check.py C2,C3,C5 --no-parity > gpurun_out/k2_cc_mc_$i.log 2>&1
done
tail -3 gpurun_out/k2_pytest.log; tail -12 gpurun_out/k2_cc_1.log gpurun_out/k2_cc_mc_1.log gpurun_out/k2_cc_2.log gpurun_out/k2_cc_mc_2.log
