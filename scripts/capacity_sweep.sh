#!/bin/bash
# Capacity experiment: event-timed sweep, then one ncu
# pass per (N, variant) with the L2 / DRAM / fabric counters.  Under gpurun.
set -u
mkdir -p gpurun_out
V=${VARIANTS:-hf,shf,shf_alt}
NS=${NS:-32768,65536,98304,131072}
timeout 900 python scripts/capacity_sweep.py --time --ns $NS --variants $V --json gpurun_out/capacity_time.json \
  > gpurun_out/capacity_time.log 2>&1
timeout 1500 ncu --clock-control none --cache-control all -k regex:attn_fwd_sm100 --csv \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sector_op_read_hit_rate.pct,lts__t_sectors.sum,lts__t_sectors_srcunit_ltcfabric.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second \
  --log-file gpurun_out/capacity_ncu.csv python scripts/capacity_sweep.py --ns $NS --variants $V \
  > gpurun_out/capacity_ncu.log 2>&1
echo "ncu rc=$?"
