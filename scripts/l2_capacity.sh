#!/bin/bash
# L2 capacity per die: timed sweep, then ncu DRAM bytes per launch.  Under gpurun.
set -u
mkdir -p gpurun_out
timeout 600 python scripts/l2_capacity.py --json gpurun_out/l2cap_time.json > gpurun_out/l2cap_time.log 2>&1
timeout 900 ncu --csv --print-units base --clock-control none --cache-control all -k regex:l2cap_kernel \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_ltcfabric.sum,lts__t_sectors.sum \
  --log-file gpurun_out/l2cap_ncu.csv python scripts/l2_capacity.py > gpurun_out/l2cap_ncu.log 2>&1
echo "l2cap ncu rc=$?"
