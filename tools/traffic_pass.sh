#!/usr/bin/env bash
# The ncu metrics pass of tools/measure_round.sh alone: DRAM bytes, duration,
# DRAM throughput % and DMMA pipe % of every config's and row's kernel
# (one launch each), summarised into gpurun_out/traffic.json.
#   gpurun -- 'bash tools/traffic_pass.sh r02'
set -u
R=${1:-r02}
O=gpurun_out
mkdir -p $O
timeout 900 python tools/profile_all.py > $O/profile_order_plain.log 2>&1 || { tail -3 $O/profile_order_plain.log; exit 1; }
timeout 1800 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none --csv --log-file $O/traffic_$R.csv python tools/profile_all.py \
  > $O/profile_order.log 2>&1
echo "ncu rc=$?"
python tools/ncu_summary.py traffic $O/traffic_$R.csv $O/profile_order.log $O/traffic.json
