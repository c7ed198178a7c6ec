#!/bin/bash
# HBM-bound kernels at >= 256 MB: one C2-model step with V = 10^5 under ncu,
# per-kernel duration and DRAM bytes (the 2nd step's launches).
o=gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
  --clock-control none --csv --log-file $o/hbm_large.csv python scripts/run_c2.py 2 c2big > $o/hbm_large.log 2>&1
echo "rc=$?"
