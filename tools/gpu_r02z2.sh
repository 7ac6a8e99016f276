#!/bin/bash
# ncu --set full of the CCL-select kernels and the feature-stage Canny on one config-2 tile
O=gpurun_out/r02z2; mkdir -p $O
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k 'regex:k_canny_nms|k_cs_' -s 18 -c 18 -o $O/ncu_ccls python tools/one_tile.py 2 > $O/ncu.log 2>&1; echo "rc=$?"
ncu -i $O/ncu_ccls.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread > $O/raw.csv 2>&1
tail -3 $O/ncu.log
