#!/bin/bash
O=gpurun_out/r02cn; mkdir -p $O
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k 'regex:k_canny_nms|k_cs_local' -s 4 -c 4 -o $O/ncu_cn python tools/one_tile.py 2 > $O/ncu.log 2>&1; echo "rc=$?"
ncu -i $O/ncu_cn.ncu-rep --page source --csv --print-source cuda,sass > $O/mix.csv 2>&1
ncu -i $O/ncu_cn.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active > $O/raw.csv 2>&1
