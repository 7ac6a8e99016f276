#!/bin/bash
# r02a: compute-sanitizer on the whole path (VERDICT r1 missing #5) and the isolated
# per-stage ncu table of a config-2 tile, cold and warm.
mkdir -p gpurun_out/r02a
O=gpurun_out/r02a
export CUDA_DEVICE_MAX_CONNECTIONS=32
python tools/sanitize_run.py > $O/plain.log 2>&1; echo "rc=$?" >> $O/plain.log
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck initcheck; do
  timeout -s KILL 600 $CS --tool $tool --print-limit 50 \
     python tools/sanitize_run.py > $O/sanitizer_$tool.log 2>&1
  echo "rc=$?" >> $O/sanitizer_$tool.log
  tail -3 $O/sanitizer_$tool.log
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
for cc in all none; do
  timeout -s KILL 900 ncu --metrics $M --cache-control $cc --clock-control none --csv \
    --kernel-name regex:hp:: --log-file $O/stages_cache_$cc.csv python tools/one_tile.py 2 > $O/stages_cache_$cc.log 2>&1
  echo "rc=$?" >> $O/stages_cache_$cc.log
done
