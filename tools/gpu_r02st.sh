#!/bin/bash
# per-stage ncu table of one config-2 tile at the final build (cold / warm caches)
O=gpurun_out/r02st; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
for cc in all none; do
  timeout -s KILL 600 ncu --metrics $M --cache-control $cc --clock-control none --csv \
    --kernel-name regex:^k_ --log-file $O/stages_cache_$cc.csv python tools/one_tile.py 2 > $O/stages_cache_$cc.log 2>&1
  echo "rc=$?"
done
python tools/stage_table.py $O/stages_cache_all.csv $O/stages_cache_none.csv $O/stage_table
cat $O/stage_table.md
