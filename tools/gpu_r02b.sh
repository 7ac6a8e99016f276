#!/bin/bash
# r02b: full GPU suite (with the new hot-path stage and bench-config parity tests), the
# default bench line, and the per-stage ncu table of one config-2 tile (cold / warm caches)
O=gpurun_out/r02b; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
timeout -s KILL 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
tail -c 600 $O/bench.json
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
for cc in all none; do
  timeout -s KILL 600 ncu --metrics $M --cache-control $cc --clock-control none --csv \
    --kernel-name regex:^k_ --log-file $O/stages_cache_$cc.csv python tools/one_tile.py 2 > $O/stages_cache_$cc.log 2>&1
  echo "rc=$?" >> $O/stages_cache_$cc.log
done
