#!/bin/bash
# Final one-GPU measurements of a round: the default bench line, its ncu launch list (the
# contract's gpu__time_duration pass), one ncu --set full capture of the dominant kernel
# (k_region_mr8) inside the bench, the per-config report (configs 1, 2, 3, 5) and smoke().
O=${OUT:-gpurun_out/final}; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout -s KILL 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -c 400 $O/bench.json
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_launches.log 2>&1; echo "launches rc=$?"
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_region_mr8 -s 20 -c 1 -o $O/ncu_region_full \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_full.log 2>&1; echo "full rc=$?"
timeout -s KILL 900 python tools/configs_report.py --configs 1,2,5,3 --out $O/configs_report.json > $O/configs.log 2>&1; echo "configs rc=$?"
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
