#!/bin/bash
# A/B of two library builds: config-2 stage table and the bench, alternating
# usage: tools/gpu_ab.sh OUTDIR A.so B.so
O=gpurun_out/$1; mkdir -p $O; A=$PWD/$2; B=$PWD/$3
export CUDA_DEVICE_MAX_CONNECTIONS=32
for v in A B A B; do
  so=$A; [ $v = B ] && so=$B
  HP_SO=$so timeout -s KILL 300 python tools/configs_report.py --configs 2 --out $O/cfg_$v.json > $O/cfg_$v.log 2>&1
  python -c "import json;d=json.load(open('$O/cfg_$v.json'));r=d['results'][0];print('$v cfg2',r['ms_median'],r['stage_ms_median'])"
  HP_SO=$so timeout -s KILL 400 python bench.py --no-e2e --no-cpu-baseline --steps 20 > $O/bench_$v.json 2> $O/bench_$v.err
  python -c "import json;d=json.loads(open('$O/bench_$v.json').read().strip().splitlines()[-1]);print('$v bench',d['value'],d['ms_per_step'])"
done
