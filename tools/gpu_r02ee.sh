#!/bin/bash
O=gpurun_out/r02ee; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
for cfg in "12 12 0" "16 16 0" "24 24 0" "12 12 74" "12 12 40" "12 12 0"; do
  set -- $cfg; b=$1; sl=$2; g=$3; tag=b${b}s${sl}g${g}
  if [ $g = 0 ]; then unset HP_RG_GRID; else export HP_RG_GRID=$g; fi
  timeout -s KILL 400 python bench.py --no-e2e --no-cpu-baseline --batch $b --slots $sl > $O/bench_$tag.json 2> $O/bench_$tag.err
  python -c "import json;d=json.loads(open('$O/bench_$tag.json').read().strip().splitlines()[-1]);print('$tag',d['value'])"
done
