#!/bin/bash
O=gpurun_out/r02l; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
for bs in "12 12" "12 16" "16 16" "24 24" "12 8" "24 16"; do
  set -- $bs; b=$1; sl=$2
  timeout -s KILL 400 python bench.py --no-e2e --no-cpu-baseline --batch $b --slots $sl > $O/bench_b${b}s${sl}.json 2> $O/bench_b${b}s${sl}.err
  python -c "import json;d=json.loads(open('$O/bench_b${b}s${sl}.json').read().strip().splitlines()[-1]);print('b$b s$sl',d['value'],d['ms_per_step'])"
done
