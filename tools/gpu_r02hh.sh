#!/bin/bash
O=gpurun_out/r02hh; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
for v in "" w2 w8 cbps3 fbps2 poll800 "" w2 cbps3; do
  so=$PWD/paper_1209_3332_b200/libhp${v:+_$v}.so; tag=${v:-default}
  HP_SO=$so timeout -s KILL 400 python bench.py --no-e2e --no-cpu-baseline > $O/bench_$tag.json 2> $O/bench_$tag.err
  python -c "import json;d=json.loads(open('$O/bench_$tag.json').read().strip().splitlines()[-1]);print('$tag',d['value'])"
done
