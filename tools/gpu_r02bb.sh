#!/bin/bash
O=gpurun_out/r02bb; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
for v in "" ret48 ret28 ret816 poll ""; do
  so=$PWD/paper_1209_3332_b200/libhp${v:+_$v}.so; tag=${v:-default}
  HP_SO=$so timeout -s KILL 400 python bench.py --no-e2e --no-cpu-baseline > $O/bench_$tag.json 2> $O/bench_$tag.err
  python -c "import json;d=json.loads(open('$O/bench_$tag.json').read().strip().splitlines()[-1]);print('$tag',d['value'])"
done
