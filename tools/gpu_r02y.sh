#!/bin/bash
# Marginal-cost decomposition of the bench step (variant builds run one step twice per tile).
O=gpurun_out/${OUTN:-r02y}; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
for v in default dup1 dup2 dup3 dup5 dup6 dup8 dup9 s4x2 default; do
  so=$PWD/paper_1209_3332_b200/libhp_$v.so; [ $v = default ] && so=$PWD/paper_1209_3332_b200/libhp.so
  HP_SO=$so timeout -s KILL 400 python bench.py --no-e2e --no-cpu-baseline --steps 20 > $O/bench_$v.json 2> $O/bench_$v.err
  python -c "import json;d=json.loads(open('$O/bench_$v.json').read().strip().splitlines()[-1]);print('$v',d['value'],d['ms_per_step'])"
done
