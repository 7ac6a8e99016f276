#!/bin/bash
# blocks-per-SM re-sweep of the component / fill kernels at the current build (bench, alternating)
O=gpurun_out/${OUTN:-r02bps}; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
for v in ${VARS:-default cb2 cb3 fb4 default cb2 cb3 fb4}; do
  so=$PWD/paper_1209_3332_b200/libhp_$v.so; [ $v = default ] && so=$PWD/paper_1209_3332_b200/libhp.so
  HP_SO=$so timeout -s KILL 400 python bench.py --no-e2e --no-cpu-baseline --steps 20 > $O/b_$v.json 2> $O/b_$v.err
  python -c "import json;d=json.loads(open('$O/b_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['value'],1))"
done
