#!/bin/bash
# idle back-off variants of the S4 engine: bench (alternating) and config-2 S4 alone
O=gpurun_out/${OUTN:-r02po}; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
for v in ${VARS:-default p1 p2 default p1 p2}; do
  so=$PWD/paper_1209_3332_b200/libhp_$v.so; [ $v = default ] && so=$PWD/paper_1209_3332_b200/libhp.so
  HP_SO=$so timeout -s KILL 400 python bench.py --no-e2e --no-cpu-baseline --steps 20 > $O/b_$v.json 2> $O/b_$v.err
  HP_SO=$so timeout -s KILL 300 python tools/configs_report.py --configs 2 --out $O/c_$v.json > /dev/null 2>&1
  python -c "
import json;d=json.loads(open('$O/b_$v.json').read().strip().splitlines()[-1]);c=json.load(open('$O/c_$v.json'))['results'][0]
print('$v', round(d['value'],1), 'cfg2', round(c['ms_median'],3), 'S4', c['stage_ms_median']['S4 recon'])"
done
