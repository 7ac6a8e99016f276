#!/bin/bash
O=gpurun_out/r02dd; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
for v in ret48 ret44 ret42 ret24 "" ret48 ret44; do
  so=$PWD/paper_1209_3332_b200/libhp${v:+_$v}.so; tag=${v:-default}
  HP_SO=$so timeout -s KILL 400 python bench.py --no-e2e --no-cpu-baseline > $O/bench_$tag.json 2> $O/bench_$tag.err
  python -c "import json;d=json.loads(open('$O/bench_$tag.json').read().strip().splitlines()[-1]);print('$tag',d['value'])"
done
for v in ret48 ret44; do
  HP_SO=$PWD/paper_1209_3332_b200/libhp_$v.so timeout -s KILL 600 python tools/configs_report.py --configs 2,5 --out $O/configs_$v.json > /dev/null 2>&1
  python -c "
import json;d=json.load(open('$O/configs_$v.json'))
for r in d['results']:
  if r['config']==2: print('$v cfg2', r['ms_median'], r['stage_ms_median'].get('S4 recon'))
  if r['config']==5: print('$v cfg5', [ (c['case'], round(c['ms'],1)) for c in r['cases']])
"
done
