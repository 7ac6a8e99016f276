#!/bin/bash
# r02i: hybrid S4 engine gated by region visits (HP_RG_THIN rows, HP_RG_CHAIN visits)
O=gpurun_out/r02i; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout -s KILL 1500 python -m pytest tests/test_gpu_variants.py -q -x -p no:cacheprovider > $O/pytest_var.log 2>&1; echo "rc=$?" >> $O/pytest_var.log
tail -2 $O/pytest_var.log
for cfg in "0 0" "4096 8" "4096 16" "4096 32" "64 8"; do
  set -- $cfg; thin=$1; chain=$2; tag=t${thin}c${chain}
  HP_RG_THIN=$thin HP_RG_CHAIN=$chain timeout -s KILL 600 python tools/configs_report.py --configs 2,5 --out $O/configs_$tag.json > $O/configs_$tag.log 2>&1
  python -c "
import json;d=json.load(open('$O/configs_$tag.json'))
for r in d['results']:
  if r['config']==2: print('$tag cfg2', r['ms_median'], r['stage_ms_median'].get('S4 recon'))
  if r['config']==5: print('$tag cfg5', [ (c['case'], round(c['ms'],1), c['recon_eq_mask']) for c in r['cases']])
"
  HP_RG_THIN=$thin HP_RG_CHAIN=$chain timeout -s KILL 300 python bench.py --no-e2e --no-cpu-baseline > $O/bench_$tag.json 2> $O/bench_$tag.err
  python -c "import json;d=json.loads(open('$O/bench_$tag.json').read().strip().splitlines()[-1]);print('$tag bench',d['value'],[ (p['stage'][:3],p['ms_isolated'],p['ms_in_situ']) for p in d['per_stage']][3])"
done
