#!/bin/bash
O=gpurun_out/r02x; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
SO=$PWD/paper_1209_3332_b200/libhp_firstrow.so
HP_SO=$SO timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "iwpp or recon or pipeline_config1 or pipeline_random_small or pipeline_islands or hot_path_stages" > $O/pytest_var.log 2>&1; echo "rc=$?" >> $O/pytest_var.log; tail -2 $O/pytest_var.log
for v in firstrow default firstrow default; do
  so=$PWD/paper_1209_3332_b200/libhp.so; [ $v = firstrow ] && so=$SO
  HP_SO=$so timeout -s KILL 400 python bench.py --no-e2e --no-cpu-baseline > $O/bench_$v.json 2> $O/bench_$v.err
  python -c "import json;d=json.loads(open('$O/bench_$v.json').read().strip().splitlines()[-1]);print('$v',d['value'],[ (p['stage'][:3],p['ms_isolated']) for p in d['per_stage']][3])"
done
HP_SO=$SO timeout -s KILL 600 python tools/configs_report.py --configs 2,5 --out $O/configs.json > $O/configs.log 2>&1
python -c "
import json;d=json.load(open('$O/configs.json'))
for r in d['results']:
  if r['config']==2: print('cfg2', r['ms_median'], r['stage_ms_median'].get('S4 recon'))
  if r['config']==5: print('cfg5', [ (c['case'], round(c['ms'],1), c['recon_eq_mask']) for c in r['cases']])
"
