#!/bin/bash
O=gpurun_out/r02z; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout -s KILL 1200 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "variant or iwpp or recon or pipeline or hot_path or components" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
timeout -s KILL 600 python tools/configs_report.py --configs 2,5 --out $O/configs.json > $O/configs.log 2>&1
python -c "
import json;d=json.load(open('$O/configs.json'))
for r in d['results']:
  if r['config']==2: print('cfg2', r['ms_median'], r['stage_ms_median'].get('S4 recon'))
  if r['config']==5: print('cfg5', [ (c['case'], round(c['ms'],1), c['jobs'], c['recon_eq_mask']) for c in r['cases']])
"
for i in 1 2; do
  timeout -s KILL 400 python bench.py --no-e2e --no-cpu-baseline > $O/bench_$i.json 2> $O/bench_$i.err
  python -c "import json;d=json.loads(open('$O/bench_$i.json').read().strip().splitlines()[-1]);print('bench',d['value'],[ (p['stage'][:3],p['ms_isolated']) for p in d['per_stage']][3])"
done
timeout -s KILL 600 python tools/stress_determinism.py 20 12 jpeg > $O/stress.log 2>&1; tail -1 $O/stress.log
