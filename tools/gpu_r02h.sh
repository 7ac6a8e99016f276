#!/bin/bash
# r02h: hybrid S4 engine (HP_RG_THIN: thin jobs by alternating phases), ADI race fix
O=gpurun_out/r02h; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout -s KILL 1200 python -m pytest tests/test_gpu_variants.py -q -x -p no:cacheprovider > $O/pytest_var.log 2>&1; echo "rc=$?" >> $O/pytest_var.log
tail -3 $O/pytest_var.log
for thin in 0 4 16 64; do
  HP_RG_THIN=$thin timeout -s KILL 600 python tools/configs_report.py --configs 2,5 --out $O/configs_thin$thin.json > $O/configs_thin$thin.log 2>&1
  python -c "
import json;d=json.load(open('$O/configs_thin$thin.json'))
for r in d['results']:
  if r['config']==2: print('thin $thin cfg2', r['ms_median'], r['stage_ms_median'].get('S4 recon'))
  if r['config']==5: print('thin $thin cfg5', [ (c['case'], round(c['ms'],1), c['recon_eq_mask']) for c in r['cases']])
"
  HP_RG_THIN=$thin timeout -s KILL 300 python bench.py --no-e2e --no-cpu-baseline > $O/bench_thin$thin.json 2> $O/bench_thin$thin.err
  python -c "import json;d=json.loads(open('$O/bench_thin$thin.json').read().strip().splitlines()[-1]);print('thin',$thin,d['value'],[ (p['stage'][:3],p['ms_isolated'],p['ms_in_situ']) for p in d['per_stage']][3])"
done
HP_RG_ADI=1 timeout -s KILL 300 python bench.py --no-e2e --no-cpu-baseline > $O/bench_adi1.json 2> $O/bench_adi1.err
python -c "import json;d=json.loads(open('$O/bench_adi1.json').read().strip().splitlines()[-1]);print('adi1',d['value'])"
