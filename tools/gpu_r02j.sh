#!/bin/bash
# r02j: defaults now THIN=4096 / CHAIN=8; JPEG fast-AC tables; chain-gate sweep; full suite
O=gpurun_out/r02j; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout -s KILL 600 python -m pytest tests/test_gpu_jpeg.py -q -x -p no:cacheprovider > $O/pytest_jpeg.log 2>&1; echo "rc=$?" >> $O/pytest_jpeg.log; tail -2 $O/pytest_jpeg.log
timeout -s KILL 300 python tools/jpeg_probe.py 10 > $O/jpeg_probe.json 2> $O/jpeg_probe.err; cat $O/jpeg_probe.json
for chain in 3 5 8; do
  HP_RG_CHAIN=$chain timeout -s KILL 600 python tools/configs_report.py --configs 2,5 --out $O/configs_c$chain.json > $O/configs_c$chain.log 2>&1
  python -c "
import json;d=json.load(open('$O/configs_c$chain.json'))
for r in d['results']:
  if r['config']==2: print('c$chain cfg2', r['ms_median'], r['stage_ms_median'].get('S4 recon'))
  if r['config']==5: print('c$chain cfg5', [ (c['case'], round(c['ms'],1), c['recon_eq_mask']) for c in r['cases']])
"
  HP_RG_CHAIN=$chain timeout -s KILL 300 python bench.py --no-e2e --no-cpu-baseline > $O/bench_c$chain.json 2> $O/bench_c$chain.err
  python -c "import json;d=json.loads(open('$O/bench_c$chain.json').read().strip().splitlines()[-1]);print('c$chain bench',d['value'],[ (p['stage'][:3],p['ms_isolated'],p['ms_in_situ']) for p in d['per_stage']][3])"
done
timeout -s KILL 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
