#!/bin/bash
# r02g: the ADI region engine (HP_RG_ADI=1) -- parity under both settings, config 2 / 5 times,
# bench value; ncu --set full of the JPEG decode kernel and of k_region_adi
O=gpurun_out/r02g; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout -s KILL 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_jpeg.py -q -x -p no:cacheprovider > $O/pytest_new.log 2>&1; echo "rc=$?" >> $O/pytest_new.log
tail -3 $O/pytest_new.log
for adi in 1 0; do
  HP_RG_ADI=$adi timeout -s KILL 600 python tools/configs_report.py --configs 2,5 --out $O/configs_adi$adi.json > $O/configs_adi$adi.log 2>&1
  python -c "
import json;d=json.load(open('$O/configs_adi$adi.json'))
for r in d['results']:
  if r['config']==2: print('adi $adi cfg2', r['ms_median'], r['stage_ms_median'].get('S4 recon'))
  if r['config']==5:
    for c in r['cases']: print('adi $adi', c['case'], round(c['ms'],1), c['jobs'], c['recon_eq_mask'])
"
  HP_RG_ADI=$adi timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline > $O/bench_adi$adi.json 2> $O/bench_adi$adi.err
  python -c "import json;d=json.loads(open('$O/bench_adi$adi.json').read().strip().splitlines()[-1]);print('adi',$adi,d['value'],[ (p['stage'][:3],p['ms_isolated'],p['ms_in_situ']) for p in d['per_stage']])"
done
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:k_jpeg_decode -c 1 -o $O/ncu_jpeg_decode python tools/jpeg_probe.py 1 > $O/ncu_jpeg.log 2>&1
HP_RG_ADI=1 timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:k_region_adi -c 1 -o $O/ncu_region_adi python tools/one_tile.py 1 > $O/ncu_adi.log 2>&1
ls -la $O
