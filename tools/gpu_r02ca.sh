#!/bin/bash
# S4 register carry (HP_RG_CARRY=1 variant): parity, A/B bench + config 2 / config 5
O=gpurun_out/${OUTN:-r02ca}; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
SO=$PWD/paper_1209_3332_b200/libhp_${VAR:-carry}.so
HP_SO=$SO timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "recon or iwpp or pipeline or hot_path or bench_tiles" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
for v in A B A B; do
  so=$PWD/paper_1209_3332_b200/libhp.so; [ $v = B ] && so=$SO
  HP_SO=$so timeout -s KILL 400 python bench.py --no-e2e --no-cpu-baseline --steps 20 > $O/b_$v.json 2> $O/b_$v.err
  HP_SO=$so timeout -s KILL 300 python tools/configs_report.py --configs 2 --out $O/c_$v.json > /dev/null 2>&1
  python -c "
import json;d=json.loads(open('$O/b_$v.json').read().strip().splitlines()[-1]);c=json.load(open('$O/c_$v.json'))['results'][0]
print('$v', round(d['value'],1), 'cfg2', round(c['ms_median'],3), 'S4', c['stage_ms_median']['S4 recon'])"
done
for v in A B; do
  so=$PWD/paper_1209_3332_b200/libhp.so; [ $v = B ] && so=$SO
  HP_SO=$so timeout -s KILL 600 python tools/configs_report.py --configs 5 --out $O/c5_$v.json > /dev/null 2>&1
  python -c "
import json;c=json.load(open('$O/c5_$v.json'))['results'][0]
print('$v cfg5', [(x['case'], round(x['ms'],1), x['recon_eq_mask']) for x in c['cases']])"
done
