#!/bin/bash
# r02e: JPEG decoder v2 (int32 IDCT fast path, 8-byte refill, 256-thread blocks) and the S4
# raster/anti-raster initialisation experiment (HP_RG_INIT)
O=gpurun_out/r02e; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout -s KILL 600 python -m pytest tests/test_gpu_jpeg.py tests/test_gpu_variants.py -q -x -p no:cacheprovider > $O/pytest_new.log 2>&1; echo "rc=$?" >> $O/pytest_new.log
tail -3 $O/pytest_new.log
timeout -s KILL 300 python tools/jpeg_probe.py 10 > $O/jpeg_probe.json 2> $O/jpeg_probe.err; cat $O/jpeg_probe.json
for init in 0 1; do
  HP_RG_INIT=$init timeout -s KILL 600 python tools/configs_report.py --configs 2,5 --out $O/configs_init$init.json > $O/configs_init$init.log 2>&1
  HP_RG_INIT=$init timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline > $O/bench_init$init.json 2> $O/bench_init$init.err
  python -c "import json;d=json.loads(open('$O/bench_init$init.json').read().strip().splitlines()[-1]);print('init',$init,d['value'],[ (p['stage'][:3],p['ms_isolated'],p['ms_in_situ']) for p in d['per_stage']])"
  grep -o '"case": "[a-z ]*", "path_px": [0-9]*, "ms": [0-9.]*' $O/configs_init$init.json
done
HP_RG_INIT=1 timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --kernel-name regex:^k_ --log-file $O/launches_init1.csv python tools/one_tile.py 2 > /dev/null 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --kernel-name regex:^k_ --log-file $O/jpeg_launches.csv python tools/jpeg_probe.py 1 > /dev/null 2>&1
