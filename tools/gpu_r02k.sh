#!/bin/bash
O=gpurun_out/r02k; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
for sch in rotate join fixed rotate; do
  timeout -s KILL 300 python bench.py --no-e2e --no-cpu-baseline --schedule $sch > $O/bench_$sch.json 2> $O/bench_$sch.err
  python -c "import json;d=json.loads(open('$O/bench_$sch.json').read().strip().splitlines()[-1]);print('$sch',d['value'],d['ms_per_step'])"
done
timeout -s KILL 300 python tools/jpeg_probe.py 10 > $O/jpeg_probe.json 2> $O/jpeg_probe.err; cat $O/jpeg_probe.json
