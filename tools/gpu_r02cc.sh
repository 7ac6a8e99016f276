#!/bin/bash
O=gpurun_out/r02cc; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
for es in 14 18 24 10; do
  timeout -s KILL 400 python bench.py --no-cpu-baseline --e2e-slots $es > $O/bench_e$es.json 2> $O/bench_e$es.err
  python -c "import json;d=json.loads(open('$O/bench_e$es.json').read().strip().splitlines()[-1]);print('e2e slots $es',d['value'],d['e2e']['value'],d['e2e']['jpeg']['value'])"
done
