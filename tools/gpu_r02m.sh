#!/bin/bash
O=gpurun_out/r02m; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
for g in ${GRIDS:-111 148 74 222}; do
  HP_RG_GRID=$g timeout -s KILL 400 python bench.py --no-e2e --no-cpu-baseline > $O/bench_grid$g.json 2> $O/bench_grid$g.err
  python -c "import json;d=json.loads(open('$O/bench_grid$g.json').read().strip().splitlines()[-1]);print('grid $g',d['value'])"
done
for bps in 3 4; do :; done
timeout -s KILL 300 python tools/jpeg_probe.py 10 > $O/jpeg_probe.json 2> $O/jpeg_probe.err; cat $O/jpeg_probe.json
