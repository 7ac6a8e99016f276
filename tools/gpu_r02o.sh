#!/bin/bash
# r02o: launch-shape variants of the persistent component / morphology kernels (variant builds)
O=gpurun_out/r02o; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
for v in "" cbps2 cbps6 mbps2 minb3 ""; do
  so=paper_1209_3332_b200/libhp${v:+_$v}.so; tag=${v:-default}
  HP_SO=$PWD/$so timeout -s KILL 400 python bench.py --no-e2e --no-cpu-baseline > $O/bench_$tag.json 2> $O/bench_$tag.err
  python -c "import json;d=json.loads(open('$O/bench_$tag.json').read().strip().splitlines()[-1]);print('$tag',d['value'],[ (p['stage'][:3],p['ms_isolated']) for p in d['per_stage']])"
done
