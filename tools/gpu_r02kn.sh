#!/bin/bash
# S4 knob re-sweep at the final build: bench (20 steps) and the JPEG probe's decoded-tile S4
O=gpurun_out/r02kn; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
for e in "HP_X=0" "HP_RG_CHAIN=6" "HP_RG_CHAIN=12" "HP_RG_THIN=1024" "HP_RG_THIN=16384" "HP_RG_CHAIN=16" "HP_X=0"; do
  n=$(echo $e | tr '=' '_')
  env $e timeout -s KILL 400 python bench.py --no-e2e --no-cpu-baseline --steps 20 > $O/b_$n.json 2> $O/b_$n.err
  env $e timeout -s KILL 300 python tools/jpeg_probe.py 5 > $O/p_$n.json 2>/dev/null
  python -c "
import json;d=json.loads(open('$O/b_$n.json').read().strip().splitlines()[-1]);p=json.load(open('$O/p_$n.json'))
print('$e', round(d['value'],1), 'S4 raw/decoded', p['stages_raw_ms']['S4'], p['stages_decoded_ms']['S4'])"
done
