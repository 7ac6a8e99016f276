#!/bin/bash
# re-sweep of the S4 grid and the bench slot count on the current build (bench 20 steps each)
O=gpurun_out/r02sw; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
run() {  # name, env..., -- bench args
  local name=$1; shift
  env "$@" timeout -s KILL 400 python bench.py --no-e2e --no-cpu-baseline --steps 20 $BARGS > $O/b_$name.json 2> $O/b_$name.err
  python -c "import json;d=json.loads(open('$O/b_$name.json').read().strip().splitlines()[-1]);print('$name',d['value'])"
}
BARGS="" run default HP_X=0
BARGS="" run grid40 HP_RG_GRID=40
BARGS="" run grid74 HP_RG_GRID=74
BARGS="" run grid96 HP_RG_GRID=96
BARGS="--slots 16" run slots16 HP_X=0
BARGS="--slots 16" run slots16_g40 HP_RG_GRID=40
BARGS="--batch 24 --slots 24" run b24s24 HP_X=0
BARGS="" run default2 HP_X=0
