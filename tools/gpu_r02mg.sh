#!/bin/bash
# bench.py at 2 and 4 GPUs (device-resident + e2e legs) at the final build, plus 1 GPU on the same box
O=${OUT:-gpurun_out/r02mg}; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
nvidia-smi -L > $O/gpus.txt
timeout -s KILL 600 python bench.py > $O/bench_1gpu.json 2> $O/bench_1gpu.err; echo "bench 1 rc=$?"
port=29700
for n in 2 4; do
  port=$((port+1))
  timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port \
    bench.py --gpus $n > $O/bench_${n}gpu.json 2> $O/bench_${n}gpu.err
  echo "bench $n rc=$?"
done
for n in 1 2 4; do python -c "
import json;d=json.loads(open('$O/bench_${n}gpu.json').read().strip().splitlines()[-1])
print($n, round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'jpeg', round(d['e2e'].get('jpeg',{}).get('value',0),1))"; done
