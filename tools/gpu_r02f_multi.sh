#!/bin/bash
# r02f: BASELINE configs[3] (config 4) at full size, 36,848 tiles demand-driven over 1 / 2 / 4
# GPUs, raw RGB and JPEG ingest, rows in device arenas, device-to-device gather to rank 0;
# then bench.py at 2 and 4 GPUs.
O=${OUT:-gpurun_out/r02f}; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
nvidia-smi -L > $O/gpus.txt
port=29600
for mode in raw jpeg; do
  for n in 1 2 4; do
    port=$((port+1))
    extra=""; [ $mode = jpeg ] && extra="--jpeg"
    timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port \
      tools/run_dataset.py --config 4 $extra --out $O/config4_${mode}_${n}gpu.json > $O/config4_${mode}_${n}gpu.log 2>&1
    echo "$mode $n rc=$?"; tail -c 400 $O/config4_${mode}_${n}gpu.json 2>/dev/null; echo
  done
done
for n in 2 4; do
  port=$((port+1))
  timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port \
    bench.py --gpus $n > $O/bench_${n}gpu.json 2> $O/bench_${n}gpu.err
  echo "bench $n rc=$?"; tail -c 300 $O/bench_${n}gpu.json
done
