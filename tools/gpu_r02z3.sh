#!/bin/bash
# parity + bench + ncu of the CCL-select kernels and Canny (OUT dir from $1)
O=gpurun_out/${1:-r02z3}; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
for i in 1 2; do
  timeout -s KILL 400 python bench.py --no-e2e --no-cpu-baseline --steps 20 > $O/bench_$i.json 2> $O/bench_$i.err
  python -c "import json;d=json.loads(open('$O/bench_$i.json').read().strip().splitlines()[-1]);print('bench',d['value'],d['ms_per_step'])"
done
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k 'regex:k_canny_nms|k_cs_' -s 18 -c 18 -o $O/ncu_canny python tools/one_tile.py 2 > $O/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $O/ncu_canny.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum > $O/raw.csv 2>&1; tail -1 $O/raw.csv
