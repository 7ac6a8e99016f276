#!/bin/bash
O=gpurun_out/r02d; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout -s KILL 600 python -m pytest tests/test_gpu_jpeg.py -q -x -p no:cacheprovider > $O/pytest_jpeg.log 2>&1; echo "rc=$?" >> $O/pytest_jpeg.log
tail -2 $O/pytest_jpeg.log
timeout -s KILL 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
tail -c 1500 $O/bench.json
timeout -s KILL 900 python tools/run_dataset.py --config 4 --tiles 2000 --out $O/ds4_2000_raw.json > $O/ds4_raw.log 2>&1; echo "rc=$?" >> $O/ds4_raw.log
tail -2 $O/ds4_raw.log
timeout -s KILL 900 python tools/run_dataset.py --config 4 --tiles 2000 --jpeg --out $O/ds4_2000_jpeg.json > $O/ds4_jpeg.log 2>&1; echo "rc=$?" >> $O/ds4_jpeg.log
tail -2 $O/ds4_jpeg.log
timeout -s KILL 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
