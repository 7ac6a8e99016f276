#!/bin/bash
# r02c: JPEG ingest tests first (new code), then the full GPU suite, the JPEG probe and a
# launch list of the probe
O=gpurun_out/r02c; mkdir -p $O
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout -s KILL 600 python -m pytest tests/test_gpu_jpeg.py -q -x -p no:cacheprovider > $O/pytest_jpeg.log 2>&1; echo "rc=$?" >> $O/pytest_jpeg.log
tail -3 $O/pytest_jpeg.log
timeout -s KILL 300 python tools/jpeg_probe.py 10 > $O/jpeg_probe.json 2> $O/jpeg_probe.err; echo "rc=$?" >> $O/jpeg_probe.err
cat $O/jpeg_probe.json
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --kernel-name regex:^k_ --log-file $O/jpeg_launches.csv python tools/jpeg_probe.py 1 > $O/jpeg_ncu.log 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
