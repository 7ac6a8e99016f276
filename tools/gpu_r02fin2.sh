#!/bin/bash
export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/${FINAL_OUT:-final2}; mkdir -p $O
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
OUT=$O bash tools/gpu_final_1gpu.sh
