#!/bin/bash
# usage: tools/gpu_check.sh TAG  -- GPU parity tests (stop at first failure) + IWPP/stage diagnostic
TAG=${1:-x}
timeout -s KILL 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
timeout -s KILL 300 python tools/diag_iwpp.py > gpurun_out/diag_$TAG.log 2>&1
echo "diag rc=$?" >> gpurun_out/diag_$TAG.log
