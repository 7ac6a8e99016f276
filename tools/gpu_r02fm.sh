set -e
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
HP_CS_FUSED=0 timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "rbc or area or fill or canny or pipeline_config1 or hot_path" 2>&1 | tail -1
bash tools/gpu_ab_env.sh r02fm "HP_CS_FUSED=0" "HP_CS_FUSED=1"
