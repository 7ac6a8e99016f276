set -e
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -q -x -p no:cacheprovider 2>&1 | tail -2
bash tools/gpu_ab_ncu.sh ${OUTN:-r02cw} paper_1209_3332_b200/libhp_old.so paper_1209_3332_b200/libhp.so
bash tools/gpu_ab.sh ${OUTN:-r02cw}b paper_1209_3332_b200/libhp_old.so paper_1209_3332_b200/libhp.so
