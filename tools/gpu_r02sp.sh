set -e
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
bash tools/gpu_ab_ncu.sh r02sp paper_1209_3332_b200/libhp_old.so paper_1209_3332_b200/libhp.so
timeout -s KILL 600 ncu --section LaunchStats --section Occupancy -k regex:k_comp_fused -s 1 -c 1 python tools/one_tile.py 2 2>&1 | grep -i "Block Limit Shared\|Theoretical Occ\|Dynamic Shared" | head
bash tools/gpu_ab.sh r02spb paper_1209_3332_b200/libhp_old.so paper_1209_3332_b200/libhp.so
