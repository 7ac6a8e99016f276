#!/bin/bash
# ncu --set full of the per-component kernels (S6 fill, S7-S11 fused) on a config-2 tile
O=gpurun_out/r02ff; mkdir -p $O
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k 'regex:k_fill_fused|k_comp_fused' -s 2 -c 2 -o $O/ncu_comp python tools/one_tile.py 2 > $O/ncu.log 2>&1; echo "rc=$?"
ncu -i $O/ncu_comp.ncu-rep --page details --csv > $O/details.csv 2>&1
ncu -i $O/ncu_comp.ncu-rep -k regex:k_fill_fused --page source --csv --print-source sass > $O/fill_sass.csv 2>&1
ncu -i $O/ncu_comp.ncu-rep -k regex:k_comp_fused --page source --csv --print-source sass > $O/comp_sass.csv 2>&1
ncu -i $O/ncu_comp.ncu-rep -k regex:k_fill_fused --page source --csv --print-source cuda > $O/fill_cuda.csv 2>&1
ncu -i $O/ncu_comp.ncu-rep -k regex:k_comp_fused --page source --csv --print-source cuda > $O/comp_cuda.csv 2>&1
