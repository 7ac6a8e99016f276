#!/bin/bash
O=gpurun_out/r02mo; mkdir -p $O
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k 'regex:k_morph_r' -s 2 -c 1 -o $O/ncu_morph python tools/one_tile.py 2 > $O/ncu.log 2>&1; echo "rc=$?"
ncu -i $O/ncu_morph.ncu-rep --page details --csv > $O/details.csv 2>&1
ncu -i $O/ncu_morph.ncu-rep --page source --csv --print-source cuda,sass > $O/mix.csv 2>&1
