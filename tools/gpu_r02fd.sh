O=gpurun_out/r02fd; mkdir -p $O
HP_SO=$PWD/paper_1209_3332_b200/libhp_filldbg.so timeout -s KILL 300 python tools/one_tile.py 1 > $O/out.log 2>&1
grep -c FILLDBG $O/out.log; grep HOLESDBG $O/out.log | sort -t= -k3 -n -r | head -25
