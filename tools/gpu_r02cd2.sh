O=gpurun_out/r02cdbg; mkdir -p $O
HP_SO=$PWD/paper_1209_3332_b200/libhp_compdbg.so timeout -s KILL 300 python tools/one_tile.py 3 > $O/out.log 2>&1
grep COMPSUM $O/out.log
python - $O/out.log <<'PY'
import sys,re
for l in open(sys.argv[1]):
    if l.startswith('COMPSUM'):
        d={k:int(v) for k,v in re.findall(r'(\S+)=(\d+)', l)}
        print({k: round(v/d['total'],3) for k,v in d.items() if k not in ('n','total')}, 'avg cycles/comp', d['total']//d['n'])
PY
