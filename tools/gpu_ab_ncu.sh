#!/bin/bash
# A/B of two library builds by kernel duration: ncu launch lists of tools/one_tile.py 3 (config-2 tile)
# usage: tools/gpu_ab_ncu.sh OUTDIR A.so B.so
O=gpurun_out/$1; mkdir -p $O; A=$PWD/$2; B=$PWD/$3
export CUDA_DEVICE_MAX_CONNECTIONS=32
for v in A B; do
  so=$A; [ $v = B ] && so=$B
  HP_SO=$so timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$v.csv python tools/one_tile.py 3 > $O/ncu_$v.log 2>&1
done
python - $O <<'PY'
import csv, sys, collections
O = sys.argv[1]
res = {}
for v in "AB":
    rows = [r for r in csv.reader(open(f"{O}/launches_{v}.csv")) if len(r) > 10 and r[0] != "ID"]
    hdr = next(r for r in csv.reader(open(f"{O}/launches_{v}.csv")) if r and r[0] == "ID")
    K, M, V = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    d = collections.defaultdict(float)
    for r in rows:
        if r[M] == "gpu__time_duration.sum":
            d[r[K].split("(")[0][:40]] += float(r[V].replace(",", "")) / 3
    res[v] = d
names = sorted(set(res["A"]) | set(res["B"]), key=lambda n: -res["A"].get(n, 0))
for n in names:
    a, b = res["A"].get(n, 0), res["B"].get(n, 0)
    if a > 2000 or b > 2000:
        print(f"{n:40s} {a/1000:8.1f} {b/1000:8.1f} us/tile")
print("total", sum(res["A"].values()) / 1000, sum(res["B"].values()) / 1000)
PY
