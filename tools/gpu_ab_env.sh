#!/bin/bash
# A/B of one build under two environment settings: ncu launch lists of tools/one_tile.py 3 and
# the bench, alternating.  usage: tools/gpu_ab_env.sh OUTDIR "ENV_A" "ENV_B"
O=gpurun_out/$1; mkdir -p $O; EA=$2; EB=$3
export CUDA_DEVICE_MAX_CONNECTIONS=32
for v in A B; do
  e=$EA; [ $v = B ] && e=$EB
  env $e timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$v.csv python tools/one_tile.py 3 > $O/ncu_$v.log 2>&1
done
python - $O <<'PY'
import csv, sys, collections
O = sys.argv[1]
res = {}
for v in "AB":
    rows = list(csv.reader(open(f"{O}/launches_{v}.csv")))
    hdr = next(r for r in rows if r and r[0] == "ID")
    K, M, V = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    d = collections.defaultdict(float)
    for r in rows:
        if len(r) == len(hdr) and r[0] != "ID" and r[M] == "gpu__time_duration.sum":
            d[r[K].split("(")[0][:40]] += float(r[V].replace(",", "")) / 3
    res[v] = d
for n in sorted(set(res["A"]) | set(res["B"]), key=lambda n: -res["A"].get(n, 0)):
    a, b = res["A"].get(n, 0), res["B"].get(n, 0)
    if a > 2000 or b > 2000:
        print(f"{n:40s} {a/1000:8.1f} {b/1000:8.1f} us/tile")
print("total", sum(res["A"].values()) / 1000, sum(res["B"].values()) / 1000)
PY
for v in A B A B; do
  e=$EA; [ $v = B ] && e=$EB
  env $e timeout -s KILL 400 python bench.py --no-e2e --no-cpu-baseline --steps 20 > $O/bench_$v.json 2> $O/bench_$v.err
  python -c "import json;d=json.loads(open('$O/bench_$v.json').read().strip().splitlines()[-1]);print('$v bench',d['value'])"
done
