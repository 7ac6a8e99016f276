"""Summarise ncu outputs into profiles/: a per-kernel share table from a launch list
(--metrics gpu__time_duration.sum --csv) and key metrics of a --set full report.

usage: python tools/profile_summary.py launches <launches.csv> <out.md>
       python tools/profile_summary.py full <report.ncu-rep> <out.json> [stage_index]
"""
import collections
import csv
import io
import json
import subprocess
import sys


def launches(src, out):
    rows = list(csv.reader(open(src)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(d["Metric Unit"], 1e-6)
        k = d["Kernel Name"].split("(")[0].replace("hp::<unnamed>::", "").replace("void ", "")
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    lines = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k[:80]}` | {n} | {t:.3f} | {100 * t / tot:.1f}% |")
    lines.append(f"| **total** | {sum(v[0] for v in agg.values())} | {tot:.3f} | 100% |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:12]))


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def full(rep, out, stage=None):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = {"value": vals[i], "unit": units[i]}
        res.append(d)
    doc = {"report": rep, "kernels": res}
    if stage is not None and res:
        def num(x):
            return float(x["value"].replace(",", ""))
        mb = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}
        r0 = res[0]
        tr = num(r0["dram__bytes_read.sum"]) * mb.get(r0["dram__bytes_read.sum"]["unit"], 1.0) + \
            num(r0["dram__bytes_write.sum"]) * mb.get(r0["dram__bytes_write.sum"]["unit"], 1.0)
        doc["per_stage_bytes"] = {str(stage): int(tr)}
    json.dump(doc, open(out, "w"), indent=1)
    print(json.dumps(doc, indent=1)[:2000])


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else None)
