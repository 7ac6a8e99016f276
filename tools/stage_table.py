"""Per-stage table of one config-2 tile from two ncu metric captures of tools/one_tile.py
(--cache-control all = cold caches before every kernel, none = warm), SURVEY §8(d)
"per-stage reporting": time, DRAM bytes cold and warm, L2 hit rate, atomic / reduction L2
sectors, warps active and issue active, and the stage's algorithmic floor bytes.

Kernels are assigned to steps by their launch order within one hp_process_tile (the
CCL-select kernels k_cs_* serve S2, S5 and the Canny hysteresis, so their step is the one
whose kernel preceded them).  The second tile of the capture is used (the first includes
one-time setup).

usage: python tools/stage_table.py <cold.csv> <warm.csv> <out_prefix>
"""
import collections
import csv
import json
import sys

NPX = 4096 * 4096
# SURVEY §8(d) floor bytes per pixel (read each stage input once, write each output once);
# S7-S11 run fused, so their floor is the sum of the five rows (34 B/px)
FLOOR_BPP = {"S1": 5, "S2": 2, "S3": 2, "S4": 4, "S5": 2, "S6": 2, "Canny": 2, "S7-S11": 34}
ORDER = ["S1", "S2", "S3", "S4", "S5", "S6", "Canny", "S7-S11"]


def read(fn):
    rows = [r for r in csv.reader(open(fn)) if len(r) > 10]
    hdr = rows[0]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
    ks = collections.OrderedDict()
    for r in rows[1:]:
        if r[ix["ID"]] == "ID":
            continue
        kid = int(r[ix["ID"]])
        name = r[ix["Kernel Name"]].split("(")[0].split("<")[0].split("::")[-1]
        d = ks.setdefault(kid, {"name": name})
        v = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        v *= {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e3, "msecond": 1e6}.get(unit, 1.0)
        d[r[ix["Metric Name"]]] = v
    return list(ks.values())


def assign(kernels):
    """Split the launch list into tiles (each starts with k_cd_vec16) and steps."""
    tiles, cur, step = [], None, None
    for k in kernels:
        n = k["name"]
        if n == "k_cd_vec16":
            cur = []
            tiles.append(cur)
            step = "S1"
        elif n.startswith("k_cs_"):
            step = {"S1": "S2", "S4": "S5", "Canny": "Canny"}.get(step, step)
        elif n == "k_morph_r":
            step = "S3"
        elif n.startswith("k_rg_") or n.startswith("k_region"):
            step = "S4"
        elif n in ("k_win_classify", "k_fill_fused", "k_fill_huge"):
            step = "S6"
        elif n == "k_canny_nms":
            step = "Canny"
        elif n.startswith("k_comp") or n in ("k_rows_scatter", "k_copy_i32"):
            step = "S7-S11"
        if cur is not None:
            cur.append((step, k))
    return tiles


def per_step(tile):
    agg = collections.OrderedDict((s, collections.Counter()) for s in ORDER)
    names = collections.defaultdict(list)
    for step, k in tile:
        a = agg[step]
        t = k.get("gpu__time_duration.sum", 0.0)
        a["ns"] += t
        a["dram"] += k.get("dram__bytes_read.sum", 0.0) + k.get("dram__bytes_write.sum", 0.0)
        a["atom"] += k.get("lts__t_sectors_op_atom.sum", 0.0)
        a["red"] += k.get("lts__t_sectors_op_red.sum", 0.0)
        a["l2hit_t"] += t * k.get("lts__t_sector_hit_rate.pct", 0.0)
        a["warps_t"] += t * k.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0.0)
        a["issue_t"] += t * k.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0.0)
        a["launches"] += 1
        names[step].append(k["name"])
    return agg, names


def main():
    cold, warm, out = sys.argv[1], sys.argv[2], sys.argv[3]
    peak = 6543.7
    try:
        peak = float(json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"])
    except Exception:  # noqa: BLE001
        pass
    tc = assign(read(cold))[-1]
    tw = assign(read(warm))[-1]
    ac, names = per_step(tc)
    aw, _ = per_step(tw)
    rows = []
    for s in ORDER:
        c, w = ac[s], aw[s]
        if not w["launches"]:
            continue
        ns = w["ns"]
        floor = FLOOR_BPP[s] * NPX
        rows.append({
            "step": s, "kernels": sorted(set(names[s])), "launches": int(w["launches"]),
            "ms_warm": ns / 1e6, "ms_cold": c["ns"] / 1e6,
            "dram_MB_cold": c["dram"] / 1e6, "dram_MB_warm": w["dram"] / 1e6,
            "floor_MB": floor / 1e6, "floor_GBps_warm": floor / ns if ns else None,
            "floor_frac_of_peak": (floor / ns) / peak if ns else None,
            "dram_GBps_cold": c["dram"] / c["ns"] if c["ns"] else None,
            "l2_hit_pct_warm": w["l2hit_t"] / ns if ns else None,
            "atom_sectors": w["atom"], "red_sectors": w["red"],
            "warps_active_pct": w["warps_t"] / ns if ns else None,
            "issue_active_pct": w["issue_t"] / ns if ns else None})
    doc = {"source": [cold, warm], "tile": "configs[1] 4096x4096 synthetic H&E (seed 2), hp_process_tile alone",
           "peak_GBps": peak, "note": "ncu serialises kernels; times are per kernel alone (warm: caches as the "
           "previous kernel left them; cold: flushed before each kernel)", "steps": rows}
    json.dump(doc, open(out + ".json", "w"), indent=1)
    lines = ["| step | launches | ms (warm) | ms (cold) | DRAM MB cold / warm | floor MB | floor GB/s (frac) "
             "| L2 hit % | atomic / red sectors | warps active % | issue active % |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        lines.append(f"| {r['step']} | {r['launches']} | {r['ms_warm']:.3f} | {r['ms_cold']:.3f} | "
                     f"{r['dram_MB_cold']:.1f} / {r['dram_MB_warm']:.1f} | {r['floor_MB']:.0f} | "
                     f"{r['floor_GBps_warm']:.0f} ({r['floor_frac_of_peak']:.3f}) | {r['l2_hit_pct_warm']:.1f} | "
                     f"{r['atom_sectors']:.3g} / {r['red_sectors']:.3g} | {r['warps_active_pct']:.1f} | "
                     f"{r['issue_active_pct']:.1f} |")
    tot_w = sum(r["ms_warm"] for r in rows)
    lines.append(f"| **total** | {sum(r['launches'] for r in rows)} | {tot_w:.3f} | "
                 f"{sum(r['ms_cold'] for r in rows):.3f} | | {sum(r['floor_MB'] for r in rows):.0f} | | | | | |")
    open(out + ".md", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
