"""GPU diagnostic: IWPP work statistics and timings on the config-2 tile and the stress
inputs, plus per-stage times of one tile on one slot.  Prints one JSON line per case."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1209_3332_b200 import Context  # noqa: E402
from synth import make_stress  # noqa: E402
from synth.hne import make_config_tile  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


def main():
    size = 4096
    ctx = Context(0, size, size, n_slots=1, max_objects=8192)
    pool = [a for a in sys.argv if a.startswith("--pool=")]
    src = make_config_tile(3, int(pool[0].split("=")[1])) if pool else make_config_tile(2)
    rgb = torch.from_numpy(src).cuda()
    g = torch.empty((size, size), dtype=torch.uint8, device="cuda")
    fl = torch.empty_like(g)
    nbg = torch.zeros(1, dtype=torch.int64, device="cuda")
    ctx.stage_run(0, "CD", [rgb], [g, fl, nbg], size, size)
    op = torch.empty_like(g)
    ctx.stage_run(0, "OPEN", [g], [op], size, size)
    rec = torch.empty_like(g)
    st = torch.zeros(4, dtype=torch.int64, device="cuda")
    ms = timed(lambda: ctx.stage_run(0, "IWPP_RAW", [op, g], [rec, st], size, size))
    ntiles = (size // 32) ** 2
    print(json.dumps({"case": "recon(open, g) " + (pool[0] if pool else "config2"), "ms": ms,
                      "jobs": int(st[0]), "iterations": int(st[1]),
                      "owned_ms_total": int(st[2]) / 1e6, "avg_parallel_regions": int(st[2]) / 1e6 / ms,
                      "us_per_job": int(st[2]) / 1e3 / max(1, int(st[0])), "row_closures": int(st[3])}),
          flush=True)
    for kind in ([] if "--quick" in sys.argv else ["serpentine", "spiral"]):
        for ramp in [False, True]:
            mk, mask, L = make_stress(kind, size, ramp)
            mk, mask = torch.from_numpy(mk).cuda(), torch.from_numpy(mask).cuda()
            t0 = time.time()
            ctx.stage_run(0, "IWPP_RAW", [mk, mask], [rec, st], size, size)
            torch.cuda.synchronize()
            ms = (time.time() - t0) * 1e3
            ok = bool(torch.equal(rec, mask))
            print(json.dumps({"case": f"stress {kind} ramp={ramp}", "ms": ms, "ok": ok,
                              "tile_jobs": int(st[0]), "rounds": int(st[1]), "path": L}), flush=True)
    # per-stage times of one tile, one slot
    lab = torch.empty((size, size), dtype=torch.int32, device="cuda")
    nob = torch.zeros(1, dtype=torch.int32, device="cuda")
    cap = 8192
    tl = torch.empty(cap, dtype=torch.int32, device="cuda")
    tf = torch.empty(cap, dtype=torch.int32, device="cuda")
    tt = torch.empty((cap, 36), dtype=torch.float32, device="cuda")
    nr = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.process_tile(0, rgb, lab, nob, tl, tf, tt, nr)
    torch.cuda.synchronize()
    ctx.set_stage_timing(True)
    ms = timed(lambda: ctx.process_tile(0, rgb, lab, nob, tl, tf, tt, nr), reps=3)
    sums, n = ctx.stage_times_accum()
    print(json.dumps({"case": "process_tile 1 slot", "ms": ms, "n_objects": int(nob.item()),
                      "stage_ms": [round(x / n, 3) for x in sums]}), flush=True)


if __name__ == "__main__":
    main()
