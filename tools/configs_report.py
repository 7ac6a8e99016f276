"""GPU measurements of BASELINE.json's configs (SURVEY §8(d) "the five configs") that the
bench line does not carry, one JSON object per config (written to --out):

  config 1  one 512x512 tile (seed 1): whole tile (events, median of 20 after 3 warm-ups)
            and per stage (hp stage timing, median over the same 20)
  config 2  one 4K tile (seed 2): the same, median of 5
  config 3  DEVICE-RESIDENT: the 64-tile pool (seeds 1000..1063, 3 GiB) staged in HBM, 1000
            tiles (tile i = pool[i mod 64]) through 6 slots / 6 streams; the host-fed number
            is tools/run_dataset.py's
  config 5  the IWPP stress inputs at 4096^2 through HP_STAGE_IWPP_RAW: ms (events, best of
            3 after one warm-up), pixel updates/s (pixels whose value the reconstruction
            changes / time), engine statistics, and recon == mask

GPU only (the oracle is test infrastructure and is not called here)."""
import argparse
import json
import multiprocessing as mp
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1209_3332_b200 import Context  # noqa: E402
from synth import make_stress  # noqa: E402
from synth.hne import make_config_tile  # noqa: E402

STAGES = ["S1 CD", "S2 RBC", "S3 open", "S4 recon", "S5 area", "S6 fill", "S7 EDT",
          "S8 markers", "S9 watershed", "S10 bwlabel", "S11 features"]


def ev_ms(fn):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e)


class Bufs:
    def __init__(self, size, cap, n):
        d = "cuda"
        self.lab = [torch.empty((size, size), dtype=torch.int32, device=d) for _ in range(n)]
        self.nob = [torch.zeros(1, dtype=torch.int32, device=d) for _ in range(n)]
        self.tl = [torch.empty(cap, dtype=torch.int32, device=d) for _ in range(n)]
        self.tf = [torch.empty(cap, dtype=torch.int32, device=d) for _ in range(n)]
        self.tt = [torch.empty((cap, 36), dtype=torch.float32, device=d) for _ in range(n)]
        self.nr = [torch.zeros(1, dtype=torch.int32, device=d) for _ in range(n)]

    def run(self, ctx, k, rgb, stream=None):
        ctx.process_tile(k, rgb, self.lab[k], self.nob[k], self.tl[k], self.tf[k], self.tt[k], self.nr[k],
                         stream=stream)


def one_tile(cfg, reps):
    rgb_h = make_config_tile(cfg)
    h, w = rgb_h.shape[:2]
    ctx = Context(0, w, h, n_slots=1, max_objects=8192)
    b = Bufs(max(h, w), 8192, 1)
    b.lab = [torch.empty((h, w), dtype=torch.int32, device="cuda")]
    rgb = torch.from_numpy(rgb_h).cuda()
    for _ in range(3):
        b.run(ctx, 0, rgb)
    torch.cuda.synchronize()
    whole = [ev_ms(lambda: b.run(ctx, 0, rgb)) for _ in range(reps)]
    ctx.set_stage_timing(True)
    per = []
    for _ in range(reps):
        b.run(ctx, 0, rgb)
        torch.cuda.synchronize()
        per.append(ctx.stage_times(0))
    ctx.set_stage_timing(False)
    out = {"config": cfg, "tile": f"{w}x{h}", "reps": reps, "ms_median": statistics.median(whole),
           "ms_min": min(whole), "n_objects": int(b.nob[0].item()),
           "stage_ms_median": {STAGES[i]: round(statistics.median(p[i] for p in per), 4) for i in range(6)},
           "note": "events on the slot's stream around each stage; timing serialises nothing else "
                   "but adds the event records, so the stage sum slightly exceeds ms_median"}
    # the pipeline fuses S7-S11 (and the feature-stage Canny) into one step, timed in slot 7
    out["stage_ms_median"]["S7-S11 fused per component (+ Canny)"] = round(
        statistics.median(p[7] + p[6] + p[8] + p[9] + p[10] for p in per), 4)
    ctx.close()
    return out


def _gen(seed):
    import bench
    return bench._gen((seed, 4096))


def config3_device(n_tiles, slots):
    with mp.get_context("fork").Pool(max(1, min(16, os.cpu_count() or 1))) as pool:
        t0 = time.time()
        host = pool.map(_gen, list(range(1000, 1064)))
        gen_s = time.time() - t0
    dev = [torch.from_numpy(t).cuda() for t in host]
    del host
    ctx = Context(0, 4096, 4096, n_slots=slots, max_objects=8192)
    b = Bufs(4096, 8192, slots)
    streams = [torch.cuda.Stream() for _ in range(slots)]
    main_s = torch.cuda.current_stream()

    def run(n):
        ev0 = torch.cuda.Event()
        ev0.record(main_s)
        for s in streams:
            s.wait_event(ev0)
        for i in range(n):
            k = i % slots
            b.run(ctx, k, dev[i % len(dev)], stream=streams[k])
        for s in streams:
            e = torch.cuda.Event()
            e.record(s)
            main_s.wait_event(e)

    run(2 * slots)  # warm-up (graphs are not used on this path; first-use setup only)
    torch.cuda.synchronize()
    ms = ev_ms(lambda: run(n_tiles))
    out = {"config": 3, "mode": "device-resident", "pool": len(dev), "pool_gib": len(dev) * 3 * 4096 * 4096 / 2**30,
           "tiles": n_tiles, "slots": slots, "ms": ms, "tiles_per_s": n_tiles / (ms / 1e3),
           "pool_gen_s": round(gen_s, 1),
           "host_fed": "profiles/r01f_dataset_config3_1gpu.json (hp_run_tiles from pinned host memory)"}
    ctx.close()
    return out


def config5():
    size = 4096
    ctx = Context(0, size, size, n_slots=1, max_objects=16)
    rec = torch.empty((size, size), dtype=torch.uint8, device="cuda")
    st = torch.zeros(4, dtype=torch.int64, device="cuda")
    res = []
    for kind in ["serpentine", "spiral"]:
        for ramp in [False, True]:
            mk_h, mask_h, L = make_stress(kind, size, ramp)
            changed = int(np.count_nonzero(np.minimum(mk_h, mask_h) != mask_h))
            mk, mask = torch.from_numpy(mk_h).cuda(), torch.from_numpy(mask_h).cuda()

            def call():
                ctx.stage_run(0, "IWPP_RAW", [mk, mask], [rec, st], size, size)
            call()
            torch.cuda.synchronize()
            t = [ev_ms(call) for _ in range(3)]
            ms = min(t)
            res.append({"case": f"{kind} {'ramp' if ramp else 'binary'}", "path_px": int(L), "ms": ms,
                        "ms_all": [round(x, 2) for x in t], "pixels_changed": changed,
                        "updates_per_s": changed / (ms / 1e3), "jobs": int(st[0]), "sweep_iterations": int(st[1]), "owned_ns": int(st[2]), "stat3": int(st[3]),
                        "recon_eq_mask": bool(torch.equal(rec, mask))})
    ctx.close()
    return {"config": 5, "size": size, "cases": res,
            "note": "1-px corridors: a strictly sequential dependency chain of 0.5 N pixels; the "
                    "region engine propagates it region by region (the GPU may lose to a CPU FIFO here)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/configs_report.json")
    ap.add_argument("--configs", default="1,2,3,5")
    ap.add_argument("--c3-tiles", type=int, default=1000)
    ap.add_argument("--slots", type=int, default=6)
    a = ap.parse_args()
    want = {int(x) for x in a.configs.split(",")}
    dev = torch.cuda.get_device_name(0)
    out = {"device": dev, "results": []}
    for cfg, fn in [(1, lambda: one_tile(1, 20)), (2, lambda: one_tile(2, 5)),
                    (5, config5), (3, lambda: config3_device(a.c3_tiles, a.slots))]:
        if cfg in want:
            r = fn()
            print(json.dumps(r), flush=True)
            out["results"].append(r)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
