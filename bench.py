#!/usr/bin/env python
"""bench.py -- 4K x 4K tiles/s (segmentation + features) on N B200s, one process per GPU.

A step = one pass of the whole hot path (S1..S11) over a batch of B
distinct synthetic 4096x4096 H&E tiles per GPU (BASELINE.json configs[1] tile shape).
  value  device-resident tiles/s: inputs already in HBM, CUDA events on the launching
         stream with every slot stream joined, max over ranks, all ranks' tiles counted.
  e2e    the same metric through the public multi-tile driver hp_run_tiles: pinned host
         tiles, H2D of every tile and D2H of its feature rows inside the timed region.
Tiles shard across ranks with no data-path collective ("scaling": "weak").
--impl reference times the CPU oracle (oracle/, the deliberately plain checker) on the
box's host cores on bounded samples of the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

# Every slot runs its tile chain on its own stream.  The default 8 hardware work queues alias
# more streams onto shared queues, which serialises kernels of different slots behind each
# other (r1: 12 slots 878 -> 934 tiles/s, a forked side stream per tile 674 -> 907 with 32).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "4K×4K tiles/s (seg+features) at 1/2/4/8 B200; per-stage HBM GB/s"
UNIT = "tiles/s"
STAGES = ["S1 colour deconvolution", "S2 RBC detection", "S3 morph open 19x19",
          "S4 ReconToNuclei (IWPP)", "S5 AreaThreshold", "S6 FillHoles", "S7 EDT",
          "S8 markers (IWPP f32 + RMAX)", "S9 watershed (W1-W3)", "S10 BWLabel",
          "S11 features"]
# algorithmic floor bytes per pixel of each stage (read each input once,
# write each output once, in the §8(a) layouts); DESIGN.md "Roofline" restates them.
FLOOR_BPP = [5, 2, 2, 4, 2, 2, 5, 9, 10, 5, 5]
DTYPE = "u8/i32/f32"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


# ----------------------------------------------------------------- inputs
def _gen(args):
    seed, size = args
    from synth.hne import TileSpec, make_tile
    cache = os.path.join(tempfile.gettempdir(), "hp_bench_tiles")
    os.makedirs(cache, exist_ok=True)
    fn = os.path.join(cache, f"t{seed}_{size}.npy")
    if os.path.exists(fn):
        try:
            return np.load(fn)
        except Exception:  # noqa: BLE001
            pass
    rgb = make_tile(seed, TileSpec(size, size))["rgb"]
    tmp = f"{fn}.{os.getpid()}.tmp.npy"  # per process: ranks may generate the same tile at once
    np.save(tmp, rgb)
    os.replace(tmp, fn)
    return rgb


def make_tiles(rank, batch, size):
    # configs[2] pool seeds.  Every rank gets the SAME tiles: weak scaling with identical
    # per-GPU work (tile content varies ~5x in reconstruction cost, and the max-over-ranks
    # timer would otherwise measure the unluckiest rank's draw); the e2e leg shares one
    # demand-driven queue across ranks instead.
    del rank
    seeds = [1000 + i for i in range(batch)]
    nproc = max(1, min(len(seeds), (os.cpu_count() or 2) // max(1, env_int("LOCAL_WORLD_SIZE", 1))))
    ctx = mp.get_context("fork")
    with ctx.Pool(nproc) as pool:
        return pool.map(_gen, [(s, size) for s in seeds])


# ----------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampler for the clocks line: started before the warm-up (so it is producing
    samples by the time the timed region starts), every sample timestamped, and only the
    samples inside [timed-region start, end + one period] count (at least one: stop() waits
    for the first sample after the region if the region was shorter than a period)."""
    Q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    PERIOD_MS = 50

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.fn = None
        self.t0 = self.t1 = None

    def start(self):
        try:
            fd, self.fn = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "-i", str(self.index),
                 "--format=csv,noheader,nounits", "-lms", str(self.PERIOD_MS)],
                stdout=open(self.fn, "w"), stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.proc = None

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def _read(self):
        import datetime
        rows = []
        for line in open(self.fn):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(f[1]), float(f[2]), f[4:8]))
            except ValueError:
                continue
        return rows

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t1 = self.t1 if self.t1 is not None else time.time()
        t0 = self.t0 if self.t0 is not None else t1
        hi = t1 + self.PERIOD_MS / 1000.0
        deadline = time.time() + 5.0
        rows = []
        while time.time() < deadline:  # until a sample at or after the region's end exists
            rows = self._read()
            if any(r[0] >= t1 for r in rows):
                break
            time.sleep(self.PERIOD_MS / 1000.0)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        rows = self._read()
        os.unlink(self.fn)
        inside = [r for r in rows if t0 <= r[0] <= hi]
        if not inside:  # region shorter than a period: the first sample after its start
            after = [r for r in rows if r[0] >= t0]
            inside = after[:1]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in inside:
            for n, v in zip(names, r[3]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        sm = [r[1] for r in inside]
        mx = [r[2] for r in inside]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm), "sample_ms": self.PERIOD_MS}


def peaks():
    fn = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(fn))
        return float(d["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


def traffic_for(stage_idx):
    """dram bytes per launch of the dominant stage's kernels from a committed ncu capture."""
    fn = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(fn))
        return d.get("per_stage_bytes", {}).get(str(stage_idx))
    except Exception:  # noqa: BLE001
        return None


# ----------------------------------------------------------------- CPU oracle leg
def _oracle_tile(i):
    import oracle
    t0 = time.perf_counter()
    oracle.process_tile(_POOL_TILES[i % len(_POOL_TILES)], cap=65536)
    return time.perf_counter() - t0


_POOL_TILES = []


def oracle_rate(tiles, n_tiles, workers):
    """Oracle tiles/s on `workers` host processes over n_tiles tiles (one tile per task)."""
    global _POOL_TILES
    _POOL_TILES = tiles
    import oracle
    oracle.build()
    ctx = mp.get_context("fork")
    with ctx.Pool(workers) as pool:
        t0 = time.perf_counter()
        pool.map(_oracle_tile, range(n_tiles), chunksize=1)
        wall = time.perf_counter() - t0
    return n_tiles / wall, wall


def cpu_workers():
    return max(1, min(os.cpu_count() or 1, 32))


# ----------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="hp", choices=["hp", "reference"])
    ap.add_argument("--batch", type=int, default=12, help="distinct 4K tiles per GPU per step")
    ap.add_argument("--slots", type=int, default=12, help="tiles in flight per GPU (n_slots)")
    ap.add_argument("--e2e-slots", type=int, default=24,
                    help="context slots used by hp_run_tiles (e2e); r2 sweep: 10 947, 14 953, 18 963, 24 963 tiles/s")
    ap.add_argument("--size", type=int, default=4096)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--schedule", default="rotate", choices=["rotate", "join", "fixed"],
                    help="one GPU: steps unjoined with tiles rotating over slots (default), every step "
                         "joined (r1), or unjoined with fixed slots")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    workload = (f"configs[1] tile shape: {args.size}x{args.size} synthetic H&E RGB tiles, "
                f"segmentation+features; {args.batch} distinct tiles per GPU per step")
    config = {"workload": workload, "tile": f"{args.size}x{args.size}x3 u8",
              "batch_per_gpu": args.batch, "slots": args.slots, "e2e_slots": max(args.slots, args.e2e_slots),
              "l2": "inputs larger than L2 (each step reads %d distinct tiles = %.0f MB)"
                    % (args.batch, args.batch * 3 * args.size * args.size / 1e6),
              "parallelism": (f"tiles sharded over {world} GPU(s) by a shared demand-driven tile queue "
                              f"({world}x{args.batch} tiles per step), no data-path collective" if world > 1 else
                              "one GPU, all tiles of a step in flight")}

    if args.impl == "reference":
        if rank != 0:
            return 0
        tiles = make_tiles(0, args.batch, args.size)
        P = cpu_workers()
        for _ in range(args.warmup):
            oracle_rate(tiles, P, P)
        vals, walls = [], []
        for _ in range(args.steps):
            v, w = oracle_rate(tiles, P, P)
            vals.append(v)
            walls.append(w)
        total_t = sum(walls)
        value = P * args.steps / total_t
        sample = f"{P} tiles per step (one per host process), cycling {len(tiles)} distinct tiles"
        line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1000 * total_t / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": DTYPE,
                "data": "synthetic (seeded H&E painter, synth/hne.py)", "config": config,
                "cpu_baseline": {"value": value, "unit": UNIT, "cores": P, "kind": "oracle",
                                 "sample": sample},
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    from paper_1209_3332_b200.dist import bind_to_gpu_numa
    all_cores = sorted(os.sched_getaffinity(0))
    near = bind_to_gpu_numa(local)  # pinned tiles and the feeder thread on the GPU's NUMA node
    log(f"[rank {rank}] bound to {len(near) if near else 'all'} cores near GPU {local}")
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1209_3332_b200 import Context, hp

    B, S, size = args.batch, args.slots, args.size
    t_gen = time.time()
    tiles = make_tiles(rank, B, size)
    log(f"[rank {rank}] generated {B} tiles in {time.time() - t_gen:.1f}s")
    cap = 8192
    # the device-resident step uses S slots; hp_run_tiles (e2e) uses every slot of the context:
    # more tiles in flight hide each slot's own H2D behind the others' compute
    ctx = Context(local, size, size, n_slots=max(S, args.e2e_slots), max_objects=cap)
    dev = [torch.from_numpy(t).cuda() for t in tiles]
    lab = [torch.empty((size, size), dtype=torch.int32, device="cuda") for _ in range(S)]
    nob = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(S)]
    tl = [torch.empty(cap, dtype=torch.int32, device="cuda") for _ in range(S)]
    tf = [torch.empty(cap, dtype=torch.int32, device="cuda") for _ in range(S)]
    tt = [torch.empty((cap, 36), dtype=torch.float32, device="cuda") for _ in range(S)]
    nr = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(S)]
    streams = [torch.cuda.Stream() for _ in range(S)]
    main_s = torch.cuda.current_stream()

    def process(tid, k):
        ctx.process_tile(k, dev[tid % B], lab[k], nob[k], tl[k], tf[k], tt[k], nr[k], stream=streams[k])

    def step(key, nsteps=1):
        """nsteps steps of B tiles per GPU.  One GPU: all B tiles of a step in flight on the S
        slot streams, steps queued back to back.  N GPUs: the N*B*nsteps tiles are pulled from
        the shared demand-driven tile queue -- a slot takes the next tile id
        when its previous tile is done, so a faster GPU takes more tiles, and no GPU idles at
        a step boundary; tile id t is pool tile t mod B (every rank holds the pool in HBM)."""
        ev0 = torch.cuda.Event()
        ev0.record(main_s)
        for s in streams:
            s.wait_event(ev0)
        if world == 1:
            # steps are not joined: each slot stream runs its tiles back to back, and tile i of
            # step k goes to slot (i + k) mod S, so the chain-bound tiles (3 of the 12 take
            # 3-6x longer) rotate over the slots instead of piling up on three streams
            for k in range(nsteps):
                if args.schedule == "join" and k:  # r1 schedule: every step joined, fixed slots
                    e = torch.cuda.Event()
                    for st in streams:
                        e2 = torch.cuda.Event()
                        e2.record(st)
                        main_s.wait_event(e2)
                    e.record(main_s)
                    for st in streams:
                        st.wait_event(e)
                for i in range(B):
                    process(i, (i + k) % S if args.schedule == "rotate" else i % S)
        else:
            from paper_1209_3332_b200.dist import TileQueue
            q = TileQueue(world * B * nsteps, block=2, key=key)
            ids, free, busy = iter(()), list(range(S)), {}
            drained = False
            while True:
                while free and not drained:
                    tid = next(ids, None)
                    if tid is None:
                        blk = q.grab()
                        if blk is None:
                            drained = True
                            break
                        ids = iter(blk)
                        continue
                    k = free.pop()
                    process(tid, k)
                    e = torch.cuda.Event()
                    e.record(streams[k])
                    busy[k] = e
                    taken[0] += 1
                if not busy:
                    break
                fin = [k for k, e in busy.items() if e.query()]
                if not fin:
                    time.sleep(20e-6)
                for k in fin:
                    del busy[k]
                    free.append(k)
        for s in streams:
            e = torch.cuda.Event()
            e.record(s)
            main_s.wait_event(e)

    taken = [0]

    def barrier():
        if world > 1:
            dist.barrier()

    clocks = Clocks(local)
    clocks.start()  # before the warm-up: nvidia-smi takes a while to produce its first sample
    step("hp/dev/warm", args.warmup)
    torch.cuda.synchronize()
    objs = sum(int(n.item()) for n in nr)
    taken[0] = 0

    # per-stage events inside the timed region (the roofline's in-situ stage times);
    # HP_BENCH_NO_TIMING=1 measures the value without them (experiments)
    stage_timing = os.environ.get("HP_BENCH_NO_TIMING") != "1"
    ctx.set_stage_timing(stage_timing)
    barrier()
    torch.cuda.synchronize()
    l0 = hp.launch_count()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks.mark_start()
    start.record(main_s)
    step("hp/dev/timed", args.steps)
    end.record(main_s)
    torch.cuda.synchronize()
    clocks.mark_end()
    barrier()
    launches = hp.launch_count() - l0
    clk = clocks.stop()
    ms = start.elapsed_time(end)
    stage_sum, ntiles_timed = ctx.stage_times_accum() if stage_timing else ([0.0] * 11, 0)
    ctx.set_stage_timing(False)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * B * args.steps / (ms_max / 1000.0)
    log(f"[rank {rank}] device-resident {value:.1f} tiles/s ({ms_max / args.steps:.2f} ms per step)")

    # Per stage: (a) isolated -- each of the B tiles alone on one slot, nothing else on the GPU,
    # stage events on its stream: what bounds the stage; (b) in situ -- the same events inside
    # the timed region, where ~B tiles share the GPU (the roofline object's basis, as the
    # contract asks).  Floor bytes are SURVEY §8(d)'s per stage (S7-S11, fused in one launch
    # chain per tile, take the sum of their five floors: 34 B/px); the Canny of the feature
    # stage is timed inside S7-S11 (events 7..11).
    iso_sum, iso_n = [0.0] * 11, 0
    if stage_timing:
        ctx.set_stage_timing(True)
        for i in range(B):
            process(i, 0)
            torch.cuda.synchronize()
        iso_sum, iso_n = ctx.stage_times_accum()
        ctx.set_stage_timing(False)
    npx = size * size
    peak, peak_kind = peaks()
    per_stage = []
    fused = os.environ.get("HP_GLOBAL_S8S10", "0") != "1"
    groups = [(STAGES[k], [k], FLOOR_BPP[k]) for k in range(6)]
    if fused:
        groups.append(("S7-S11 fused per component (Canny, EDT, markers, watershed, BWLabel, features)",
                       list(range(6, 11)), sum(FLOOR_BPP[6:11])))
    else:
        groups += [(STAGES[k], [k], FLOOR_BPP[k]) for k in range(6, 11)]
    for name, ks, bpp in groups:
        ms_in = sum(stage_sum[k] for k in ks) / max(1, ntiles_timed)
        ms_iso = sum(iso_sum[k] for k in ks) / max(1, iso_n)
        g_in = bpp * npx / (ms_in / 1e3) / 1e9 if ms_in > 0 else None
        g_iso = bpp * npx / (ms_iso / 1e3) / 1e9 if ms_iso > 0 else None
        per_stage.append({"stage": name, "alg_bytes_per_tile": bpp * npx,
                          "ms_isolated": round(ms_iso, 4),
                          "alg_GBps_isolated": None if g_iso is None else round(g_iso, 1),
                          "frac_isolated": None if g_iso is None else round(g_iso / peak, 4),
                          "ms_in_situ": round(ms_in, 4),
                          "alg_GBps_in_situ": None if g_in is None else round(g_in, 1),
                          "frac_in_situ": None if g_in is None else round(g_in / peak, 4)})
    dom = max(range(len(per_stage)), key=lambda k: per_stage[k]["ms_in_situ"])
    dstage = per_stage[dom]
    roofline = {"bound": "hbm", "kernel": dstage["stage"], "achieved": dstage["alg_GBps_in_situ"],
                "peak": peak, "unit": "GB/s",
                "frac": dstage["frac_in_situ"], "traffic": traffic_for(dom),
                "peak_kind": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)",
                "basis": "in-situ stage events (its stream, inside the timed region, ~B tiles sharing the GPU)",
                "achieved_isolated": dstage["alg_GBps_isolated"], "frac_isolated": dstage["frac_isolated"],
                "share_of_step": round(dstage["ms_in_situ"] / max(1e-9, sum(p["ms_in_situ"] for p in per_stage)), 4)}
    if dstage["stage"].startswith("S4"):
        # what actually bounds it (DESIGN.md §11 "S4 latency bound", profiles/r02_final_stage_table.md)
        roofline["limiter"] = ("latency: dependent chains of region jobs / row closures (ncu: ~25% warps "
                               "active, ~34% issue active, ~82% L2 hit; DRAM bytes below the floor)")

    # e2e through hp_run_tiles: pinned host tiles, H2D + D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        # the production path: a demand-driven tile queue shared by all ranks (PAPER.md:
        # 370-389) and hp_run_tiles with per-slot H2D/compute/D2H streams, each tile's rows
        # delivered to the host; the NCCL gather of all rows to rank 0 follows, untimed
        from paper_1209_3332_b200.dist import DistTileSource, TileQueue, gather_rows, table_digest
        pinned = [torch.from_numpy(x).pin_memory() for x in tiles]
        rows_copied = min(cap, 4096)
        d2h_per_tile = 4 + rows_copied * (4 + 4 + 36 * 4)

        def run(ntiles, key):
            q = TileQueue(ntiles, block=S, key=key)
            src = DistTileSource(q, lambda tid: pinned[tid % B])
            results = {}

            def done(tid, l, f, ft, st):
                if st != 0:
                    raise RuntimeError(f"tile {tid} status {st}")
                results[tid] = (l, f, ft)

            ctx.run_tiles(src, done, size, size)
            torch.cuda.synchronize()
            return results, len(src.taken)

        run(world * B * max(1, args.warmup), "hp/warm")
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        results, mine = run(world * B * args.steps, "hp/timed")
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        barrier()
        tw = torch.tensor([wall], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tw, op=dist.ReduceOp.MAX)
        # after the timed region: the cross-rank gather of every row to rank 0 (NCCL), which
        # proves the sharded table equals the 1-GPU one (digest) -- reported, not timed
        tg = time.perf_counter()
        table = gather_rows(results, device=torch.device("cuda", local))
        gather_ms = 1e3 * (time.perf_counter() - tg)
        e2e = {"value": world * B * args.steps / float(tw.item()), "unit": UNIT,
               "h2d_bytes_per_step": world * B * 3 * size * size,
               "d2h_bytes_per_step": world * B * d2h_per_tile,
               "api": "hp_run_tiles fed by the shared demand-driven tile queue; every tile's rows "
                      "delivered to its rank's host by the sink callback inside the timed region",
               "timer": "host wall clock bracketed by device synchronize and barriers, max over ranks",
               "rows_gathered": None if table is None else int(len(table)),
               "gather_ms_untimed": round(gather_ms, 1),
               "table_digest": None if table is None else table_digest(table)}

        # NEXT-3 compressed ingest: the same tiles as quality-90 4:4:4
        # baseline JPEG files (restart interval 4 MCUs) through hp_run_tiles_jpeg -- only the
        # file crosses PCIe, decoding runs on the GPU fused into S1.  Reported beside e2e (the
        # decoded tiles differ from the raw ones by the JPEG loss, so the table does too).
        from synth.jpeg import encode_tile
        jp = [torch.from_numpy(encode_tile(x)).pin_memory() for x in tiles]

        def run_jpeg(ntiles, key):
            q = TileQueue(ntiles, block=S, key=key)
            ids, got, nbytes = iter(()), {}, [0]

            def nxt():
                nonlocal ids
                while True:
                    tid = next(ids, None)
                    if tid is not None:
                        b = jp[tid % B]
                        nbytes[0] += int(b.numel())
                        return b.data_ptr(), int(b.numel()), tid
                    blk = q.grab()
                    if blk is None:
                        return None
                    ids = iter(blk)

            def done(tid, l, f, ft, st):
                if st != 0:
                    raise RuntimeError(f"jpeg tile {tid} status {st}")
                got[tid] = len(l)

            ctx.run_tiles_jpeg(nxt, done, size, size)
            torch.cuda.synchronize()
            return got, nbytes[0]

        run_jpeg(world * B * max(1, args.warmup), "hp/jwarm")
        barrier()
        t0 = time.perf_counter()
        got, jbytes = run_jpeg(world * B * args.steps, "hp/jtimed")
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        barrier()
        tw = torch.tensor([wall, jbytes], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tw[:1], op=dist.ReduceOp.MAX)
            dist.all_reduce(tw[1:], op=dist.ReduceOp.SUM)
        e2e["jpeg"] = {"value": world * B * args.steps / float(tw[0].item()), "unit": UNIT,
                       "h2d_bytes_per_step": float(tw[1].item()) / args.steps,
                       "d2h_bytes_per_step": world * B * d2h_per_tile,
                       "api": "hp_run_tiles_jpeg (NEXT-3): JPEG files q90 4:4:4, restart interval 4 MCUs, "
                              "decoded on the GPU inside S1",
                       "raw_over_jpeg_bytes": round(3 * size * size * B / sum(int(b.numel()) for b in jp), 2),
                       "rows_per_tile": sum(got.values()) / max(1, len(got))}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        os.sched_setaffinity(0, all_cores)  # the CPU baseline uses every host core
        P = cpu_workers()
        n = 2 * P
        v, w = oracle_rate(tiles, n, P)
        cpu = {"value": v, "unit": UNIT, "cores": P, "kind": "oracle",
               "sample": f"{n} tiles of the same workload ({len(tiles)} distinct 4K tiles cycled), "
                         f"one tile per host process, {w:.1f}s wall"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": DTYPE,
                "data": "synthetic (seeded H&E painter, synth/hne.py)", "config": config,
                "e2e": e2e, "gpu_launches": int(launches), "roofline": roofline,
                "per_stage": per_stage, "cpu_baseline": cpu, "clocks": clk,
                "objects_per_tile": objs / max(1, S), "impl": "hp"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    ctx.close()
    return 0


if __name__ == "__main__":
    try:
        rc = main()
    except BaseException:  # report loudly: a rank that dies silently is undiagnosable
        import traceback
        traceback.print_exc()
        sys.stderr.flush()
        raise
    sys.exit(rc)
