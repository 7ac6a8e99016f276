"""Dataset runs of BASELINE.json configs[2] and configs[3]:

  config 3: 1,000 synthetic 4K tiles from a pool of P distinct tiles, 1 GPU
  config 4: 36,848 tiles (340 "slides" x ~108 tiles, per-slide nucleus density, per-tile
            tissue fraction) demand-driven across N GPUs; the gathered
            table's digest must be the same for every N.

Tile i is pool[i mod P]; the P pool tiles are spread over the whole dataset (pool k = dataset
tile k * T / P), so a tile's content depends only on its id and the table is comparable
across GPU counts.  Each rank runs hp_run_tiles (or hp_run_tiles_jpeg with --jpeg: the pool
held as quality-90 JPEG files, NEXT-3) from pinned host memory with the rows appended to a
device row arena (they never leave the GPU during the run); at the end every rank's rows go
to rank 0 device to device (gather_rows_device, NCCL point-to-point), and the per-slide
aggregation (NEXT-4) runs on every rank's own rows with two NCCL all-reduces.

usage: python tools/run_dataset.py --config 3 [--tiles 1000] [--pool 64]
       torchrun --nproc-per-node N tools/run_dataset.py --config 4 [--jpeg] [--pool 128]
"""
import argparse
import hashlib
import json
import os

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # one stream per slot (see bench.py)
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pool_index(config, k, pool, n_tiles):
    return k if config == 3 else (k * n_tiles) // pool


def _cache(name):
    import tempfile
    d = os.path.join(tempfile.gettempdir(), "hp_ds_tiles")
    os.makedirs(d, exist_ok=True)
    return os.path.join(d, name)


def pool_tile(args):
    """Generate (or load) one pool tile; returns its raw RGB and, with jpeg, its JPEG bytes."""
    config, idx, jpeg = args
    from synth.hne import make_config_tile
    fn = _cache(f"c{config}_{idx}.npy")
    if os.path.exists(fn):
        rgb = np.load(fn)
    else:
        rgb = make_config_tile(config, idx)
        tmp = f"{fn}.{os.getpid()}.tmp.npy"  # per process: ranks may generate the same tile at once
        np.save(tmp, rgb)
        os.replace(tmp, fn)
    if not jpeg:
        return rgb, None
    from synth.jpeg import encode_tile
    jf = _cache(f"c{config}_{idx}.jpg")
    if os.path.exists(jf):
        buf = np.fromfile(jf, dtype=np.uint8)
    else:
        buf = encode_tile(rgb)
        tmp = f"{jf}.{os.getpid()}.tmp"
        buf.tofile(tmp)
        os.replace(tmp, jf)
    return rgb, buf


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4, choices=[3, 4])
    ap.add_argument("--tiles", type=int, default=None)
    ap.add_argument("--pool", type=int, default=None)
    ap.add_argument("--slots", type=int, default=14)
    ap.add_argument("--jpeg", action="store_true", help="NEXT-3: feed the pool as JPEG files")
    ap.add_argument("--rows-per-tile", type=int, default=3000, help="arena capacity per tile taken")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    n_tiles = args.tiles or (1000 if args.config == 3 else 36848)
    P = args.pool or (64 if args.config == 3 else 128)

    import multiprocessing as mp

    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1209_3332_b200.dist import (RowArena, TileQueue, aggregate_groups, bind_to_gpu_numa,
                                           gather_rows_device, sort_rows)
    from paper_1209_3332_b200 import Context

    # pool: rank r generates every world-th tile (shared cache), then every rank loads all
    t0 = time.time()
    ncpu = max(1, (os.cpu_count() or 2) // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", 1))))
    mine = [(args.config, pool_index(args.config, k, P, n_tiles), args.jpeg) for k in range(P) if k % world == rank]
    with mp.get_context("fork").Pool(min(ncpu, max(1, len(mine)))) as pl:
        pl.map(pool_tile, mine)
    if world > 1:
        dist.barrier()
    with mp.get_context("fork").Pool(min(ncpu, P)) as pl:
        loaded = pl.map(pool_tile, [(args.config, pool_index(args.config, k, P, n_tiles), args.jpeg) for k in range(P)])
    gen_s = time.time() - t0
    bind_to_gpu_numa(local)  # pinned pool and feeder thread on the GPU's NUMA node
    if args.jpeg:
        pool = [torch.from_numpy(b).pin_memory() for _, b in loaded]
        pool_bytes = sum(int(b.numel()) for b in pool)
    else:
        pool = [torch.from_numpy(r).pin_memory() for r, _ in loaded]
        pool_bytes = sum(int(r.numel()) for r in pool)
    del loaded
    ctx = Context(local, 4096, 4096, n_slots=args.slots, max_objects=16384)
    cap_rows = args.rows_per_tile * (n_tiles // world + 4 * args.slots) + 65536
    arena = RowArena(cap_rows, torch.device("cuda", local))
    bad = []

    def done(tid, n, st):
        if st != 0:
            bad.append((tid, st))

    q = TileQueue(n_tiles, block=2, key=f"hp/ds/{args.config}/{int(args.jpeg)}")
    taken = []

    def nxt():
        if not hasattr(nxt, "it") or nxt.it is None:
            nxt.it = None
        while True:
            if nxt.it is not None:
                tid = next(nxt.it, None)
                if tid is not None:
                    taken.append(tid)
                    t = pool[tid % P]
                    return t.data_ptr(), (t.numel() if args.jpeg else t.stride(0)), tid
            blk = q.grab()
            if blk is None:
                return None
            nxt.it = iter(blk)

    nxt.it = None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    if args.jpeg:
        ctx.run_tiles_jpeg(nxt, done, 4096, 4096, arena=arena.arena)
    else:
        ctx.run_tiles(nxt, done, 4096, 4096, arena=arena.arena)
    torch.cuda.synchronize()
    t_run = time.perf_counter() - t1
    mine_rows = arena.rows()
    n_mine = len(mine_rows)
    if world > 1:
        # NCCL sets up its point-to-point channels on the first send/recv between two ranks;
        # a one-row gather does that outside the timed gather
        from paper_1209_3332_b200.dist import DeviceRows
        gather_rows_device(DeviceRows(mine_rows.tile[:1], mine_rows.label[:1], mine_rows.flags[:1],
                                      mine_rows.feat[:1]))
        torch.cuda.synchronize()
        dist.barrier()
    tg = time.perf_counter()
    gstats = {}
    table = gather_rows_device(mine_rows, stats=gstats)
    torch.cuda.synchronize()
    t_gather = time.perf_counter() - tg
    # per-slide aggregation on each rank's own rows, two NCCL all-reduces
    per_slide = 108 if args.config == 4 else n_tiles
    n_groups = (n_tiles + per_slide - 1) // per_slide
    ta = time.perf_counter()
    cnt, mean, std = aggregate_groups(sort_rows(mine_rows), lambda t: t // per_slide, n_groups, reduce=ctx,
                                      device=torch.device("cuda", local))
    agg_ms = 1e3 * (time.perf_counter() - ta)
    tt = torch.tensor([t_run, t_gather], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    nb = torch.tensor([len(bad), n_mine, len(taken)], dtype=torch.int64, device="cuda")
    if world > 1:
        dist.all_reduce(nb, op=dist.ReduceOp.SUM)
    if rank == 0:
        host = table.to_host()
        h = hashlib.sha256()
        for name in ("tile", "label", "flags", "feat"):
            h.update(np.ascontiguousarray(getattr(host, name)).view(np.uint8).tobytes())
        gathered_bytes = (len(table) - n_mine) * (8 + 4 + 4 + 4 * 36)  # rows received from other ranks
        line = {"config": args.config, "tiles": n_tiles, "n_gpus": world, "pool": P, "slots": args.slots,
                "ingest": "jpeg q90 4:4:4 rst4 (hp_run_tiles_jpeg)" if args.jpeg else "raw RGB (hp_run_tiles)",
                "host_bytes_per_tile": pool_bytes / P,
                "tiles_per_s": n_tiles / float(tt[0]), "run_s": float(tt[0]), "gather_s": float(tt[1]),
                "gather_GBps": gathered_bytes / float(tt[1]) / 1e9 if float(tt[1]) > 0 else None,
                "gather_transfer_s": gstats.get("transfer_s"), "gather_merge_s": gstats.get("merge_s"),
                "gather_transfer_GBps": (gathered_bytes / gstats["transfer_s"] / 1e9
                                         if gstats.get("transfer_s") else None),
                "rows": int(len(table)), "rows_rank0": n_mine, "tiles_taken_total": int(nb[2]),
                "failed_tiles": int(nb[0]), "digest": h.hexdigest()[:16], "pool_gen_s": round(gen_s, 1),
                "groups": n_groups, "group_rows": int(cnt.sum()), "agg_ms": round(agg_ms, 1),
                "agg_checksum": float(np.nansum(mean) + np.nansum(std))}
        print(json.dumps(line), flush=True)
        if args.out:
            with open(args.out, "w") as f:
                json.dump(line, f, indent=1)
    if world > 1:
        dist.destroy_process_group()
    ctx.close()


if __name__ == "__main__":
    main()
