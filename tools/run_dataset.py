"""Dataset runs of BASELINE.json configs[2] and configs[3]:

  config 3: 1,000 synthetic 4K tiles from a pool of P distinct tiles, 1 GPU, async prefetch
  config 4: 36,848 tiles (340 "slides" x ~108 tiles, per-slide nucleus density, per-tile tissue
            fraction) demand-driven across N GPUs; the gathered table's digest must be the
            same for every N.

Tile i is pool[i mod P] (P distinct tiles generated once per rank, cached under /tmp), so a
tile's content depends only on its id -- the table is comparable across GPU counts.

usage: python tools/run_dataset.py --config 3 [--tiles 1000] [--pool 16] [--slots 2]
       torchrun --nproc-per-node N tools/run_dataset.py --config 4 --tiles 36848 --pool 16
"""
import argparse
import json
import os

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # one stream per slot (see bench.py)
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pool_tile(config, k):
    import tempfile
    from synth.hne import make_config_tile
    fn = os.path.join(tempfile.gettempdir(), "hp_ds_tiles", f"c{config}_{k}.npy")
    os.makedirs(os.path.dirname(fn), exist_ok=True)
    if os.path.exists(fn):
        return np.load(fn)
    rgb = make_config_tile(config, k)
    tmp = f"{fn}.{os.getpid()}.tmp.npy"  # per process: ranks may generate the same tile at once
    np.save(tmp, rgb)
    os.replace(tmp, fn)
    return rgb


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3, choices=[3, 4])
    ap.add_argument("--tiles", type=int, default=None)
    ap.add_argument("--pool", type=int, default=16)
    ap.add_argument("--slots", type=int, default=2)
    args = ap.parse_args()
    n_tiles = args.tiles or (1000 if args.config == 3 else 36848)

    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1209_3332_b200.dist import bind_to_gpu_numa
    bind_to_gpu_numa(local)  # pinned pool and feeder thread on the GPU's NUMA node
    from paper_1209_3332_b200 import Context
    from paper_1209_3332_b200.dist import DistTileSource, TileQueue, aggregate_groups, gather_rows, table_digest, to_rows

    t0 = time.time()
    pool = [torch.from_numpy(pool_tile(args.config, k)).pin_memory() for k in range(args.pool)]
    gen_s = time.time() - t0
    ctx = Context(local, 4096, 4096, n_slots=args.slots, max_objects=16384)
    results = {}

    def done(tid, l, f, ft, st):
        if st != 0:
            raise RuntimeError(f"tile {tid}: status {st}")
        results[tid] = (l, f, ft)

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    q = TileQueue(n_tiles, block=args.slots)
    src = DistTileSource(q, lambda tid: pool[tid % args.pool])
    ctx.run_tiles(src, done, 4096, 4096)
    torch.cuda.synchronize()
    t_run = time.perf_counter() - t1
    table = gather_rows(results, device=torch.device("cuda", local))
    t_all = time.perf_counter() - t1
    # per-slide aggregation: device segmented sums per rank, NCCL all-reduce
    per_slide = 108 if args.config == 4 else n_tiles
    n_groups = (n_tiles + per_slide - 1) // per_slide
    ta = time.perf_counter()
    cnt, mean, std = aggregate_groups(to_rows(results), lambda t: t // per_slide, n_groups, reduce=ctx,
                                      device=torch.device("cuda", local))
    agg_ms = 1e3 * (time.perf_counter() - ta)
    tt = torch.tensor([t_all, t_run], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"config": args.config, "tiles": n_tiles, "n_gpus": world, "pool": args.pool,
                          "slots": args.slots, "tiles_per_s": n_tiles / float(tt[0]),
                          "tiles_per_s_excl_gather": n_tiles / float(tt[1]),
                          "rows": int(len(table)), "digest": table_digest(table),
                          "my_tiles_rank0": len(src.taken), "pool_gen_s": round(gen_s, 1),
                          "groups": n_groups, "group_rows": int(cnt.sum()), "agg_ms": round(agg_ms, 1),
                          "agg_checksum": float(np.nansum(mean) + np.nansum(std))}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    ctx.close()


if __name__ == "__main__":
    main()
