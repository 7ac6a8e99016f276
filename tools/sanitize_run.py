"""Target for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): the whole
per-tile path (hp_process_tile) on BASELINE configs[0] (512x512) and on a 1024x1024 tile,
then hp_run_tiles with graphs over both tiles twice, and the IWPP stress stage on a small
serpentine.  Prints a digest of every output so a run under the tool can be compared with
a plain run.  usage: python tools/sanitize_run.py [size ...]"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def digest(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(a.tobytes())
    return h.hexdigest()[:16]


def main():
    import numpy as np
    import torch
    from paper_1209_3332_b200 import Context
    from synth.hne import TileSpec, make_tile
    from synth.stress import make_stress

    sizes = [int(a) for a in sys.argv[1:]] or [512, 1024]
    cap = 8192
    mx = max(sizes)
    tiles = [make_tile(1 + i, TileSpec(s, s))["rgb"] for i, s in enumerate(sizes)]
    with Context(0, mx, mx, n_slots=2, max_objects=cap) as ctx:
        for rgb in tiles:
            h, w = rgb.shape[:2]
            t = torch.from_numpy(rgb).cuda()
            lab = torch.zeros((h, w), dtype=torch.int32, device="cuda")
            nobj = torch.zeros(1, dtype=torch.int32, device="cuda")
            tl = torch.zeros(cap, dtype=torch.int32, device="cuda")
            tf = torch.zeros(cap, dtype=torch.int32, device="cuda")
            tt = torch.zeros((cap, 36), dtype=torch.float32, device="cuda")
            nr = torch.zeros(1, dtype=torch.int32, device="cuda")
            ctx.process_tile(0, t, lab, nobj, tl, tf, tt, nr)
            torch.cuda.synchronize()
            k = int(nr.item())
            print(f"process_tile {w}x{h}: {k} rows, digest "
                  f"{digest(lab.cpu().numpy(), tl[:k].cpu().numpy(), tt[:k].cpu().numpy())}", flush=True)
        # hp_run_tiles (graph capture on the second tile of a slot, replay after), one size
        s0 = sizes[0]
        pinned = [torch.from_numpy(make_tile(50 + i, TileSpec(s0, s0))["rgb"]).pin_memory() for i in range(2)]
        order = iter(range(6))
        res = {}

        def nxt():
            i = next(order, None)
            if i is None:
                return None
            t = pinned[i % 2]
            return t.data_ptr(), t.stride(0), i

        def done(tid, l, f, ft, st):
            res[tid] = (st, digest(l, f, ft))

        ctx.run_tiles(nxt, done, s0, s0)
        for tid in sorted(res):
            print(f"run_tiles tile {tid}: status {res[tid][0]} digest {res[tid][1]}", flush=True)
        assert res[0][1] == res[2][1] == res[4][1] and res[1][1] == res[3][1] == res[5][1]
        # IWPP stress (config 5 shape, small): serpentine corridor, binary mask
        marker, mask, _ = make_stress("serpentine", 256)
        mk = torch.from_numpy(marker).cuda()
        ms = torch.from_numpy(mask).cuda()
        out = torch.zeros_like(ms)
        ctx.stage_run(0, "IWPP_RAW", [mk, ms], [out], 256, 256)
        torch.cuda.synchronize()
        print("iwpp stress recon == mask:", bool((out == ms).all()), flush=True)
    print("sanitize_run done", flush=True)


if __name__ == "__main__":
    main()
