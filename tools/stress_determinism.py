"""Determinism / race stress: the bench's tiles processed REPS times each with S slots in
flight (as in bench.py); every run's labels + feature table must be bit-identical to the first
run of that tile.  With "jpeg" the tiles are first passed through a quality-90 JPEG round trip
(smoother images: longer S4 propagation, more regions on the alternating-phase closure).
usage: python tools/stress_determinism.py [REPS] [SLOTS] [jpeg]"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from paper_1209_3332_b200 import Context
    from synth.hne import TileSpec, make_tile
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    S = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    tiles = [make_tile(1000 + i, TileSpec())["rgb"] for i in range(12)]
    if len(sys.argv) > 3 and sys.argv[3] == "jpeg":
        import cv2
        from synth.jpeg import encode_tile
        tiles = [np.ascontiguousarray(cv2.imdecode(encode_tile(t), cv2.IMREAD_COLOR)[:, :, ::-1]) for t in tiles]
    dev = [torch.from_numpy(t).cuda() for t in tiles]
    size, cap = 4096, 16384
    ctx = Context(0, size, size, n_slots=S, max_objects=cap)
    lab = [torch.empty((size, size), dtype=torch.int32, device="cuda") for _ in range(S)]
    nob = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(S)]
    tl = [torch.empty(cap, dtype=torch.int32, device="cuda") for _ in range(S)]
    tf = [torch.empty(cap, dtype=torch.int32, device="cuda") for _ in range(S)]
    tt = [torch.empty((cap, 36), dtype=torch.float32, device="cuda") for _ in range(S)]
    nr = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(S)]
    streams = [torch.cuda.Stream() for _ in range(S)]
    ref, bad, runs = {}, 0, 0
    for r in range(reps):
        for i0 in range(0, len(tiles), S):
            batch = list(range(i0, min(i0 + S, len(tiles))))
            for k, i in enumerate(batch):
                ctx.process_tile(k, dev[i], lab[k], nob[k], tl[k], tf[k], tt[k], nr[k], stream=streams[k])
            torch.cuda.synchronize()
            for k, i in enumerate(batch):
                n = int(nr[k].item())
                h = hashlib.sha256()
                for t in (lab[k], nob[k], tl[k][:n], tf[k][:n], tt[k][:n]):
                    h.update(t.cpu().numpy().tobytes())
                d = h.hexdigest()
                runs += 1
                if i not in ref:
                    ref[i] = d
                elif ref[i] != d:
                    bad += 1
                    print(f"MISMATCH tile {i} rep {r}", flush=True)
    print(json.dumps({"runs": runs, "mismatches": bad, "tiles": len(tiles), "slots": S,
                      "input": sys.argv[3] if len(sys.argv) > 3 else "raw"}), flush=True)
    ctx.close()
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
