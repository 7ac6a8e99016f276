"""Run the full pipeline (segmentation + features) on one config-2 tile, REPS times, on
cuda:0 -- the target for ncu launch lists:  ncu --metrics gpu__time_duration.sum --csv
python tools/one_tile.py [REPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from paper_1209_3332_b200 import Context
    from synth.hne import make_config_tile
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    size, cap = 4096, 16384
    rgb = torch.from_numpy(np.ascontiguousarray(make_config_tile(2))).cuda()
    ctx = Context(0, size, size, n_slots=1, max_objects=cap)
    lab = torch.empty((size, size), dtype=torch.int32, device="cuda")
    nob = torch.zeros(1, dtype=torch.int32, device="cuda")
    tl = torch.empty(cap, dtype=torch.int32, device="cuda")
    tf = torch.empty(cap, dtype=torch.int32, device="cuda")
    tt = torch.empty((cap, 36), dtype=torch.float32, device="cuda")
    nr = torch.zeros(1, dtype=torch.int32, device="cuda")
    for _ in range(reps):
        ctx.process_tile(0, rgb, lab, nob, tl, tf, tt, nr)
    torch.cuda.synchronize()
    print("objects", int(nob.item()), "rows", int(nr.item()))
    ctx.close()


if __name__ == "__main__":
    main()
