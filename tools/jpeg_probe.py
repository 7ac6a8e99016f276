"""NEXT-3 probe: one config-2 tile as a quality-90 4:4:4 JPEG (restart interval 4 MCUs) on
cuda:0 -- CUDA-event times of hp_process_tile (raw RGB already on the device) vs
hp_process_tile_jpeg (JPEG bytes from pinned host memory, decode fused into S1), and the
decode alone (hp_decode_jpeg, RGB out).  Also the ncu target for the decode kernels.
usage: python tools/jpeg_probe.py [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from paper_1209_3332_b200 import Context
    from synth.hne import make_config_tile
    from synth.jpeg import encode_tile
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    size, cap = 4096, 16384
    rgb = make_config_tile(2)
    buf = torch.from_numpy(encode_tile(rgb, 90, 4)).pin_memory()
    ctx = Context(0, size, size, n_slots=1, max_objects=cap)
    dev = torch.from_numpy(np.ascontiguousarray(rgb)).cuda()
    lab = torch.empty((size, size), dtype=torch.int32, device="cuda")
    nob = torch.zeros(1, dtype=torch.int32, device="cuda")
    tl = torch.empty(cap, dtype=torch.int32, device="cuda")
    tf = torch.empty(cap, dtype=torch.int32, device="cuda")
    tt = torch.empty((cap, 36), dtype=torch.float32, device="cuda")
    nr = torch.zeros(1, dtype=torch.int32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = torch.empty((size, size, 3), dtype=torch.uint8, device="cuda")

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    res = {"jpeg_bytes": int(buf.numel()), "raw_bytes": int(rgb.nbytes)}
    res["process_tile_ms"] = timed(lambda: ctx.process_tile(0, dev, lab, nob, tl, tf, tt, nr))
    n_raw = int(nr.item())
    res["process_tile_jpeg_ms"] = timed(lambda: ctx.process_tile_jpeg(0, buf, lab, nob, tl, tf, tt, nr, decode_err=err))
    res["rows_equal"] = int(nr.item()) == n_raw
    res["decode_err"] = int(err.item())
    res["decode_jpeg_ms_incl_sync"] = timed(lambda: ctx.decode_jpeg(0, buf, out))
    # the same tile as 4:2:0 (decode to planes + upsampling / colour / S1 kernel)
    b420 = torch.from_numpy(encode_tile(rgb, 90, 4, sampling="420")).pin_memory()
    res["jpeg420_bytes"] = int(b420.numel())
    res["process_tile_jpeg420_ms"] = timed(lambda: ctx.process_tile_jpeg(0, b420, lab, nob, tl, tf, tt, nr,
                                                                        decode_err=err))
    res["decode_jpeg420_ms_incl_sync"] = timed(lambda: ctx.decode_jpeg(0, b420, out))
    # the same pipeline on the decoded RGB tile already on the device: the difference to
    # process_tile_jpeg is the ingest (copy + decode), the difference to process_tile is what
    # the JPEG loss does to the later steps
    ctx.decode_jpeg(0, buf, out)
    dec = out.clone()
    res["process_tile_on_decoded_ms"] = timed(lambda: ctx.process_tile(0, dec, lab, nob, tl, tf, tt, nr))
    # per-stage times (S1..S11 events) of the raw and the decoded tile, and their object counts
    names = ["S1", "S2", "S3", "S4", "S5", "S6", "S7", "S8-S11+Canny", "-", "-", "-"]
    for tag, t in (("raw", dev), ("decoded", dec)):
        ctx.set_stage_timing(True)
        per = []
        for _ in range(5):
            ctx.process_tile(0, t, lab, nob, tl, tf, tt, nr)
            torch.cuda.synchronize()
            per.append(ctx.stage_times(0))
        ctx.set_stage_timing(False)
        med = [sorted(p[i] for p in per)[2] for i in range(11)]
        res[f"stages_{tag}_ms"] = {names[i]: round(med[i], 4) for i in range(8)}
        res[f"objects_{tag}"] = int(nob.item())
    res["decoded_equals_raw_within"] = int((out.cpu().numpy().astype(int) - rgb).__abs__().max())
    print(json.dumps(res))
    ctx.close()


if __name__ == "__main__":
    main()
