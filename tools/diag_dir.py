"""Direction sensitivity of the u8 IWPP: reconstruct recon(open(g), g) of a config-2 tile as
is, transposed and flipped, printing time and region jobs (tools/diag_iwpp.py conventions)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1209_3332_b200 import Context
    from synth.hne import make_config_tile
    from tools.diag_iwpp import timed
    size = 4096
    ctx = Context(0, size, size, n_slots=1, max_objects=8192)
    rgb = torch.from_numpy(make_config_tile(2)).cuda()
    g = torch.empty((size, size), dtype=torch.uint8, device="cuda")
    fl = torch.empty_like(g)
    nbg = torch.zeros(1, dtype=torch.int64, device="cuda")
    ctx.stage_run(0, "CD", [rgb], [g, fl, nbg], size, size)
    op = torch.empty_like(g)
    ctx.stage_run(0, "OPEN", [g], [op], size, size)
    ref = None
    for name, f in [("identity", lambda t: t), ("transpose", lambda t: t.t()), ("flip_y", lambda t: t.flip(0)),
                    ("flip_x", lambda t: t.flip(1))]:
        m, r0 = f(g).contiguous(), f(op).contiguous()
        rec = torch.empty_like(g)
        st = torch.zeros(4, dtype=torch.int64, device="cuda")
        ms = timed(lambda: ctx.stage_run(0, "IWPP_RAW", [r0, m], [rec, st], size, size))
        out = f(rec) if name != "transpose" else rec.t()
        if ref is None:
            ref = out.clone()
        print(json.dumps({"case": name, "ms": round(ms, 3), "jobs": int(st[0]), "row_closures": int(st[3]),
                          "same": bool(torch.equal(out, ref)),
                          "changed_px": int((rec != r0).sum())}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
