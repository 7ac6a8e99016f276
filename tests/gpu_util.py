"""Helpers for the -m gpu parity tests: run one libhp stage on numpy inputs through the
C ABI (hp_stage_run) and compare with the oracle under reading C18's tolerance."""
import numpy as np

TOL_REL, TOL_ABS = 1e-5, 1e-6   # DESIGN.md reading C18


def to_dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def empty(shape, dtype):
    import torch
    tdt = {np.uint8: torch.uint8, np.int32: torch.int32, np.float32: torch.float32,
           np.uint32: torch.int32, np.int64: torch.int64}[dtype]
    return torch.zeros(shape, dtype=tdt, device="cuda")


def stage(ctx, name, ins, outs, w, h, slot=0):
    """ins: numpy arrays (or None); outs: list of (shape, dtype) or None -> numpy results."""
    import torch
    din = [None if a is None else to_dev(a) for a in ins]
    dout = [None if o is None else empty(*o) for o in outs]
    ctx.stage_run(slot, name, din, dout, w, h)
    torch.cuda.synchronize()
    res = []
    for o, t in zip(outs, dout):
        if t is None:
            res.append(None)
            continue
        a = t.cpu().numpy()
        if o[1] == np.uint32:
            a = a.view(np.uint32)
        res.append(a)
    return res


def features_close(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    diff = np.abs(a - b)
    ok = (diff <= TOL_REL * np.maximum(np.abs(a), np.abs(b))) | (diff <= TOL_ABS)
    ok |= (a == b)  # also covers inf == inf
    return ok


def assert_features_equal(gl, gf, gt, ol, of, ot):
    assert np.array_equal(gl, ol), "row labels differ"
    assert np.array_equal(gf, of), "row flags differ"
    ok = features_close(gt, ot)
    if not ok.all():
        bad = np.argwhere(~ok)
        r, c = bad[0]
        raise AssertionError(f"{len(bad)} feature values out of tolerance; first row {r} col {c}: "
                             f"gpu {gt[r, c]!r} oracle {ot[r, c]!r}")
