"""GPU parity of the compressed-ingest path through the C
ABI: the device JPEG decoder (hp_decode_jpeg) bit-exact against the oracle's T.81 decoder
(itself pinned to cv2.imdecode), and the decoder fused into S1 (hp_process_tile_jpeg,
hp_run_tiles_jpeg) against the oracle's pipeline on the oracle's decoded tile -- labels
bit-exact, features within reading C18.  Corrupt and out-of-scope files are rejected."""
import numpy as np
import pytest

import oracle
from synth.hne import TileSpec, make_config_tile, make_tile
from synth.jpeg import encode_tile
from tests.gpu_util import assert_features_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1209_3332_b200 import Context
    c = Context(0, 4096, 4096, n_slots=4, max_objects=65536)
    yield c
    c.close()


def _decode(ctx, buf, h, w):
    import torch
    out = torch.full((h, w, 3), 7, dtype=torch.uint8, device="cuda")
    ctx.decode_jpeg(0, buf, out)
    return out.cpu().numpy()


@pytest.mark.parametrize("shape,q,rst", [((64, 64), 90, 4), ((37, 53), 75, 1), ((300, 257), 95, 0),
                                         ((512, 512), 90, 4), ((129, 200), 50, 17), ((8, 8), 100, 1),
                                         ((1, 300), 90, 2), ((301, 1), 85, 3), ((1000, 1016), 90, 64)])
def test_decode_tiles(ctx, shape, q, rst):
    rgb = make_tile(sum(shape) + q, TileSpec(*shape))["rgb"]
    buf = encode_tile(rgb, q, rst)
    assert np.array_equal(_decode(ctx, buf, *shape), oracle.jpeg_decode(buf))


@pytest.mark.parametrize("shape,q,rst", [((64, 64), 90, 4), ((37, 53), 75, 1), ((300, 257), 95, 0),
                                         ((512, 512), 90, 4), ((1, 300), 90, 2), ((301, 1), 85, 3),
                                         ((2, 2), 90, 1), ((9, 3), 90, 1), ((7, 4), 90, 2), ((5, 5), 90, 1),
                                         ((17, 33), 60, 2), ((2, 300), 90, 1), ((1000, 1016), 90, 16)])
def test_decode_tiles_420(ctx, shape, q, rst):
    """4:2:0: the decode kernel writes component planes, the upsampling kernel applies reading
    J4's triangle filter (replication for chroma <= 2 samples wide) -- bit-exact with the oracle."""
    rgb = make_tile(sum(shape) + q + 7, TileSpec(*shape))["rgb"]
    buf = encode_tile(rgb, q, rst, sampling="420")
    assert np.array_equal(_decode(ctx, buf, *shape), oracle.jpeg_decode(buf))


@pytest.mark.parametrize("kind", ["noise", "checker", "flat"])
@pytest.mark.parametrize("q", [60, 100])
def test_decode_hard_images(ctx, kind, q):
    rng = np.random.default_rng(11)
    h, w = 96, 136
    if kind == "noise":
        rgb = rng.integers(0, 256, (h, w, 3)).astype(np.uint8)
    elif kind == "checker":
        yy, xx = np.indices((h, w))
        rgb = np.repeat(((yy + xx) % 2 * 255).astype(np.uint8)[:, :, None], 3, axis=2)
        rgb[:, :, 1] = 255 - rgb[:, :, 1]
    else:
        rgb = np.full((h, w, 3), (200, 30, 90), np.uint8)
    buf = encode_tile(rgb, q, 5)
    assert np.array_equal(_decode(ctx, buf, h, w), oracle.jpeg_decode(buf))


def _tables(cap):
    import torch
    return (torch.zeros(cap, dtype=torch.int32, device="cuda"), torch.zeros(cap, dtype=torch.int32, device="cuda"),
            torch.zeros((cap, 36), dtype=torch.float32, device="cuda"), torch.zeros(1, dtype=torch.int32, device="cuda"))


def _check_tile_jpeg(ctx, rgb, q=90, rst=4, sampling="444"):
    import torch
    buf = encode_tile(rgb, q, rst, sampling=sampling)
    dec = oracle.jpeg_decode(buf)
    h, w = rgb.shape[:2]
    cap = 65536
    lab = torch.zeros((h, w), dtype=torch.int32, device="cuda")
    nob = torch.zeros(1, dtype=torch.int32, device="cuda")
    err = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    tl, tf, tt, nr = _tables(cap)
    ctx.process_tile_jpeg(1, buf, lab, nob, tl, tf, tt, nr, decode_err=err)
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    olab, ol, of, ot = oracle.process_tile(dec)
    assert np.array_equal(lab.cpu().numpy(), olab)
    n = int(nr.item())
    assert n == len(ol)
    assert_features_equal(tl[:n].cpu().numpy(), tf[:n].cpu().numpy(), tt[:n].cpu().numpy(), ol, of, ot)
    return n


def test_process_tile_jpeg_config1(ctx):
    assert _check_tile_jpeg(ctx, make_config_tile(1)) > 10


@pytest.mark.parametrize("seed,shape,rst", [(41, (300, 404), 3), (42, (257, 129), 0), (43, (512, 384), 1)])
def test_process_tile_jpeg_ragged(ctx, seed, shape, rst):
    _check_tile_jpeg(ctx, make_tile(seed, TileSpec(*shape))["rgb"], 85, rst)


@pytest.mark.parametrize("seed,shape,rst", [(44, (300, 404), 2), (45, (257, 129), 0)])
def test_process_tile_jpeg_420(ctx, seed, shape, rst):
    _check_tile_jpeg(ctx, make_tile(seed, TileSpec(*shape))["rgb"], 85, rst, sampling="420")


@pytest.mark.slow
def test_process_tile_jpeg_config2_420(ctx):
    assert _check_tile_jpeg(ctx, make_config_tile(2), sampling="420") > 1000


@pytest.mark.slow
def test_process_tile_jpeg_config2(ctx):
    assert _check_tile_jpeg(ctx, make_config_tile(2)) > 1000


def _corrupt_rst(buf):
    b = buf.copy()
    i = next(k for k in range(len(b) - 1) if b[k] == 0xFF and 0xD0 <= b[k + 1] <= 0xD7)
    b[i:i + 2] = 0   # one restart marker fewer than the restart interval says
    return b


def _corrupt_codes(buf):
    b = buf.copy()
    sos = next(k for k in range(len(b) - 1) if b[k] == 0xFF and b[k + 1] == 0xDA)
    start = sos + 2 + (int(b[sos + 2]) << 8 | int(b[sos + 3]))
    b[start:start + 64:2] = 0xFF    # runs of 1-bits (stuffed 0xFF 0x00): no valid code is all ones
    b[start + 1:start + 64:2] = 0x00
    return b


def test_corrupt_and_unsupported_files(ctx):
    from paper_1209_3332_b200.hp import HPError
    rgb = make_tile(50, TileSpec(128, 128))["rgb"]
    buf = encode_tile(rgb, 90, 2)
    with pytest.raises(HPError) as e:
        _decode(ctx, _corrupt_rst(buf), 128, 128)
    assert e.value.status == 1
    with pytest.raises(HPError) as e:
        _decode(ctx, _corrupt_codes(buf), 128, 128)
    assert e.value.status == 1
    with pytest.raises(HPError) as e:
        _decode(ctx, encode_tile(rgb, 90, 2, sampling="422"), 128, 128)
    assert e.value.status == 5
    with pytest.raises(HPError) as e:
        _decode(ctx, encode_tile(rgb, 90, 0, progressive=True), 128, 128)
    assert e.value.status == 5
    with pytest.raises(HPError) as e:
        _decode(ctx, buf[:100], 128, 128)
    assert e.value.status == 1
    # the context is still usable afterwards
    assert np.array_equal(_decode(ctx, buf, 128, 128), oracle.jpeg_decode(buf))


def test_run_tiles_jpeg(ctx):
    """hp_run_tiles_jpeg with per-slot graphs: 10 files over 4 slots (each slot captures and
    replays), 4:4:4 and 4:2:0 files mixed (a slot rebuilds its graph when the sampling
    changes), two of them bad -- the bad ones come back with a nonzero status and no rows,
    every other table equals the oracle's on the decoded tile."""
    import torch
    h, w = 256, 384
    tiles = [make_tile(900 + i, TileSpec(h, w))["rgb"] for i in range(4)]
    bufs = [torch.from_numpy(encode_tile(t, 90, 4, sampling="420" if i == 2 else "444")).pin_memory()
            for i, t in enumerate(tiles)]
    bad = {3: torch.from_numpy(_corrupt_rst(bufs[1].numpy())).pin_memory(),
           7: torch.from_numpy(encode_tile(tiles[2], 90, 4, sampling="422")).pin_memory()}
    ref = [oracle.process_tile(oracle.jpeg_decode(b.numpy()))[1:] for b in bufs]
    order = iter(range(10))
    got = {}

    def nxt():
        i = next(order, None)
        if i is None:
            return None
        b = bad.get(i, bufs[i % 4])
        return b.data_ptr(), b.numel(), i

    def done(tid, l, f, ft, st):
        got[tid] = (st, l, f, ft)

    ctx.run_tiles_jpeg(nxt, done, w, h)
    assert sorted(got) == list(range(10))
    assert got[3][0] == 1 and got[7][0] == 5 and len(got[3][1]) == len(got[7][1]) == 0
    for tid, (st, l, f, ft) in got.items():
        if tid in bad:
            continue
        assert st == 0
        ol, of, ot = ref[tid % 4]
        assert_features_equal(l, f, ft, ol, of, ot)


def _oracle_jpeg_rows(buf):
    return oracle.process_tile(oracle.jpeg_decode(buf))[1:]


@pytest.mark.slow
@pytest.mark.parametrize("sampling", ["444", "420"])
def test_bench_jpeg_e2e_launch_config(sampling):
    """bench.py's e2e.jpeg leg in its exact configuration at full size: the bench's 12 4K tiles
    as quality-90 JPEG files (restart interval 4), hp_run_tiles_jpeg on 24 slots with per-slot
    graphs, 32 hardware queues, the files twice each from a demand-driven queue -- every
    delivered table equals the oracle's on the oracle's decode of the same file."""
    import multiprocessing as mp
    import os

    import torch
    from paper_1209_3332_b200 import Context
    from paper_1209_3332_b200.dist import DistTileSource, TileQueue
    from tests.test_gpu_parity import BENCH_BATCH, BENCH_E2E_SLOTS, BENCH_SLOTS, _pool_tile
    K = BENCH_BATCH
    with mp.get_context("fork").Pool(max(1, min(K, os.cpu_count() or 1))) as pool:
        tiles = pool.map(_pool_tile, range(1000, 1000 + K))
        bufs = [encode_tile(t, 90, 4, sampling=sampling) for t in tiles]
        ref = pool.map(_oracle_jpeg_rows, bufs)
    c = Context(0, 4096, 4096, n_slots=max(BENCH_SLOTS, BENCH_E2E_SLOTS), max_objects=8192)
    try:
        pinned = [torch.from_numpy(b).pin_memory() for b in bufs]
        q = TileQueue(2 * K, block=BENCH_SLOTS, store=None)
        ids = iter(())
        got = {}

        def nxt():
            nonlocal ids
            while True:
                tid = next(ids, None)
                if tid is not None:
                    b = pinned[tid % K]
                    return b.data_ptr(), b.numel(), tid
                blk = q.grab()
                if blk is None:
                    return None
                ids = iter(blk)

        def done(tid, l, f, ft, st):
            assert st == 0, f"tile {tid} status {st}"
            got[tid] = (l, f, ft)

        c.run_tiles_jpeg(nxt, done, 4096, 4096)
        assert sorted(got) == list(range(2 * K))
        for tid, (l, f, ft) in got.items():
            assert_features_equal(l, f, ft, *ref[tid % K])
    finally:
        c.close()
