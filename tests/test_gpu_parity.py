"""GPU parity: every libhp stage (called through the C ABI) against the oracle, fed the
oracle's own inputs, bit-exact on integer outputs and within reading C18's tolerance on
float features; then the whole pipeline end to end, the IWPP stress inputs and the
multi-tile driver.  Needs a B200 (-m gpu)."""
import numpy as np
import pytest

import oracle
from synth import make_stress
from synth.hne import TileSpec, make_config_tile, make_tile
from tests.gpu_util import assert_features_equal, features_close, stage

pytestmark = pytest.mark.gpu

U8, I32, F32, U32, I64 = np.uint8, np.int32, np.float32, np.uint32, np.int64


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1209_3332_b200 import Context
    c = Context(0, 4096, 4096, n_slots=2, max_objects=65536)
    yield c
    c.close()


def _oracle_chain(rgb):
    """The oracle's intermediates of every step of one tile."""
    p = oracle.default_params()
    d = {"rgb": rgb}
    d["g"], d["flags"], d["nbg"] = oracle.cd(rgb, p)
    d["rbc"] = oracle.rbc(d["flags"])
    d["open"] = oracle.open_(d["g"], 19)
    d["cand"], d["recon"] = oracle.recon_to_nuclei(d["g"], d["open"], d["rbc"], 50, with_recon=True)
    d["big0"] = oracle.area_threshold(d["cand"], 11, 1000)
    d["F"] = oracle.fill_holes(d["big0"])
    d["d2"], d["dist"] = oracle.edt(d["F"])
    d["ML"], d["J"], _ = oracle.markers(d["dist"], d["F"], 1.0)
    d["split"], d["c"], d["d"], d["L"] = oracle.watershed(d["dist"], d["ML"], d["F"])
    d["labels"], d["nobj"] = oracle.bwlabel(d["split"], 21, 1000)
    d["rows"] = oracle.features(d["labels"], d["g"])
    return d


@pytest.fixture(scope="module")
def chain():
    """Oracle intermediates of the config-1 tile."""
    return _oracle_chain(make_config_tile(1))


def test_cd(ctx, chain):
    h, w = chain["g"].shape
    g, fl, nbg = stage(ctx, "CD", [chain["rgb"]], [((h, w), U8), ((h, w), U8), ((1,), I64)], w, h)
    assert np.array_equal(g, chain["g"]) and np.array_equal(fl, chain["flags"])
    assert int(nbg[0]) == chain["nbg"]


def test_rbc(ctx, chain):
    h, w = chain["g"].shape
    (r,) = stage(ctx, "RBC", [chain["flags"]], [((h, w), U8)], w, h)
    assert np.array_equal(r, chain["rbc"]) and r.sum() > 0


def test_open(ctx, chain):
    h, w = chain["g"].shape
    (o,) = stage(ctx, "OPEN", [chain["g"]], [((h, w), U8)], w, h)
    assert np.array_equal(o, chain["open"])


def test_recon(ctx, chain):
    h, w = chain["g"].shape
    cand, rec = stage(ctx, "RECON", [chain["g"], chain["open"], chain["rbc"]],
                      [((h, w), U8), ((h, w), U8)], w, h)
    assert np.array_equal(rec, chain["recon"])
    assert np.array_equal(cand, chain["cand"])


@pytest.mark.parametrize("kind", ["uniform", "blobs", "ramp"])
def test_recon_cand_random_planes(ctx, kind):
    # S4 on planes unlike the tiles (uniform noise, bright blobs, ramps with noise); check it against
    # the oracle's plain recon + threshold
    rng = np.random.default_rng({"uniform": 1, "blobs": 2, "ramp": 3}[kind])
    h, w = 300, 400
    if kind == "uniform":
        g = rng.integers(0, 256, size=(h, w)).astype(U8)
    elif kind == "blobs":
        g = (10 + rng.integers(0, 6, size=(h, w))).astype(np.int32)
        yy, xx = np.mgrid[:h, :w]
        for _ in range(40):
            cy, cx, r, v = rng.uniform(0, h), rng.uniform(0, w), rng.uniform(3, 9), rng.integers(60, 250)
            g = np.where((yy - cy) ** 2 + (xx - cx) ** 2 <= r * r, v, g)
        g = g.astype(U8)
    else:
        g = ((np.add.outer(np.arange(h), np.arange(w)) % 256) ^ rng.integers(0, 64, size=(h, w))).astype(U8)
    op = oracle.open_(g, 19)
    rbc = (rng.random((h, w)) < 0.01).astype(U8)
    cand, rec = stage(ctx, "RECON", [g, op, rbc], [((h, w), U8), ((h, w), U8)], w, h)
    ecand, erec = oracle.recon_to_nuclei(g, op, rbc, 50, with_recon=True)
    assert np.array_equal(rec, erec)
    assert np.array_equal(cand, ecand)


def test_area_fill(ctx, chain):
    h, w = chain["g"].shape
    (b,) = stage(ctx, "AREA", [chain["cand"]], [((h, w), U8)], w, h)
    assert np.array_equal(b, chain["big0"])
    (F,) = stage(ctx, "FILL", [chain["big0"]], [((h, w), U8)], w, h)
    assert np.array_equal(F, chain["F"])


def _check_hot_path_stages(ctx, d, cap=65536):
    """The pipeline's own S5 (CCL-select on the top-hat), S6 (per-component fill) and S7-S11
    (per-component EDT .. features) kernels, each fed the oracle's input of that step:
    integer outputs bit-exact, features within reading C18 (north_star: "bit-exact for every
    integer/labeling stage when each stage is fed the oracle's own input")."""
    h, w = d["g"].shape
    big0, nk = stage(ctx, "AREA_TOPHAT", [d["g"], d["recon"], d["rbc"]], [((h, w), U8), ((1,), I32)], w, h)
    assert np.array_equal(big0, d["big0"])
    assert int(nk[0]) == oracle.ccl(d["big0"], 8)[1]
    (F,) = stage(ctx, "FILL_COMP", [d["big0"]], [((h, w), U8)], w, h)
    assert np.array_equal(F, d["F"])
    lab, nob, lf, ft = stage(ctx, "COMPONENTS", [d["F"], d["g"]],
                             [((h, w), I32), ((1,), I32), ((2, cap), I32), ((cap, 36), F32)], w, h)
    assert np.array_equal(lab, d["labels"])
    n = int(nob[0])
    assert n == d["nobj"]
    ol, of, ot = d["rows"]
    assert_features_equal(lf[0, :n], lf[1, :n], ft[:n], ol, of, ot)


def test_hot_path_stages_config1(ctx, chain):
    _check_hot_path_stages(ctx, chain)


@pytest.mark.parametrize("seed,shape", [(31, (300, 400)), (32, (257, 129)), (33, (512, 384))])
def test_hot_path_stages_random(ctx, seed, shape):
    _check_hot_path_stages(ctx, _oracle_chain(make_tile(seed, TileSpec(*shape))["rgb"]))


@pytest.mark.slow
def test_hot_path_stages_config2(ctx):
    _check_hot_path_stages(ctx, _oracle_chain(make_config_tile(2)))


@pytest.mark.parametrize("shape", [(20, 30), (64, 64), (1, 40)])
def test_components_all_foreground(ctx, shape):
    """F covering the whole tile: no background anywhere, so the EDT is +inf on every pixel
    (reading C11) -- the fused kernel's "component = whole tile" branch.  (20, 30): one object
    of 600 px; (64, 64): 4096 px, above obj_max_area, so no object (global-memory window)."""
    h, w = shape
    rng = np.random.default_rng(h * 1000 + w)
    F = np.ones((h, w), U8)
    g = rng.integers(0, 256, size=(h, w)).astype(U8)
    d2, dist = oracle.edt(F)
    assert np.isinf(dist).all()
    ML, _, _ = oracle.markers(dist, F, 1.0)
    split, _, _, _ = oracle.watershed(dist, ML, F)
    labels, nobj = oracle.bwlabel(split, 21, 1000)
    cap = 65536   # hp_stage_run's table capacity is the context's max_objects (hp.h)
    lab, nob, lf, ft = stage(ctx, "COMPONENTS", [F, g], [((h, w), I32), ((1,), I32), ((2, cap), I32),
                                                        ((cap, 36), F32)], w, h)
    assert np.array_equal(lab, labels) and int(nob[0]) == nobj == (1 if h * w <= 1000 and h * w >= 21 else 0)
    if nobj:
        ol, of, ot = oracle.features(labels, g)
        assert_features_equal(lf[0, :1], lf[1, :1], ft[:1], ol, of, ot)


def test_edt(ctx, chain):
    h, w = chain["g"].shape
    d2, dist = stage(ctx, "EDT", [chain["F"]], [((h, w), U32), ((h, w), F32)], w, h)
    assert np.array_equal(d2, chain["d2"])
    assert np.array_equal(dist, chain["dist"])


def test_markers_watershed(ctx, chain):
    h, w = chain["g"].shape
    ML, J = stage(ctx, "MARKERS", [chain["dist"], chain["F"]], [((h, w), I32), ((h, w), F32)], w, h)
    assert np.array_equal(J, chain["J"])
    assert np.array_equal(ML, chain["ML"])
    split, c, d, L = stage(ctx, "WATERSHED", [chain["dist"], chain["ML"], chain["F"]],
                           [((h, w), U8), ((h, w), F32), ((h, w), I32), ((h, w), I32)], w, h)
    assert np.array_equal(c, chain["c"])
    assert np.array_equal(d, chain["d"])
    assert np.array_equal(L, chain["L"])
    assert np.array_equal(split, chain["split"])


def test_bwlabel_features(ctx, chain):
    h, w = chain["g"].shape
    lab, n = stage(ctx, "BWLABEL", [chain["split"]], [((h, w), I32), ((1,), I32)], w, h)
    assert np.array_equal(lab, chain["labels"]) and int(n[0]) == chain["nobj"]
    cap = 65536
    rl, rf, ft, nr = stage(ctx, "FEATURES", [chain["labels"], chain["g"]],
                           [((cap,), I32), ((cap,), I32), ((cap, 36), F32), ((1,), I32)], w, h)
    k = int(nr[0])
    ol, of, ot = chain["rows"]
    assert k == len(ol)
    assert_features_equal(rl[:k], rf[:k], ft[:k], ol, of, ot)


SHAPES = [(1, 1), (1, 77), (77, 1), (33, 65), (100, 257), (257, 100), (64, 64)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("dens", [0.0, 0.3, 0.6, 1.0])
def test_ccl_random(ctx, shape, dens):
    h, w = shape
    fg = (np.random.default_rng(h * 1000 + w + int(dens * 10)).random(shape) < dens).astype(U8)
    for conn, name in [(8, "CCL8"), (4, "CCL4")]:
        (lab,) = stage(ctx, name, [fg], [((h, w), I32)], w, h)
        exp, _ = oracle.ccl(fg, conn)
        assert np.array_equal(lab, exp), (name, shape, dens)


@pytest.mark.parametrize("shape,dens", [((100, 257), 0.6), ((300, 333), 0.55), ((512, 512), 0.6)])
def test_ccl_repeated_no_races(ctx, shape, dens):
    # union-find with concurrent hooking: repeat to expose schedule-dependent losses
    # (a shared-memory path compression lost unions in ~5% of runs before it was removed)
    h, w = shape
    fg = (np.random.default_rng(h * 1000 + w + int(dens * 10)).random(shape) < dens).astype(U8)
    for conn, name in [(4, "CCL4"), (8, "CCL8")]:
        exp, _ = oracle.ccl(fg, conn)
        for rep in range(25):
            (lab,) = stage(ctx, name, [fg], [((h, w), I32)], w, h)
            if not np.array_equal(lab, exp):
                d = np.argwhere(lab != exp)
                raise AssertionError(f"{name} {shape} rep {rep}: {len(d)} px differ, e.g. "
                                     f"{[(int(y), int(x), int(lab[y, x]), int(exp[y, x])) for y, x in d[:6]]}")


@pytest.mark.parametrize("shape", SHAPES)
def test_open_ragged(ctx, shape):
    h, w = shape
    g = np.random.default_rng(w * 7 + h).integers(0, 256, size=shape).astype(U8)
    (o,) = stage(ctx, "OPEN", [g], [((h, w), U8)], w, h)
    assert np.array_equal(o, oracle.open_(g, 19))


@pytest.mark.parametrize("shape", SHAPES + [(300, 333)])
@pytest.mark.parametrize("levels", [2, 256])
def test_iwpp_random(ctx, shape, levels):
    h, w = shape
    rng = np.random.default_rng(h * 31 + w + levels)
    mask = (rng.integers(0, levels, size=shape) * (255 // (levels - 1))).astype(U8)
    marker = rng.integers(0, 256, size=shape).astype(U8)
    marker[rng.random(shape) < 0.8] = 0
    rec, _ = stage(ctx, "IWPP_RAW", [marker, mask], [((h, w), U8), ((4,), I64)], w, h)
    assert np.array_equal(rec, oracle.recon_u8(marker, mask))


@pytest.mark.parametrize("shape", [(37, 53), (130, 70), (256, 256)])
def test_recon_f32_domain(ctx, shape):
    h, w = shape
    rng = np.random.default_rng(h + w)
    dom = (rng.random(shape) < 0.75).astype(U8)
    mask = (rng.integers(0, 20, size=shape) * 0.25).astype(F32)
    marker = np.where(rng.random(shape) < 0.05, mask, -np.inf).astype(F32)
    (rec,) = stage(ctx, "RECON_F32", [marker, mask, dom], [((h, w), F32)], w, h)
    exp = oracle.recon_f32(marker, mask, dom)
    assert np.array_equal(rec[dom == 1], exp[dom == 1])


@pytest.mark.parametrize("shape", SHAPES + [(512, 300)])
@pytest.mark.parametrize("dens", [0.5, 0.9, 1.0])
def test_edt_random(ctx, shape, dens):
    h, w = shape
    F = (np.random.default_rng(h + 3 * w).random(shape) < dens).astype(U8)
    d2, dist = stage(ctx, "EDT", [F], [((h, w), U32), ((h, w), F32)], w, h)
    e2, ed = oracle.edt(F)
    assert np.array_equal(dist, ed)
    if (F == 0).any():
        assert np.array_equal(d2, e2)


# (300, 512) and (96, 1024): 16-B-aligned rows, so interior tiles stage g by bulk async copies
# (k_canny_nms) while edge tiles keep the per-word loop
@pytest.mark.parametrize("shape,blur", [((37, 53), False), ((70, 300), True), ((129, 97), True), ((8, 8), False),
                                        ((300, 512), True), ((96, 1024), False)])
def test_canny_random(ctx, shape, blur):
    import cv2
    h, w = shape
    g = np.random.default_rng(h * 7 + w).integers(0, 256, size=shape).astype(U8)
    if blur:
        g = cv2.GaussianBlur(g, (5, 5), 1.5)
    (e,) = stage(ctx, "CANNY", [g], [((h, w), U8)], w, h)
    assert np.array_equal(e, oracle.canny(g))


def test_canny_chain(ctx, chain):
    h, w = chain["g"].shape
    (e,) = stage(ctx, "CANNY", [chain["g"]], [((h, w), U8)], w, h)
    ref = oracle.canny(chain["g"])
    assert ref.sum() > 100 and np.array_equal(e, ref)


def test_edt_far_background(ctx):
    # one background column far from most pixels: exercises the Meijster fallback rows
    h, w = 64, 1500
    F = np.ones((h, w), U8)
    F[:, 3] = 0
    d2, dist = stage(ctx, "EDT", [F], [((h, w), U32), ((h, w), F32)], w, h)
    e2, ed = oracle.edt(F)
    assert np.array_equal(d2, e2) and np.array_equal(dist, ed)


def _gpu_process(ctx, rgb, slot=0, cap=65536):
    import torch
    h, w = rgb.shape[:2]
    t = torch.from_numpy(np.ascontiguousarray(rgb)).cuda()
    lab = torch.zeros((h, w), dtype=torch.int32, device="cuda")
    nobj = torch.zeros(1, dtype=torch.int32, device="cuda")
    tl = torch.zeros(cap, dtype=torch.int32, device="cuda")
    tf = torch.zeros(cap, dtype=torch.int32, device="cuda")
    tt = torch.zeros((cap, 36), dtype=torch.float32, device="cuda")
    nr = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.process_tile(slot, t, lab, nobj, tl, tf, tt, nr)
    torch.cuda.synchronize()
    k = int(nr.item())
    return (lab.cpu().numpy(), int(nobj.item()), tl[:k].cpu().numpy(), tf[:k].cpu().numpy(),
            tt[:k].cpu().numpy())


def _check_pipeline(ctx, rgb):
    lab, nobj, gl, gf, gt = _gpu_process(ctx, rgb)
    olab, ol, of, ot = oracle.process_tile(rgb)
    agree = (lab == olab).mean()
    assert np.array_equal(lab, olab), f"pixel agreement {agree:.6f}"
    assert nobj == len(ol)
    assert_features_equal(gl, gf, gt, ol, of, ot)
    return nobj


@pytest.mark.parametrize("seed", [21, 22])
def test_segment_then_features(ctx, seed):
    """The two-call ABI path: hp_segment_tile (S1-S10, no features), then hp_features_tile
    on its labels (S1 again, Canny, S11 from the label plane) -- equal to the oracle, and to
    hp_process_tile's fused rows."""
    import torch
    rgb = make_tile(seed, TileSpec(384, 448))["rgb"]
    h, w = rgb.shape[:2]
    t = torch.from_numpy(np.ascontiguousarray(rgb)).cuda()
    lab = torch.zeros((h, w), dtype=torch.int32, device="cuda")
    nobj = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.segment_tile(1, t, lab, nobj)
    cap = 4096
    tl = torch.zeros(cap, dtype=torch.int32, device="cuda")
    tf = torch.zeros(cap, dtype=torch.int32, device="cuda")
    tt = torch.zeros((cap, 36), dtype=torch.float32, device="cuda")
    nr = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.features_tile(1, t, lab, nobj, tl, tf, tt, nr)
    torch.cuda.synchronize()
    olab, ol, of, ot = oracle.process_tile(rgb)
    assert np.array_equal(lab.cpu().numpy(), olab) and int(nobj.item()) == len(ol)
    k = int(nr.item())
    gl, gf, gt = tl[:k].cpu().numpy(), tf[:k].cpu().numpy(), tt[:k].cpu().numpy()
    assert_features_equal(gl, gf, gt, ol, of, ot)
    _, _, fl, ff, ft = _gpu_process(ctx, rgb)
    assert np.array_equal(fl, gl) and np.array_equal(ff, gf)
    assert features_close(ft, gt).all()


def test_two_devices_one_process():
    """Contexts on two GPUs in one process: per-device kernel attributes and grid sizes."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    from paper_1209_3332_b200 import Context
    rgb = make_tile(31, TileSpec(320, 384))["rgb"]
    olab, ol, of, ot = oracle.process_tile(rgb)
    for dev in (1, 0):
        with torch.cuda.device(dev):
            c = Context(dev, 1024, 1024, n_slots=1, max_objects=4096)
            h, w = rgb.shape[:2]
            t = torch.from_numpy(np.ascontiguousarray(rgb)).cuda(dev)
            lab = torch.zeros((h, w), dtype=torch.int32, device=f"cuda:{dev}")
            nobj = torch.zeros(1, dtype=torch.int32, device=f"cuda:{dev}")
            tl = torch.zeros(4096, dtype=torch.int32, device=f"cuda:{dev}")
            tf = torch.zeros(4096, dtype=torch.int32, device=f"cuda:{dev}")
            tt = torch.zeros((4096, 36), dtype=torch.float32, device=f"cuda:{dev}")
            nr = torch.zeros(1, dtype=torch.int32, device=f"cuda:{dev}")
            c.process_tile(0, t, lab, nobj, tl, tf, tt, nr)
            torch.cuda.synchronize(dev)
            k = int(nr.item())
            assert np.array_equal(lab.cpu().numpy(), olab)
            assert_features_equal(tl[:k].cpu().numpy(), tf[:k].cpu().numpy(), tt[:k].cpu().numpy(), ol, of, ot)
            c.close()


def test_table_capacity(ctx):
    """More objects than table rows: n_rows is still the true count and the rows written are
    the first ones in label order (hp_run_tiles reports HP_ERR_CAPACITY to its sink)."""
    import torch
    rgb = make_tile(41, TileSpec(384, 384))["rgb"]
    h, w = rgb.shape[:2]
    _, ol, of, ot = oracle.process_tile(rgb)
    assert len(ol) > 8
    t = torch.from_numpy(np.ascontiguousarray(rgb)).cuda()
    lab = torch.zeros((h, w), dtype=torch.int32, device="cuda")
    nobj = torch.zeros(1, dtype=torch.int32, device="cuda")
    cap = 5
    tl = torch.zeros(cap, dtype=torch.int32, device="cuda")
    tf = torch.zeros(cap, dtype=torch.int32, device="cuda")
    tt = torch.zeros((cap, 36), dtype=torch.float32, device="cuda")
    nr = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.process_tile(0, t, lab, nobj, tl, tf, tt, nr)
    torch.cuda.synchronize()
    assert int(nr.item()) == len(ol)
    assert_features_equal(tl.cpu().numpy(), tf.cpu().numpy(), tt.cpu().numpy(), ol[:cap], of[:cap], ot[:cap])


def test_stage_missing_buffer_rejected(ctx):
    from paper_1209_3332_b200.hp import HPError
    with pytest.raises(HPError) as e:
        stage(ctx, "CANNY", [None], [((8, 8), U8)], 8, 8)
    assert e.value.status == 1


def test_pipeline_config1(ctx):
    assert _check_pipeline(ctx, make_config_tile(1)) > 10


@pytest.mark.parametrize("seed,t", [(7, 0.4), (8, 0.7)])
def test_pipeline_partial_tissue(ctx, seed, t):
    rgb = make_tile(seed, TileSpec(1024, 768, tissue_frac=t))["rgb"]
    _check_pipeline(ctx, rgb)


def _painted_tile():
    """A sparse synthetic tile with a thin dark ring (a candidate whose bounding box is far
    larger than any shared-memory window, with a large hole: the huge-window S6 path and the
    global S7-S11 fallback) and a 1-px diagonal line (area < 1000 px, window ~160K px)."""
    rgb = make_tile(11, TileSpec(1024, 1024, density=2e-5))["rgb"].copy()
    yy, xx = np.mgrid[0:1024, 0:1024]
    ring = np.abs(np.hypot(xx - 400, yy - 400) - 70) < 1.0
    line = (np.abs((xx - 600) - (yy - 500)) < 1) & (xx > 600) & (xx < 1000)
    for m in (ring, line):
        rgb[m] = (70, 30, 110)
    return rgb


def test_pipeline_huge_windows(ctx):
    rgb = _painted_tile()
    # the painted structures do reach S6 as candidates (else the test would test nothing)
    g, fl, _ = oracle.cd(rgb)
    cand = oracle.recon_to_nuclei(g, oracle.open_(g), oracle.rbc(fl))
    big0 = oracle.area_threshold(cand)
    assert big0[328:472, 328:472].sum() > 300        # the ring (bbox 142 x 142)
    assert big0[500:900, 600:1000].sum() > 200       # the line (bbox ~400 x 400)
    _check_pipeline(ctx, rgb)


def _island_tile():
    """Candidates inside other candidates' holes: a ring with a separate dot inside, and two
    nested rings around a dot (islands must be solved with their enclosing component)."""
    rgb = make_tile(12, TileSpec(512, 512, density=2e-5))["rgb"].copy()
    yy, xx = np.mgrid[0:512, 0:512]
    paint = np.zeros((512, 512), bool)
    r1 = np.hypot(xx - 120, yy - 140)
    paint |= (np.abs(r1 - 13) < 1.0) | (r1 < 3.2)                       # ring + dot
    r2 = np.hypot(xx - 330, yy - 300)
    paint |= (np.abs(r2 - 22) < 1.0) | (np.abs(r2 - 11) < 1.0) | (r2 < 3.2)  # nested rings + dot
    rgb[paint] = (70, 30, 110)
    return rgb


def test_pipeline_islands(ctx):
    rgb = _island_tile()
    g, fl, _ = oracle.cd(rgb)
    big0 = oracle.area_threshold(oracle.recon_to_nuclei(g, oracle.open_(g), oracle.rbc(fl)))
    _, n_in = oracle.ccl(big0[100:180, 80:160])
    assert n_in >= 2                                   # ring and dot are separate candidates
    F = oracle.fill_holes(big0)
    assert F[135:145, 115:125].all()                   # ... merged into one F component
    _check_pipeline(ctx, rgb)


@pytest.mark.parametrize("seed", range(8))
def test_pipeline_random_small(ctx, seed):
    """Small tiles of varied size, nucleus density and tissue fraction (ragged tile grids,
    components touching tile borders, touching / overlapping nuclei, vesicular nuclei)."""
    rng = np.random.default_rng(500 + seed)
    h, w = int(rng.integers(96, 400)), int(rng.integers(96, 400))
    spec = TileSpec(w, h, tissue_frac=float(rng.uniform(0.3, 1.0)), density=float(rng.uniform(0.5e-4, 4e-4)))
    _check_pipeline(ctx, make_tile(600 + seed, spec)["rgb"])


def test_pipeline_edge_cases(ctx):
    _check_pipeline(ctx, np.full((64, 80, 3), 255, U8))          # glass only
    _check_pipeline(ctx, np.zeros((50, 70, 3), U8))               # black
    _check_pipeline(ctx, make_tile(3, TileSpec(96, 136))["rgb"])  # small ragged tile


@pytest.mark.slow
def test_pipeline_config2_4k(ctx):
    assert _check_pipeline(ctx, make_config_tile(2)) > 1000


def test_determinism(ctx):
    rgb = make_config_tile(1)
    a = _gpu_process(ctx, rgb, slot=0)
    b = _gpu_process(ctx, rgb, slot=1)
    for x, y in zip(a, b):
        assert np.array_equal(np.asarray(x), np.asarray(y))


@pytest.mark.parametrize("kind", ["serpentine", "spiral"])
@pytest.mark.parametrize("ramp", [False, True])
def test_iwpp_stress(ctx, kind, ramp):
    size = 1024
    marker, mask, _ = make_stress(kind, size, ramp)
    rec, st = stage(ctx, "IWPP_RAW", [marker, mask], [((size, size), U8), ((4,), I64)], size, size)
    assert np.array_equal(rec, mask)


@pytest.mark.slow
@pytest.mark.parametrize("kind", ["serpentine", "spiral"])
@pytest.mark.parametrize("ramp", [False, True])
def test_iwpp_stress_4k(ctx, kind, ramp):
    """BASELINE configs[4] at its real size: 4096^2 1-px corridors, one 8.4 M-pixel dependency
    chain; regions re-entered many times go through the alternating-phase closure.  The
    reconstruction of the single-pixel marker under the corridor mask is the mask itself."""
    size = 4096
    marker, mask, _ = make_stress(kind, size, ramp)
    rec, st = stage(ctx, "IWPP_RAW", [marker, mask], [((size, size), U8), ((4,), I64)], size, size)
    assert np.array_equal(rec, mask)


def test_reduce_rows(ctx):
    """hp_reduce_rows (segmented fp64 sums) against numpy, with empty groups,
    and bit-identical run to run."""
    import torch
    rng = np.random.default_rng(5)
    sizes = [0, 1, 7, 300, 0, 2049, 5]
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    feat = (rng.standard_normal((int(off[-1]), 36)) * rng.uniform(0.1, 1e3, 36)).astype(np.float32)
    ft, ot = torch.from_numpy(feat).cuda(), torch.from_numpy(off).cuda()
    outs = []
    for _ in range(2):
        out = torch.full((len(sizes), 36, 2), np.nan, dtype=torch.float64, device="cuda")
        cnt = torch.full((len(sizes),), -1, dtype=torch.int64, device="cuda")
        ctx.reduce_rows(ft, ot, out, cnt)
        torch.cuda.synchronize()
        outs.append((out.cpu().numpy(), cnt.cpu().numpy()))
    (o, c), (o2, c2) = outs
    assert np.array_equal(c, sizes) and np.array_equal(o, o2)      # deterministic
    for g in range(len(sizes)):
        f = feat[off[g]:off[g + 1]].astype(np.float64)
        assert np.allclose(o[g, :, 0], f.sum(axis=0), rtol=1e-12, atol=1e-9)
        assert np.allclose(o[g, :, 1], (f * f).sum(axis=0), rtol=1e-12, atol=1e-9)


def test_aggregate_groups_on_gpu(ctx):
    """dist.aggregate_groups through the device kernel == numpy on a pipeline table."""
    import torch
    from paper_1209_3332_b200.dist import aggregate_groups, to_rows
    tiles = {i: make_tile(800 + i, TileSpec(256, 256))["rgb"] for i in range(4)}
    res = {}
    for i, rgb in tiles.items():
        _, _, gl, gf, gt = _gpu_process(ctx, rgb)
        res[i] = (gl, gf, gt)
    rows = to_rows(res)
    cnt, mean, std = aggregate_groups(rows, lambda t: t // 2, 3, reduce=ctx, device=torch.device("cuda"))
    off = np.searchsorted(rows.tile // 2, np.arange(4))
    rc, rm, rs = oracle.aggregate(rows.feat, off)   # group 2 is empty: NaN on both sides
    assert np.array_equal(cnt, rc) and cnt[0] > 0 and cnt[1] > 0 and cnt[2] == 0
    assert np.allclose(mean, rm, rtol=1e-12, atol=1e-12, equal_nan=True)
    assert np.allclose(std, rs, rtol=1e-10, atol=1e-12, equal_nan=True)


def test_aggregate_groups_no_rows(ctx):
    """A rank with an empty table: the device kernels accept the NULL feature
    pointer of an empty tensor and report zero counts and NaN statistics."""
    import torch
    from paper_1209_3332_b200.dist import Rows, aggregate_groups
    cnt, mean, std = aggregate_groups(Rows.concat([]), lambda t: t, 2, reduce=ctx, device=torch.device("cuda"))
    assert list(cnt) == [0, 0] and np.isnan(mean).all() and np.isnan(std).all()


def test_run_tiles_size_change(ctx):
    """hp_run_tiles replays a per-slot CUDA graph; a new tile size must rebuild it."""
    import torch
    for (h, w, base) in [(256, 384, 700), (320, 200, 710), (256, 384, 720)]:
        tiles = [make_tile(base + i, TileSpec(h, w))["rgb"] for i in range(7)]
        pinned = [torch.from_numpy(t).pin_memory() for t in tiles]
        it = iter(range(len(tiles)))
        got = {}

        def nxt():
            try:
                i = next(it)
            except StopIteration:
                return None
            return pinned[i].data_ptr(), 3 * w, i

        def done(tid, lab, fl, ft, st):
            assert st == 0
            got[tid] = (lab, fl, ft)

        ctx.run_tiles(nxt, done, w, h)
        assert sorted(got) == list(range(len(tiles)))
        for i, rgb in enumerate(tiles):
            _, ol, of, ot = oracle.process_tile(rgb)
            assert_features_equal(got[i][0], got[i][1], got[i][2], ol, of, ot)


def test_run_tiles(ctx):
    import torch
    tiles = [make_tile(100 + i, TileSpec(512, 512))["rgb"] for i in range(5)]
    pinned = [torch.from_numpy(t).pin_memory() for t in tiles]
    order = list(range(len(tiles))) * 2
    it = iter(order)
    got = {}

    def nxt():
        try:
            i = next(it)
        except StopIteration:
            return None
        return pinned[i].data_ptr(), 3 * 512, i

    def done(tid, lab, fl, ft, st):
        assert st == 0
        if tid in got:
            assert np.array_equal(got[tid][2], ft)  # repeats are byte-identical
        got[tid] = (lab, fl, ft)

    ctx.run_tiles(nxt, done, 512, 512)
    assert sorted(got) == list(range(len(tiles)))
    for i, rgb in enumerate(tiles):
        _, ol, of, ot = oracle.process_tile(rgb)
        assert_features_equal(got[i][0], got[i][1], got[i][2], ol, of, ot)


@pytest.mark.parametrize("where", ["next_tile", "on_done"])
def test_run_tiles_callback_errors_propagate(ctx, where):
    """An exception raised in either Python callback of run_tiles is re-raised by run_tiles
    itself once the driver returns (ctypes would print and swallow it: ADVICE r1), no further
    tile is fed after it, and the context stays usable."""
    import torch
    tiles = [torch.from_numpy(make_tile(140 + i, TileSpec(256, 256))["rgb"]).pin_memory() for i in range(3)]
    fed = []

    def nxt():
        k = len(fed)
        if where == "next_tile" and k == 1:
            raise ValueError("feeder failed")
        if k >= len(tiles):
            return None
        fed.append(k)
        return tiles[k].data_ptr(), 3 * 256, k

    def done(tid, lab, fl, ft, st):
        assert st == 0
        if where == "on_done":
            raise KeyError("sink failed")

    with pytest.raises(ValueError if where == "next_tile" else KeyError):
        ctx.run_tiles(nxt, done, 256, 256)
    if where == "next_tile":
        assert fed == [0]
    # the context still runs tiles afterwards
    got = []
    it = iter(range(len(tiles)))

    def nxt2():
        k = next(it, None)
        return None if k is None else (tiles[k].data_ptr(), 3 * 256, k)

    ctx.run_tiles(nxt2, lambda tid, lab, fl, ft, st: got.append((tid, st)), 256, 256)
    assert sorted(got) == [(k, 0) for k in range(len(tiles))]


def _arena(torch, cap):
    from paper_1209_3332_b200.hp import NFEAT
    dev = "cuda"
    a = dict(tile=torch.full((cap,), -1, dtype=torch.int64, device=dev),
             label=torch.zeros(cap, dtype=torch.int32, device=dev),
             flags=torch.zeros(cap, dtype=torch.int32, device=dev),
             feat=torch.zeros(cap, NFEAT, dtype=torch.float32, device=dev),
             cursor=torch.zeros(1, dtype=torch.int64, device=dev))
    ptrs = (a["tile"].data_ptr(), a["label"].data_ptr(), a["flags"].data_ptr(),
            a["feat"].data_ptr(), cap, a["cursor"].data_ptr())
    return a, ptrs


def test_run_tiles_arena(ctx):
    """S12 into the device arena: every tile's rows land as one contiguous run tagged with
    its tile id; after sorting by (tile, label) the table is the oracle's.  Tiles repeat
    (the per-slot graph is captured and replayed with the arena) and a second call with the
    same arena continues at the cursor."""
    import torch
    tiles = [make_tile(300 + i, TileSpec(384, 448))["rgb"] for i in range(5)]
    pinned = [torch.from_numpy(t).pin_memory() for t in tiles]
    ref = [oracle.process_tile(rgb)[1:] for rgb in tiles]
    total = sum(len(r[0]) for r in ref)
    a, ptrs = _arena(torch, 4 * total + 8)
    counts = {}
    for call in range(2):
        ids = [(call, i) for i in range(len(tiles))] * 2
        it = iter(ids)

        def nxt():
            try:
                c, i = next(it)
            except StopIteration:
                return None
            return pinned[i].data_ptr(), 3 * 448, 10 * c + i

        def done(tid, n, st):
            assert st == 0
            counts.setdefault(tid, []).append(n)

        ctx.run_tiles(nxt, done, 448, 384, arena=ptrs)
    torch.cuda.synchronize()
    n = int(a["cursor"].item())
    assert n == 4 * total
    tile = a["tile"][:n].cpu().numpy()
    lab = a["label"][:n].cpu().numpy()
    fl = a["flags"][:n].cpu().numpy()
    ft = a["feat"][:n].cpu().numpy()
    assert int(a["tile"][n:].cpu().numpy().max(initial=-1)) == -1  # nothing past the cursor
    assert sorted(counts) == sorted(10 * c + i for c in range(2) for i in range(len(tiles)))
    for tid, ns in counts.items():
        i = tid % 10
        m = len(ref[i][0])
        assert ns == [m, m]
        idx = np.flatnonzero(tile == tid)
        assert len(idx) == 2 * m
        # each delivery is one contiguous run in label order, equal to the oracle's table
        runs = np.split(idx, np.flatnonzero(np.diff(idx) != 1) + 1)
        runs = [r for run in runs for r in np.split(run, range(m, len(run), m))] if m else []
        assert len(runs) == (2 if m else 0)
        for r in runs:
            assert len(r) == m and np.array_equal(r, np.arange(r[0], r[0] + m))
            assert_features_equal(lab[r], fl[r], ft[r], *ref[i])


def test_arena_device_gather(ctx):
    """dist.RowArena + gather_rows_device (one process): rows appended on the device in
    completion order come back in (tile, label) order, equal to the oracle's tables."""
    import torch
    from paper_1209_3332_b200.dist import RowArena, gather_rows_device
    tiles = [make_tile(330 + i, TileSpec(256, 320))["rgb"] for i in range(3)]
    pinned = [torch.from_numpy(t).pin_memory() for t in tiles]
    ref = [oracle.process_tile(rgb)[1:] for rgb in tiles]
    ra = RowArena(sum(len(r[0]) for r in ref) * 3 + 16, "cuda")
    order = iter([5, 1, 7, 3, 2, 0])

    def nxt():
        t = next(order, None)
        return None if t is None else (pinned[t % 3].data_ptr(), 3 * 320, t)

    ctx.run_tiles(nxt, lambda tid, n, st: None, 320, 256, arena=ra.arena)
    tab = gather_rows_device(ra.rows()).to_host()
    assert list(np.unique(tab.tile)) == [0, 1, 2, 3, 5, 7]
    assert np.all(np.diff(tab.tile) >= 0)
    for t in [0, 1, 2, 3, 5, 7]:
        sel = tab.tile == t
        assert_features_equal(tab.label[sel], tab.flags[sel], tab.feat[sel], *ref[t % 3])


def test_run_tiles_arena_overflow(ctx):
    """An arena smaller than the rows: the cursor still counts every row, rows past the
    capacity are dropped, and the tiles whose run did not fit report HP_ERR_CAPACITY."""
    import torch
    tiles = [make_tile(320 + i, TileSpec(384, 448))["rgb"] for i in range(4)]
    pinned = [torch.from_numpy(t).pin_memory() for t in tiles]
    nref = [len(oracle.process_tile(rgb)[1]) for rgb in tiles]
    cap = sum(nref) // 2
    a, ptrs = _arena(torch, cap)
    it = iter(range(len(tiles)))
    sts = {}

    def nxt():
        try:
            i = next(it)
        except StopIteration:
            return None
        return pinned[i].data_ptr(), 3 * 448, i

    def done(tid, n, st):
        sts[tid] = (n, st)

    ctx.run_tiles(nxt, done, 448, 384, arena=ptrs)
    torch.cuda.synchronize()
    assert int(a["cursor"].item()) == sum(nref)
    assert {t: v[0] for t, v in sts.items()} == dict(enumerate(nref))
    tile = a["tile"].cpu().numpy()
    assert (tile >= 0).all()  # the arena is full
    kept = np.bincount(tile, minlength=len(tiles))
    for t, (n, st) in sts.items():
        assert (st == 0) == (kept[t] == n), (t, n, st, kept[t])
        assert st in (0, 4)
    assert any(st == 4 for _, st in sts.values())


def _pool_tile(seed):
    import bench  # the bench's seeded tile cache (same seeds, same painter call)
    return bench._gen((seed, 4096))


BENCH_SLOTS, BENCH_E2E_SLOTS, BENCH_BATCH = 12, 24, 12   # bench.py's defaults


def _oracle_rows(rgb):
    import hashlib
    lab, ol, of, ot = oracle.process_tile(rgb)
    return hashlib.sha256(lab.tobytes()).hexdigest(), ol, of, ot


@pytest.fixture(scope="module")
def bench_ref():
    """bench.py's own 4K tiles (configs[2] pool seeds 1000..; HP_POOL_PARITY=N checks the
    first N, default bench.py's batch of 12, 64 = the whole configs[2] pool) and the oracle's
    result for each (label digest, rows), computed on all host cores."""
    import multiprocessing as mp
    import os
    K = int(os.environ.get("HP_POOL_PARITY", str(BENCH_BATCH)))
    pctx = mp.get_context("fork")
    with pctx.Pool(max(1, min(K, os.cpu_count() or 1))) as pool:
        tiles = pool.map(_pool_tile, range(1000, 1000 + K))
        ref = pool.map(_oracle_rows, tiles)
    return tiles, ref


@pytest.mark.slow
def test_bench_tiles_in_bench_launch_config(bench_ref):
    """Parity at BASELINE's full size in the launch configuration bench.py's device-resident
    leg times: its 12 tiles through hp_process_tile on 12 slots, one stream each, all in
    flight at once, 32 hardware work queues (conftest.py, as bench.py) -- label planes
    bit-exact, tables within reading C18."""
    import hashlib

    import torch
    from paper_1209_3332_b200 import Context
    tiles, ref = bench_ref
    S, size, cap = BENCH_SLOTS, 4096, 8192
    c = Context(0, size, size, n_slots=max(S, BENCH_E2E_SLOTS), max_objects=cap)
    try:
        lab = [torch.empty((size, size), dtype=torch.int32, device="cuda") for _ in range(S)]
        nob = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(S)]
        tl = [torch.empty(cap, dtype=torch.int32, device="cuda") for _ in range(S)]
        tf = [torch.empty(cap, dtype=torch.int32, device="cuda") for _ in range(S)]
        tt = [torch.empty((cap, 36), dtype=torch.float32, device="cuda") for _ in range(S)]
        nr = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(S)]
        streams = [torch.cuda.Stream() for _ in range(S)]
        for b0 in range(0, len(tiles), S):
            idx = list(range(b0, min(len(tiles), b0 + S)))
            dev = [torch.from_numpy(tiles[i]).cuda() for i in idx]
            torch.cuda.synchronize()
            for k in range(len(idx)):
                c.process_tile(k, dev[k], lab[k], nob[k], tl[k], tf[k], tt[k], nr[k], stream=streams[k])
            torch.cuda.synchronize()
            for k, i in enumerate(idx):
                odig, ol, of, ot = ref[i]
                gl = lab[k].cpu().numpy()
                assert hashlib.sha256(gl.tobytes()).hexdigest() == odig, f"labels of pool tile {i}"
                n = int(nr[k].item())
                assert int(nob[k].item()) == n == len(ol) > 1000
                assert_features_equal(tl[k][:n].cpu().numpy(), tf[k][:n].cpu().numpy(),
                                      tt[k][:n].cpu().numpy(), ol, of, ot)
    finally:
        c.close()


@pytest.mark.slow
def test_bench_e2e_launch_config(bench_ref):
    """Parity of bench.py's e2e leg in its exact configuration: hp_run_tiles on 24 slots with
    per-slot CUDA graphs (captured on a slot's second tile, replayed after), pinned host tiles,
    32 hardware work queues, the bench's tiles twice each in a demand-driven order -- every
    delivered table equals the oracle's (labels and flags exact, features within C18)."""
    import torch
    from paper_1209_3332_b200 import Context
    from paper_1209_3332_b200.dist import DistTileSource, TileQueue
    tiles, ref = bench_ref
    K = len(tiles)
    size, cap = 4096, 8192
    c = Context(0, size, size, n_slots=max(BENCH_SLOTS, BENCH_E2E_SLOTS), max_objects=cap)
    try:
        pinned = [torch.from_numpy(t).pin_memory() for t in tiles]
        q = TileQueue(2 * K, block=BENCH_SLOTS, store=None)
        src = DistTileSource(q, lambda tid: pinned[tid % K])
        got = {}

        def done(tid, l, f, ft, st):
            assert st == 0, f"tile {tid} status {st}"
            got[tid] = (l, f, ft)

        c.run_tiles(src, done, size, size)
        assert sorted(got) == list(range(2 * K))
        for tid, (l, f, ft) in got.items():
            _, ol, of, ot = ref[tid % K]
            assert_features_equal(l, f, ft, ol, of, ot)
    finally:
        c.close()


def test_run_tiles_errors(ctx):
    """hp_run_tiles argument errors: a size beyond the context and a bad tile pitch are
    HP_ERR_INVALID (the bad tile after the good ones in flight finished, undelivered), an
    arena with a NULL buffer is rejected; the context stays usable afterwards."""
    import torch
    from paper_1209_3332_b200.hp import HPError
    rgb = make_tile(31, TileSpec(128, 160))["rgb"]
    pinned = torch.from_numpy(rgb).pin_memory()
    with pytest.raises(HPError) as e:
        ctx.run_tiles(lambda: None, lambda *a: None, 8192, 64)
    assert e.value.status == 1
    seq = iter([(pinned.data_ptr(), 3 * 160, 0), (pinned.data_ptr(), 3 * 160, 1),
                (pinned.data_ptr(), 3 * 160 - 1, 2)])
    with pytest.raises(HPError) as e:
        ctx.run_tiles(lambda: next(seq, None), lambda *a: None, 160, 128)
    assert e.value.status == 1
    with pytest.raises(HPError) as e:
        ctx.run_tiles(lambda: None, lambda *a: None, 160, 128, arena=(0, 0, 0, 0, 10, 0))
    assert e.value.status == 1
    got = {}
    seq = iter([(pinned.data_ptr(), 3 * 160, 7)])
    ctx.run_tiles(lambda: next(seq, None), lambda t, l, f, x, s: got.setdefault(t, (l, f, x, s)), 160, 128)
    _, ol, of, ot = oracle.process_tile(rgb)
    assert got[7][3] == 0
    assert_features_equal(got[7][0], got[7][1], got[7][2], ol, of, ot)


@pytest.mark.parametrize("case", ["small_disk", "strict", "loose"])
def test_pipeline_nondefault_params(case):
    """The same hp_params drive both sides: a non-default opening diameter, thresholds, area
    bounds, h and Canny thresholds give the oracle's labels and rows."""
    from paper_1209_3332_b200 import Context
    from paper_1209_3332_b200.hp import Params as HParams
    p = oracle.default_params()
    if case == "small_disk":
        p.open_diam, p.g1, p.h = 11, 40, 2.0
    elif case == "strict":
        p.cand_min_area, p.cand_max_area, p.obj_min_area, p.obj_max_area = 30, 400, 40, 300
        p.canny_low, p.canny_high = 40, 90
    else:
        p.rbc_t1, p.rbc_t2, p.g1, p.h = 3, 2, 30, 0.5
        p.canny_low, p.canny_high = 0, 0
    rgb = make_tile(41, TileSpec(384, 512))["rgb"]
    with Context(0, 512, 384, n_slots=1, max_objects=8192, params=HParams.from_dict(p.to_dict())) as c:
        lab, nobj, gl, gf, gt = _gpu_process(c, rgb, cap=8192)
    olab, ol, of, ot = oracle.process_tile(rgb, params=p)
    assert np.array_equal(lab, olab) and nobj == len(ol)
    assert_features_equal(gl, gf, gt, ol, of, ot)


def test_background_skip():
    """bg_skip_frac <= 1 (reading C19): a tile whose BG fraction reaches it yields no
    objects on both sides; a tissue tile below it is processed as usual."""
    from paper_1209_3332_b200 import Context
    from paper_1209_3332_b200.hp import Params as HParams
    p = oracle.default_params()
    p.bg_skip_frac = 0.5
    glass = make_tile(43, TileSpec(256, 256, tissue_frac=0.2))["rgb"]   # mostly glass
    tissue = make_tile(44, TileSpec(256, 256))["rgb"]
    with Context(0, 256, 256, n_slots=1, max_objects=4096, params=HParams.from_dict(p.to_dict())) as c:
        for rgb in (glass, tissue):
            lab, nobj, gl, gf, gt = _gpu_process(c, rgb, cap=4096)
            olab, ol, of, ot = oracle.process_tile(rgb, params=p)
            assert np.array_equal(lab, olab) and nobj == len(ol)
            assert_features_equal(gl, gf, gt, ol, of, ot)
    assert len(oracle.process_tile(glass, params=p)[1]) == 0
    assert len(oracle.process_tile(tissue, params=p)[1]) > 0


def test_strided_input_and_label_pitch(ctx):
    """A tile that is a window of a wider image (pitch > 3*width) and a label plane with a
    pitch > width give the same result as the dense call."""
    import torch
    big = make_tile(45, TileSpec(320, 600))["rgb"]
    rgb = np.ascontiguousarray(big[:, 37:37 + 450])
    ref = _gpu_process(ctx, rgb, cap=8192)
    olab, ol, of, ot = oracle.process_tile(rgb)
    assert np.array_equal(ref[0], olab)
    t = torch.from_numpy(big).cuda()[:, 37:37 + 450]            # stride(0) = 3*600 bytes
    assert t.stride(0) == 3 * 600
    lab_wide = torch.full((320, 512), -7, dtype=torch.int32, device="cuda")
    lab = lab_wide[:, :450]
    nobj = torch.zeros(1, dtype=torch.int32, device="cuda")
    cap = 8192
    tl = torch.zeros(cap, dtype=torch.int32, device="cuda")
    tf = torch.zeros(cap, dtype=torch.int32, device="cuda")
    tt = torch.zeros((cap, 36), dtype=torch.float32, device="cuda")
    nr = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.process_tile(0, t, lab, nobj, tl, tf, tt, nr)
    torch.cuda.synchronize()
    k = int(nr.item())
    assert np.array_equal(lab.cpu().numpy(), olab)
    assert (lab_wide[:, 450:] == -7).all()                        # the pitch padding is untouched
    assert_features_equal(tl[:k].cpu().numpy(), tf[:k].cpu().numpy(), tt[:k].cpu().numpy(), ol, of, ot)


@pytest.mark.parametrize("hw", [(1031, 1153), (257, 16384), (4099, 65)])
def test_pipeline_ragged_and_max_width(hw):
    """Odd sizes (partial regions, tiles and vector words on both edges; rows not 4-byte
    aligned) and the maximum width hp_config allows, against the oracle."""
    from paper_1209_3332_b200 import Context
    h, w = hw
    rgb = make_tile(50 + h % 7, TileSpec(h, w))["rgb"]
    with Context(0, w, h, n_slots=1, max_objects=16384) as c:
        lab, nobj, gl, gf, gt = _gpu_process(c, rgb, cap=16384)
    olab, ol, of, ot = oracle.process_tile(rgb)
    assert np.array_equal(lab, olab) and nobj == len(ol) > 0
    assert_features_equal(gl, gf, gt, ol, of, ot)


@pytest.mark.parametrize("seed", [0, 1])
def test_components_big_windows_separable_edt(seed):
    """Components whose windows exceed shared memory (> 2432 px) take the global-memory path,
    whose S7 is the separable exact EDT (k_comp.cu); with area bounds up to 131072 the big
    objects survive S10, so their EDT -> markers -> watershed -> labels -> features are all
    observable: bit-exact labels, features within C18 (oracle chain on the same F)."""
    import torch
    from paper_1209_3332_b200 import Context
    from paper_1209_3332_b200.hp import Params as HParams
    rng = np.random.default_rng(seed)
    h, w = 300, 360
    yy, xx = np.indices((h, w))
    F = np.zeros((h, w), bool)
    for _ in range(4):  # overlapping big blobs (watershed splits) with notches and holes filled
        cy, cx, a, b = rng.uniform(60, 240), rng.uniform(60, 300), rng.uniform(25, 60), rng.uniform(25, 60)
        F |= ((yy - cy) / a) ** 2 + ((xx - cx) / b) ** 2 <= 1.0
    F &= rng.random((h, w)) > 0.002  # pinholes, filled again below: S6 output has no holes
    F = oracle.fill_holes(F.astype(U8))
    g = rng.integers(0, 256, size=(h, w)).astype(U8)
    p = oracle.default_params()
    p.obj_max_area = p.cand_max_area = 131072
    d2, dist = oracle.edt(F)
    ML, _, _ = oracle.markers(dist, F, 1.0)
    split, _, _, _ = oracle.watershed(dist, ML, F)
    labels, nobj = oracle.bwlabel(split, p.obj_min_area, p.obj_max_area)
    assert nobj >= 1 and np.bincount(labels[labels > 0]).max() > 2432
    ol, of, ot = oracle.features(labels, g)
    cap = 4096
    with Context(0, w, h, n_slots=1, max_objects=cap, params=HParams.from_dict(p.to_dict())) as c:
        lab, nob, lf, ft = stage(c, "COMPONENTS", [F, g], [((h, w), I32), ((1,), I32), ((2, cap), I32),
                                                          ((cap, 36), F32)], w, h)
    assert np.array_equal(lab, labels) and int(nob[0]) == nobj
    assert_features_equal(lf[0, :nobj], lf[1, :nobj], ft[:nobj], ol, of, ot)
