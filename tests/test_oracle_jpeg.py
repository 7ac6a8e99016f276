"""Pins of the oracle's JPEG decoder (NEXT-3 compressed ingest; oracle/jpeg.cpp, T.81 with
readings J1-J2): bit-exact against cv2.imdecode -- the IJG library, whose islow IDCT and
fixed-point JFIF colour conversion readings J1-J2 name -- on synthetic H&E tiles, noise and
extreme-contrast images over qualities, ragged sizes (partial MCUs) and restart intervals;
the level-shift/clamp closed form on flat images; and loud refusal of what is out of scope."""
import cv2
import numpy as np
import pytest

import oracle
from synth.hne import TileSpec, make_tile
from synth.jpeg import encode_tile


def _cv2_rgb(buf):
    return cv2.imdecode(buf, cv2.IMREAD_COLOR)[:, :, ::-1]


@pytest.mark.parametrize("shape,q,rst", [((64, 64), 90, 4), ((37, 53), 75, 1), ((300, 257), 95, 0),
                                         ((512, 512), 90, 4), ((129, 200), 50, 17), ((8, 8), 100, 1),
                                         ((1, 300), 90, 2), ((301, 1), 85, 3)])
def test_matches_cv2_on_tiles(shape, q, rst):
    rgb = make_tile(sum(shape) + q, TileSpec(*shape))["rgb"]
    buf = encode_tile(rgb, q, rst)
    assert np.array_equal(oracle.jpeg_decode(buf), _cv2_rgb(buf))


@pytest.mark.parametrize("kind", ["noise", "checker", "ramp"])
@pytest.mark.parametrize("q", [60, 100])
def test_matches_cv2_hard_images(kind, q):
    rng = np.random.default_rng(7)
    h, w = 96, 136
    if kind == "noise":
        rgb = rng.integers(0, 256, (h, w, 3)).astype(np.uint8)
    elif kind == "checker":   # 0/255 pixel checkerboard: maximal overshoot, exercises the clamp
        yy, xx = np.indices((h, w))
        rgb = np.repeat(((yy + xx) % 2 * 255).astype(np.uint8)[:, :, None], 3, axis=2)
        rgb[:, :, 1] = 255 - rgb[:, :, 1]
    else:
        yy, xx = np.indices((h, w))
        rgb = np.stack([(xx * 2) % 256, (yy * 3) % 256, (xx + yy) % 256], axis=2).astype(np.uint8)
    buf = encode_tile(rgb, q, 5)
    assert np.array_equal(oracle.jpeg_decode(buf), _cv2_rgb(buf))


@pytest.mark.parametrize("v", [0, 1, 77, 128, 200, 254, 255])
def test_flat_grey_closed_form(v):
    """A flat grey image has Cb = Cr = 128 and only DC terms: the IDCT gives the constant
    DC*Q/8 + 128 (A.3.3 with u = v = 0) and the colour step leaves grey unchanged, so a
    quality-100 encoding (Q = 1) decodes to the input exactly."""
    rgb = np.full((24, 40, 3), v, np.uint8)
    out = oracle.jpeg_decode(encode_tile(rgb, 100, 1))
    assert np.array_equal(out, rgb)


@pytest.mark.parametrize("shape,q,rst", [((64, 64), 90, 4), ((37, 53), 75, 1), ((300, 257), 95, 0),
                                         ((512, 512), 90, 4), ((1, 300), 90, 2), ((301, 1), 85, 3),
                                         ((2, 2), 90, 1), ((9, 3), 90, 1), ((7, 4), 90, 2), ((5, 5), 90, 1),
                                         ((17, 33), 60, 2), ((2, 300), 90, 1)])
def test_matches_cv2_420(shape, q, rst):
    """4:2:0 (Y 2x2, chroma 1x1): reading J4's triangle-filter upsampling (the IJG "fancy"
    path; chroma at most 2 samples wide is replicated instead), bit for bit with OpenCV --
    ragged sizes exercise the first / last column and row special cases."""
    rgb = make_tile(sum(shape) + q + 7, TileSpec(*shape))["rgb"]
    buf = encode_tile(rgb, q, rst, sampling="420")
    assert np.array_equal(oracle.jpeg_decode(buf), _cv2_rgb(buf))


@pytest.mark.parametrize("rgbv", [(200, 30, 90), (12, 240, 7), (128, 128, 128)])
def test_420_flat_colour_closed_form(rgbv):
    """A flat colour has constant chroma planes; the filter's weights sum to 16 with rounding
    offsets 8 / 7, so (16 c + 8) >> 4 = (16 c + 7) >> 4 = c: the upsampled chroma, hence the
    decoded image, is uniform -- and equal to the 4:4:4 decode of the same colour."""
    rgb = np.full((40, 56, 3), rgbv, np.uint8)
    a = oracle.jpeg_decode(encode_tile(rgb, 95, 2, sampling="420"))
    assert (a == a[0, 0]).all()
    b = oracle.jpeg_decode(encode_tile(rgb, 95, 2, sampling="444"))
    assert np.array_equal(a[0, 0], b[0, 0])


def test_out_of_scope_refused():
    rgb = make_tile(3, TileSpec(64, 64))["rgb"]
    with pytest.raises(RuntimeError):
        oracle.jpeg_decode(encode_tile(rgb, 90, 4, sampling="422"))
    with pytest.raises(RuntimeError):
        oracle.jpeg_decode(encode_tile(rgb, 90, 0, progressive=True))
    with pytest.raises(RuntimeError):
        oracle.jpeg_decode(np.zeros(16, np.uint8))
