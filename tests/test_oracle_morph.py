"""Pins of the oracle's S3 (Morph. Open, 19x19 disk) and of the
Vincent MR used by S2/S4/S8/S9.

Pinned against: OpenCV's own erode/dilate/morphologyEx with MORPH_ELLIPSE (the library the
paper names), the golden 19x19 row widths, idempotence/anti-extensivity of the opening, and
the textbook definition of reconstruction as the fixed point of iterated geodesic dilation.
"""
import os

import cv2
import numpy as np
import pytest
from hypothesis import given, settings, strategies as st
from scipy import ndimage as ndi

import oracle
from synth import make_stress

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_ellipse_golden():
    widths = [int(v) for l in open(os.path.join(GOLDEN, "ellipse19.txt"))
              if not l.startswith("#") for v in l.split()]
    se = cv2.getStructuringElement(cv2.MORPH_ELLIPSE, (19, 19))
    assert list(se.sum(1)) == widths and sum(widths) == 269
    # the oracle's element: erode a single dark pixel with a white background -> its footprint
    img = np.full((41, 41), 255, np.uint8)
    img[20, 20] = 0
    er = oracle.erode(img, 19)
    fp = (er == 0).astype(np.uint8)
    assert list(fp[11:30, 11:30].sum(1)) == widths and fp.sum() == 269


@pytest.mark.parametrize("diam", [3, 5, 7, 11, 19])
@pytest.mark.parametrize("shape", [(1, 37), (37, 1), (23, 41), (64, 64)])
def test_against_opencv(diam, shape):
    rng = np.random.default_rng(diam * 1000 + shape[0])
    g = rng.integers(0, 256, size=shape, dtype=np.uint8)
    se = cv2.getStructuringElement(cv2.MORPH_ELLIPSE, (diam, diam))
    assert np.array_equal(oracle.erode(g, diam), cv2.erode(g, se))
    assert np.array_equal(oracle.dilate(g, diam), cv2.dilate(g, se))
    assert np.array_equal(oracle.open_(g, diam), cv2.morphologyEx(g, cv2.MORPH_OPEN, se))


def test_open_invariants(tile512):
    g, _, _ = oracle.cd(tile512)
    o = oracle.open_(g)
    assert np.all(o <= g)
    assert np.array_equal(oracle.open_(o), o)
    se = cv2.getStructuringElement(cv2.MORPH_ELLIPSE, (19, 19))
    assert np.array_equal(o, cv2.morphologyEx(g, cv2.MORPH_OPEN, se))


def _recon_fixed_point(marker, mask, dom=None):
    """Textbook: iterate R <- min(dilate3x3(R), mask) from min(marker, mask) to stability."""
    if dom is None:
        R = np.minimum(marker, mask)
        while True:
            nxt = np.minimum(ndi.grey_dilation(R, size=(3, 3), mode="constant",
                                               cval=np.iinfo(R.dtype).min if R.dtype.kind == "u"
                                               else -np.inf), mask)
            nxt = np.maximum(nxt, R)
            if np.array_equal(nxt, R):
                return R
            R = nxt
    NEG = np.float32(-np.inf)
    R = np.where(dom, np.minimum(marker, mask), NEG).astype(np.float32)
    mk = np.where(dom, mask, NEG).astype(np.float32)
    while True:
        d = ndi.grey_dilation(R, size=(3, 3), mode="constant", cval=-np.inf)
        nxt = np.where(dom, np.maximum(R, np.minimum(d, mk)), NEG)
        if np.array_equal(nxt, R):
            return np.where(dom, R, 0).astype(np.float32)
        R = nxt


@settings(max_examples=60, deadline=None)
@given(h=st.integers(1, 24), w=st.integers(1, 24), seed=st.integers(0, 2**31 - 1),
       levels=st.sampled_from([2, 4, 256]))
def test_recon_u8_equals_fixed_point(h, w, seed, levels):
    rng = np.random.default_rng(seed)
    mask = (rng.integers(0, levels, size=(h, w)) * (255 // max(1, levels - 1))).astype(np.uint8)
    marker = rng.integers(0, 256, size=(h, w)).astype(np.uint8)
    marker[rng.random((h, w)) < 0.7] = 0
    assert np.array_equal(oracle.recon_u8(marker, mask), _recon_fixed_point(marker, mask))


@settings(max_examples=40, deadline=None)
@given(h=st.integers(1, 20), w=st.integers(1, 20), seed=st.integers(0, 2**31 - 1))
def test_recon_f32_domain_equals_fixed_point(h, w, seed):
    rng = np.random.default_rng(seed)
    dom = (rng.random((h, w)) < 0.7).astype(np.uint8)
    mask = rng.integers(0, 6, size=(h, w)).astype(np.float32) * 0.5
    marker = np.where(rng.random((h, w)) < 0.3, mask, -np.inf).astype(np.float32)
    got = oracle.recon_f32(marker, mask, dom)
    exp = _recon_fixed_point(marker, mask, dom.astype(bool))
    assert np.array_equal(got[dom == 1], exp[dom == 1])


def test_recon_invariants(tile512):
    g, _, _ = oracle.cd(tile512)
    o = oracle.open_(g)
    R = oracle.recon_u8(o, g)
    assert np.all(o <= R) and np.all(R <= g)
    assert np.array_equal(oracle.recon_u8(g, g), g)            # GrayRecon(g, g) = g
    assert np.array_equal(oracle.recon_u8(R, g), R)            # idempotence
    assert np.array_equal(R, _recon_fixed_point(o, g))


def test_binary_recon_is_ccl_select():
    rng = np.random.default_rng(5)
    mask = (rng.random((60, 70)) < 0.55).astype(np.uint8) * 255
    marker = ((rng.random((60, 70)) < 0.02) * 255).astype(np.uint8)
    lab, n = ndi.label(mask > 0, structure=np.ones((3, 3)))
    hit = np.unique(lab[(marker > 0) & (mask > 0)])
    exp = np.isin(lab, hit[hit > 0]).astype(np.uint8) * 255
    assert np.array_equal(oracle.recon_u8(marker, mask), exp)


@pytest.mark.parametrize("kind", ["serpentine", "spiral"])
@pytest.mark.parametrize("ramp", [False, True])
def test_stress_recon_equals_mask(kind, ramp):
    marker, mask, L = make_stress(kind, 128, ramp)
    out, st_ = oracle.recon_u8(marker, mask, with_stats=True)
    assert np.array_equal(out, mask)
    assert L > 0.49 * 128 * 128
