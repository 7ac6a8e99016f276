"""Pins of the oracle's labelling stages: S2 RBC, S5 AreaThreshold, S6 FillHoles, S10
BWLabel and S7 EDT.

Pinned against: scipy.ndimage.label (partition AND numbering by min linear index),
np.bincount areas, scipy.ndimage.binary_fill_holes, scipy/OpenCV exact EDTs and brute-force
nearest-background search.
"""
import cv2
import numpy as np
import pytest
from hypothesis import given, settings, strategies as st
from scipy import ndimage as ndi

import oracle


def _canon(lab_scipy):
    """scipy label image -> canonical labels 1 + min linear index."""
    n = lab_scipy.max()
    if n == 0:
        return np.zeros_like(lab_scipy, dtype=np.int32)
    idx = np.arange(lab_scipy.size).reshape(lab_scipy.shape)
    mins = ndi.minimum(idx, lab_scipy, index=np.arange(1, n + 1)).astype(np.int64)
    lut = np.zeros(n + 1, np.int64)
    lut[1:] = mins + 1
    return lut[lab_scipy].astype(np.int32)


@settings(max_examples=80, deadline=None)
@given(h=st.integers(1, 30), w=st.integers(1, 30), seed=st.integers(0, 2**31 - 1),
       dens=st.floats(0.05, 0.95), conn=st.sampled_from([4, 8]))
def test_ccl_against_scipy(h, w, seed, dens, conn):
    fg = (np.random.default_rng(seed).random((h, w)) < dens).astype(np.uint8)
    lab, n = oracle.ccl(fg, conn)
    st_ = np.ones((3, 3)) if conn == 8 else ndi.generate_binary_structure(2, 1)
    ls, ns = ndi.label(fg, structure=st_)
    assert n == ns
    assert np.array_equal(lab, _canon(ls))
    # scipy numbers components in ascending order of their min linear index
    order = np.argsort(np.unique(lab[lab > 0]))
    assert np.array_equal(order, np.arange(len(order)))


def test_ccl_edge_cases():
    for fg in [np.zeros((5, 7), np.uint8), np.ones((5, 7), np.uint8),
               np.indices((9, 9)).sum(0) % 2, np.zeros((0, 0), np.uint8)]:
        fg = fg.astype(np.uint8)
        if fg.size == 0:
            continue
        lab, n = oracle.ccl(fg, 8)
        ls, ns = ndi.label(fg, structure=np.ones((3, 3)))
        assert n == ns and np.array_equal(lab, _canon(ls))
    # checkerboard: one 8-component, many 4-components
    cb = (np.indices((9, 9)).sum(0) % 2 == 0).astype(np.uint8)
    assert oracle.ccl(cb, 8)[1] == 1
    assert oracle.ccl(cb, 4)[1] == int(cb.sum())


@settings(max_examples=50, deadline=None)
@given(h=st.integers(1, 40), w=st.integers(1, 40), seed=st.integers(0, 2**31 - 1),
       amin=st.integers(1, 10), span=st.integers(0, 30))
def test_area_threshold_and_bwlabel(h, w, seed, amin, span):
    fg = (np.random.default_rng(seed).random((h, w)) < 0.45).astype(np.uint8)
    amax = amin + span
    ls, ns = ndi.label(fg, structure=np.ones((3, 3)))
    areas = np.bincount(ls.ravel(), minlength=ns + 1)
    keep = (areas >= amin) & (areas <= amax)
    keep[0] = False
    exp = keep[ls]
    assert np.array_equal(oracle.area_threshold(fg, amin, amax), exp.astype(np.uint8))
    lab, n = oracle.bwlabel(fg, amin, amax)
    assert n == int(keep.sum())
    assert np.array_equal(lab, np.where(exp, _canon(ls), 0))


def test_rbc_against_scipy(tile512):
    _, fl, _ = oracle.cd(tile512)
    lo = (fl & oracle.FLAG_RBC_LO) > 0
    hi = (fl & oracle.FLAG_RBC_HI) > 0
    ls, _ = ndi.label(lo, structure=np.ones((3, 3)))
    hit = np.unique(ls[hi & lo])
    exp = np.isin(ls, hit[hit > 0]) & ((fl & oracle.FLAG_R_GT_B) > 0)
    got = oracle.rbc(fl)
    assert np.array_equal(got, exp.astype(np.uint8))
    assert got.sum() > 0  # the generator paints red blood cells


@settings(max_examples=60, deadline=None)
@given(h=st.integers(1, 30), w=st.integers(1, 30), seed=st.integers(0, 2**31 - 1),
       dens=st.floats(0.2, 0.9))
def test_fill_holes_against_scipy(h, w, seed, dens):
    big0 = (np.random.default_rng(seed).random((h, w)) < dens).astype(np.uint8)
    F = oracle.fill_holes(big0)
    assert np.array_equal(F, ndi.binary_fill_holes(big0).astype(np.uint8))
    assert np.all(F >= big0)
    lb, nb = ndi.label(F == 0)  # cross structure = 4-connectivity
    border = np.zeros_like(F, bool)
    border[0, :] = border[-1, :] = border[:, 0] = border[:, -1] = True
    for k in range(1, nb + 1):
        assert (border & (lb == k)).any()


def test_fill_holes_diagonal_gap():
    # a hole whose only exit is diagonal is still a hole under 4-connected background
    big0 = np.zeros((7, 7), np.uint8)
    big0[1:6, 1:6] = 1
    big0[3, 3] = 0
    big0[2, 2] = 0  # diagonal neighbour, still enclosed
    F = oracle.fill_holes(big0)
    assert F[3, 3] == 1 and F[2, 2] == 1


def _edt_brute(F):
    bg = np.argwhere(F == 0)
    d2 = np.zeros(F.shape, np.int64)
    for y, x in np.argwhere(F != 0):
        d2[y, x] = ((bg - [y, x]) ** 2).sum(1).min()
    return d2


@settings(max_examples=80, deadline=None)
@given(h=st.integers(1, 24), w=st.integers(1, 24), seed=st.integers(0, 2**31 - 1),
       dens=st.floats(0.3, 0.98))
def test_edt_brute_force(h, w, seed, dens):
    F = (np.random.default_rng(seed).random((h, w)) < dens).astype(np.uint8)
    d2, dist = oracle.edt(F)
    if (F == 0).any():
        assert np.array_equal(d2.astype(np.int64), _edt_brute(F))
        assert np.array_equal(dist, np.sqrt(d2.astype(np.float32)))
    else:
        assert np.all(np.isinf(dist)) and np.all(d2 == np.iinfo(np.uint32).max)


def test_edt_against_scipy_and_cv2():
    rng = np.random.default_rng(11)
    F = (ndi.gaussian_filter(rng.random((300, 280)), 6) > 0.5).astype(np.uint8)
    d2, dist = oracle.edt(F)
    e = ndi.distance_transform_edt(F)
    assert np.array_equal(np.rint(e * e).astype(np.int64), d2.astype(np.int64))
    c = cv2.distanceTransform(F, cv2.DIST_L2, cv2.DIST_MASK_PRECISE)
    assert np.max(np.abs(c - dist)) < 1e-3


def test_edt_no_background():
    d2, dist = oracle.edt(np.ones((5, 9), np.uint8))
    assert np.all(np.isinf(dist))
