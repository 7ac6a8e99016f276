"""Pins of the oracle's S11 features (reading C16/C17).

Pinned against: closed forms (a w x h rectangle; a constant-intensity object; a 2-level
checkerboard's GLCM), OpenCV's Sobel (CV_16S, REFLECT_101 -- the library the paper names)
for the gradient, and an independent numpy re-implementation of every feature.
The GLCM normalisation choices are our definitions (parity unpinned beyond the numpy
re-implementation and the closed forms).
"""
import math

import cv2
import numpy as np
import pytest
from scipy import ndimage as ndi

import oracle

RTOL, ATOL = 2e-6, 1e-6


def _np_features(labels, g):
    """Independent numpy implementation, one row per label in ascending order."""
    h, w = g.shape
    gx = cv2.Sobel(g, cv2.CV_32S if False else cv2.CV_16S, 1, 0, ksize=3).astype(np.int64)
    gy = cv2.Sobel(g, cv2.CV_16S, 0, 1, ksize=3).astype(np.int64)
    mag = np.sqrt((gx * gx + gy * gy).astype(np.float32)).astype(np.float64)
    rows = []
    cross = ndi.generate_binary_structure(2, 1)
    q = (g >> 5).astype(np.int64)
    edges = cv2.Canny(g, 100, 200) > 0   # reading C22: OpenCV's Canny itself
    for lab in np.unique(labels[labels > 0]):
        P = labels == lab
        ys, xs = np.nonzero(P)
        A = len(xs)
        inner = ndi.binary_erosion(P, structure=cross, border_value=0)
        perim = int((P & ~inner).sum())
        cx, cy = xs.mean(), ys.mean()
        bw, bh = xs.max() - xs.min() + 1, ys.max() - ys.min() + 1
        mu20 = ((xs - cx) ** 2).sum()
        mu02 = ((ys - cy) ** 2).sum()
        mu11 = ((xs - cx) * (ys - cy)).sum()
        cov = np.array([[mu20 / A + 1 / 12, mu11 / A], [mu11 / A, mu02 / A + 1 / 12]])
        l2, l1 = np.linalg.eigvalsh(cov)
        shape = [A, perim, cx, cy, bw, bh, 4 * math.sqrt(l1), 4 * math.sqrt(max(l2, 0)),
                 math.sqrt(1 - l2 / l1), 0.5 * math.atan2(2 * mu11, mu20 - mu02),
                 math.sqrt(4 * A / math.pi), 4 * math.pi * A / perim ** 2, A / (bw * bh)]
        v = g[P].astype(np.float64)
        mu, sd = v.mean(), v.std()
        _, cnt = np.unique(g[P], return_counts=True)
        pv = cnt / A
        med = np.sort(g[P])[(A + 1) // 2 - 1]
        inten = [mu, sd, v.min(), v.max(), med,
                 0.0 if sd == 0 else ((v - mu) ** 3).mean() / sd ** 3,
                 0.0 if sd == 0 else ((v - mu) ** 4).mean() / sd ** 4,
                 -(pv * np.log2(pv)).sum(), (pv * pv).sum()]
        m = mag[P]
        ms = m.std() if m.min() != m.max() else 0.0
        grad = [m.mean(), ms, 0.0 if ms == 0 else ((m - m.mean()) ** 3).mean() / ms ** 3,
                0.0 if ms == 0 else ((m - m.mean()) ** 4).mean() / ms ** 4]
        C = np.zeros((8, 8), np.int64)
        for dx, dy in [(1, 0), (1, 1), (0, 1), (-1, 1)]:
            a = P[max(0, -dy):h - max(0, dy), max(0, -dx):w - max(0, dx)]
            b = P[max(0, dy):h - max(0, -dy) or None, max(0, dx):w - max(0, -dx) or None]
            qa = q[max(0, -dy):h - max(0, dy), max(0, -dx):w - max(0, dx)]
            qb = q[max(0, dy):h - max(0, -dy) or None, max(0, dx):w - max(0, -dx) or None]
            both = a & b
            np.add.at(C, (qa[both], qb[both]), 1)
            np.add.at(C, (qb[both], qa[both]), 1)
        S = C.sum()
        if S == 0:
            tex = [0.0] * 8
        else:
            Pm = C / S
            i, j = np.indices((8, 8))
            mi, mj = (i * Pm).sum(), (j * Pm).sum()
            si, sj = math.sqrt(((i - mi) ** 2 * Pm).sum()), math.sqrt(((j - mj) ** 2 * Pm).sum())
            t = i + j - mi - mj
            nz = Pm > 0
            tex = [(Pm ** 2).sum(), ((i - j) ** 2 * Pm).sum(),
                   1.0 if si * sj == 0 else ((i - mi) * (j - mj) * Pm).sum() / (si * sj),
                   (Pm / (1 + (i - j) ** 2)).sum(), -(Pm[nz] * np.log2(Pm[nz])).sum(),
                   (t ** 3 * Pm).sum(), (t ** 4 * Pm).sum(), Pm.max()]
        border = xs.min() == 0 or ys.min() == 0 or xs.max() == w - 1 or ys.max() == h - 1
        ne = int(edges[P].sum())
        rows.append((lab, int(border), shape + inten + grad + tex + [ne, ne / A]))
    return rows


def _compare(labels, g):
    rl, rf, ft = oracle.features(labels, g)
    exp = _np_features(labels, g)
    assert len(exp) == len(rl)
    for k, (lab, border, vals) in enumerate(exp):
        assert rl[k] == lab and rf[k] == border
        e = np.array(vals, np.float64).astype(np.float32).astype(np.float64)
        got = ft[k].astype(np.float64)
        # skew/kurt are ill-conditioned at small variance: relative to the scale involved
        assert np.allclose(got, e, rtol=RTOL, atol=ATOL), (k, np.nonzero(~np.isclose(got, e, rtol=RTOL, atol=ATOL)), got, e)


def test_rectangle_closed_form():
    labels = np.zeros((20, 30), np.int32)
    labels[4:11, 6:19] = 4 * 30 + 6 + 1
    g = np.full((20, 30), 77, np.uint8)
    rl, rf, ft = oracle.features(labels, g)
    w, h = 13, 7
    f = ft[0]
    assert f[0] == w * h and f[1] == 2 * (w + h) - 4
    assert f[2] == pytest.approx(6 + (w - 1) / 2) and f[3] == pytest.approx(4 + (h - 1) / 2)
    assert f[4] == w and f[5] == h and f[12] == 1.0
    # regionprops convention: major = sqrt(12)*... for a rectangle lambda = w^2/12 exactly
    assert f[6] == pytest.approx(4 * math.sqrt(w * w / 12.0), rel=1e-6)
    assert f[7] == pytest.approx(4 * math.sqrt(h * h / 12.0), rel=1e-6)
    # constant intensity: std 0, entropy 0, ASM 1, contrast 0, homogeneity 1, correlation 1
    assert f[13] == 77 and f[14] == 0 and f[15] == 77 and f[16] == 77 and f[17] == 77
    assert f[18] == 0 and f[19] == 0 and f[20] == 0 and f[21] == 1
    assert f[26] == 1 and f[27] == 0 and f[28] == 1 and f[29] == 1 and f[30] == 0
    assert f[33] == 1
    assert rf[0] == 0


def test_checkerboard_glcm():
    labels = np.zeros((10, 10), np.int32)
    labels[1:9, 1:9] = 12
    yy, xx = np.indices((10, 10))
    g = np.where((yy + xx) % 2 == 0, 0, 255).astype(np.uint8)   # q in {0, 7}
    rl, rf, ft = oracle.features(labels, g)
    f = ft[0]
    # 8x8 object: horizontal+vertical pairs always differ (2*2*56 = 224 counts of (0,7)/(7,0)),
    # diagonal pairs always equal (2*2*49 = 196 counts on the diagonal)
    S = 224 + 196
    p_off = 224 / S
    assert f[27] == pytest.approx(49 * p_off, rel=1e-6)         # contrast = (7-0)^2 * P_off
    assert f[26] == pytest.approx(2 * (112 / S) ** 2 + 2 * (98 / S) ** 2, rel=1e-6)


def test_against_numpy_random_objects():
    rng = np.random.default_rng(3)
    g = rng.integers(0, 256, size=(64, 80)).astype(np.uint8)
    blobs = ndi.gaussian_filter(rng.random((64, 80)), 2.5) > 0.52
    lab, n = oracle.ccl(blobs.astype(np.uint8), 8)
    assert n > 3
    _compare(lab, g)


def test_against_numpy_on_pipeline(tile512):
    lab, n = oracle.segment_tile(tile512)
    g, _, _ = oracle.cd(tile512)
    assert n > 10
    _compare(lab, g)


@pytest.mark.parametrize("seed", range(6))
def test_canny_matches_opencv(seed):
    """The feature-stage Canny (reading C22) is OpenCV's: cv2.Canny(g, low, high), aperture 3,
    L1 norm -- on noise, blurred noise and random thresholds, bit for bit."""
    rng = np.random.default_rng(40 + seed)
    h, w = (int(v) for v in rng.integers(8, 160, 2))
    g = rng.integers(0, 256, size=(h, w)).astype(np.uint8)
    if seed % 2:
        g = cv2.GaussianBlur(g, (5, 5), 1.5)
    lo, hi = sorted(int(v) for v in rng.integers(0, 600, 2))
    assert np.array_equal(oracle.canny(g, lo, hi), (cv2.Canny(g, lo, hi) > 0).astype(np.uint8))


def test_canny_on_tile_and_step(tile512):
    g, _, _ = oracle.cd(tile512)
    e = oracle.canny(g)
    assert np.array_equal(e, (cv2.Canny(g, 100, 200) > 0).astype(np.uint8)) and e.sum() > 100
    # a vertical step of height 60: |dx| = 240 > high on columns 7 and 8; the suppression's
    # m > left, m >= right keeps the last dark column only
    step = np.zeros((12, 16), np.uint8)
    step[:, 8:] = 60
    e = oracle.canny(step)
    assert e[:, 7].all() and e.sum() == 12
    step[:, 8:] = 40                      # |dx| = 160 < high: no strong pixel, no edges
    assert oracle.canny(step).sum() == 0


def test_sobel_reflect101_matches_cv2():
    # a 1-object image covering everything: gradient mean must use REFLECT_101 at the edges
    rng = np.random.default_rng(9)
    g = rng.integers(0, 256, size=(7, 9)).astype(np.uint8)
    labels = np.ones((7, 9), np.int32)
    _compare(labels, g)
