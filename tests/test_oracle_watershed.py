"""Pins of the oracle's S8 markers (h-maxima + RMAX) and S9 watershed
(the order-independent W1-W3 definition).

Pinned against: brute force on tiny inputs -- h-maxima as the fixed point of iterated
mask-capped dilation, RMAX by explicit flat-zone enumeration, W1 by a widest-path (maximin)
Dijkstra from the markers, W2 and W3 by Bellman-Ford style relaxation of their defining
equations to stability -- plus hand-drawn cases (two overlapping disks, a rectangle, a
dumbbell) and structural invariants.
"""
import heapq

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st
from scipy import ndimage as ndi

import oracle

N8 = [(-1, -1), (0, -1), (1, -1), (-1, 0), (1, 0), (-1, 1), (0, 1), (1, 1)]


def _nbrs(F, y, x):
    h, w = F.shape
    for dx, dy in N8:
        qy, qx = y + dy, x + dx
        if 0 <= qy < h and 0 <= qx < w and F[qy, qx]:
            yield qy, qx


def _brute_markers(dist, F, hh=1.0):
    h, w = F.shape
    NEG = -np.inf
    J = np.where(F > 0, (dist - np.float32(hh)).astype(np.float32), NEG).astype(np.float32)
    mk = np.where(F > 0, dist, NEG).astype(np.float32)
    J = np.minimum(J, mk)
    while True:
        d = ndi.grey_dilation(J, size=(3, 3), mode="constant", cval=-np.inf)
        nxt = np.where(F > 0, np.maximum(J, np.minimum(d, mk)), NEG).astype(np.float32)
        if np.array_equal(nxt, J):
            break
        J = nxt
    M = np.zeros(F.shape, bool)
    for v in np.unique(J[F > 0]):
        zl, nz = ndi.label((F > 0) & (J == v), structure=np.ones((3, 3)))
        for k in range(1, nz + 1):
            zone = zl == k
            ring = ndi.binary_dilation(zone, structure=np.ones((3, 3))) & ~zone & (F > 0)
            if not (J[ring] > v).any():
                M |= zone
    return J, M


def _brute_watershed(dist, ML, F):
    h, w = F.shape
    # W1: widest path from the markers
    c = np.full(F.shape, -np.inf, np.float32)
    heap = []
    for y, x in np.argwhere((F > 0) & (ML != 0)):
        c[y, x] = dist[y, x]
        heap.append((-float(c[y, x]), y, x))
    heapq.heapify(heap)
    done = np.zeros(F.shape, bool)
    while heap:
        nv, y, x = heapq.heappop(heap)
        if done[y, x]:
            continue
        done[y, x] = True
        for qy, qx in _nbrs(F, y, x):
            cand = min(-nv, float(dist[qy, qx]))
            if cand > c[qy, qx]:
                c[qy, qx] = cand
                heapq.heappush(heap, (-cand, qy, qx))
    # W2: least fixed point by relaxation from +inf
    INF = 10 ** 9
    d = np.full(F.shape, INF, np.int64)
    pix = [tuple(p) for p in np.argwhere(F > 0)]
    fixed = {}
    for (y, x) in pix:
        if ML[y, x] != 0:
            fixed[(y, x)] = 0
        elif any(c[q] > c[y, x] for q in _nbrs(F, y, x)):
            fixed[(y, x)] = 1
    for k, v in fixed.items():
        d[k] = v
    changed = True
    while changed:
        changed = False
        for (y, x) in pix:
            if (y, x) in fixed:
                continue
            best = min([d[q] for q in _nbrs(F, y, x) if c[q] == c[y, x]] + [INF - 1]) + 1
            if best < d[y, x]:
                d[y, x] = best
                changed = True
    # W3: relaxation of L(p) = min over argmin_{c(q) >= c(p)} (-c(q), d(q)) of L(q)
    L = np.where((F > 0) & (ML != 0), ML, INF).astype(np.int64)
    changed = True
    while changed:
        changed = False
        for (y, x) in pix:
            if ML[y, x] != 0:
                continue
            cands = [q for q in _nbrs(F, y, x) if c[q] >= c[y, x]]
            if not cands:
                continue
            key = min((-float(c[q]), int(d[q])) for q in cands)
            v = min(L[q] for q in cands if (-float(c[q]), int(d[q])) == key)
            if v < L[y, x]:
                L[y, x] = v
                changed = True
    split = np.zeros(F.shape, np.uint8)
    for (y, x) in pix:
        split[y, x] = 0 if any(L[q] < L[y, x] for q in _nbrs(F, y, x)) else 1
    return c, d, L, split


def _blob_F(seed, h, w):
    rng = np.random.default_rng(seed)
    F = np.zeros((h, w), np.uint8)
    for _ in range(rng.integers(1, 4)):
        cy, cx, r = rng.uniform(0, h), rng.uniform(0, w), rng.uniform(2, 7)
        yy, xx = np.mgrid[:h, :w]
        F |= ((yy - cy) ** 2 + (xx - cx) ** 2 <= r * r).astype(np.uint8)
    return F


@settings(max_examples=40, deadline=None)
@given(h=st.integers(3, 24), w=st.integers(3, 24), seed=st.integers(0, 2**31 - 1),
       hh=st.sampled_from([0.5, 1.0, 2.0]))
def test_markers_brute(h, w, seed, hh):
    F = _blob_F(seed, h, w)
    _, dist = oracle.edt(F)
    ML, J, n = oracle.markers(dist, F, hh)
    Jb, Mb = _brute_markers(dist, F, hh)
    assert np.array_equal(J[F > 0], Jb[F > 0])
    assert np.array_equal(ML > 0, Mb)
    ls, ns = ndi.label(Mb, structure=np.ones((3, 3)))
    assert n == ns
    # every component of F contains at least one marker
    lf, nf = ndi.label(F, structure=np.ones((3, 3)))
    for k in range(1, nf + 1):
        assert (ML[lf == k] > 0).any()


@settings(max_examples=40, deadline=None)
@given(h=st.integers(3, 24), w=st.integers(3, 24), seed=st.integers(0, 2**31 - 1))
def test_watershed_brute(h, w, seed):
    F = _blob_F(seed, h, w)
    _, dist = oracle.edt(F)
    ML, _, _ = oracle.markers(dist, F, 1.0)
    split, c, d, L = oracle.watershed(dist, ML, F)
    cb, db, Lb, sb = _brute_watershed(dist, ML, F)
    m = F > 0
    assert np.array_equal(c[m], cb[m])
    assert np.array_equal(d[m].astype(np.int64), db[m])
    assert np.array_equal(L[m].astype(np.int64), Lb[m])
    assert np.array_equal(split, sb)
    _check_invariants(F, ML, L, split)


def _check_invariants(F, ML, L, split):
    m = F > 0
    assert np.all(L[m] > 0) and np.all(L[m] < 2**31 - 1)      # every F pixel is labelled
    for lab in np.unique(L[m]):
        region = (L == lab) & m
        assert (ML[region] == lab).any()                      # contains its marker
        _, nr = ndi.label(region, structure=np.ones((3, 3)))
        assert nr == 1                                        # 8-connected
    # no 8-adjacency between different labels after line removal
    Ls = np.where(split > 0, L, 0).astype(np.int64)
    h, w = F.shape
    for dx, dy in N8:
        a = Ls[max(0, -dy):h - max(0, dy), max(0, -dx):w - max(0, dx)]
        b = Ls[max(0, dy):h - max(0, -dy) or None, max(0, dx):w - max(0, -dx) or None]
        both = (a > 0) & (b > 0)
        assert np.all(a[both] == b[both])


def _pipeline_from_F(F):
    _, dist = oracle.edt(F)
    ML, _, nm = oracle.markers(dist, F, 1.0)
    split, c, d, L = oracle.watershed(dist, ML, F)
    lab, n = oracle.ccl(split, 8)
    return n, split, L, ML


def test_two_overlapping_disks():
    yy, xx = np.mgrid[:40, :60]
    F = (((yy - 20) ** 2 + (xx - 20) ** 2 <= 100) | ((yy - 20) ** 2 + (xx - 36) ** 2 <= 100))
    n, split, L, ML = _pipeline_from_F(F.astype(np.uint8))
    assert n == 2
    cols = np.where((F > 0).any(0) & ~(split > 0).all(0, where=F > 0))[0]
    assert 26 <= cols.min() and cols.max() <= 30   # the line sits near the bisector x = 28


def test_rectangle_and_dumbbell():
    F = np.zeros((30, 40), np.uint8)
    F[5:25, 5:35] = 1
    assert _pipeline_from_F(F)[0] == 1
    yy, xx = np.mgrid[:30, :60]
    D = ((yy - 15) ** 2 + (xx - 12) ** 2 <= 81) | ((yy - 15) ** 2 + (xx - 47) ** 2 <= 81)
    D |= (abs(yy - 15) <= 1) & (xx >= 12) & (xx <= 47)
    assert _pipeline_from_F(D.astype(np.uint8))[0] == 2


def test_watershed_order_independent_on_ties():
    # plateau-heavy input: integer distances on an axis-aligned cross; compare to brute force
    F = np.zeros((21, 21), np.uint8)
    F[8:13, :] = 1
    F[:, 8:13] = 1
    _, dist = oracle.edt(F)
    ML, _, _ = oracle.markers(dist, F, 1.0)
    split, c, d, L = oracle.watershed(dist, ML, F)
    cb, db, Lb, sb = _brute_watershed(dist, ML, F)
    assert np.array_equal(split, sb)
    _check_invariants(F, ML, L, split)
