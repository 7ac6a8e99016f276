"""Pins of the oracle's per-image aggregation:
closed forms (constant rows -> std 0; a two-valued group {a, b} -> mean (a+b)/2, std |a-b|/2;
an arithmetic progression 0..n-1 -> std sqrt((n^2-1)/12)), empty groups -> NaN, and the
library special case numpy mean / std(ddof=0) on random rows."""
import numpy as np

import oracle


def test_closed_forms():
    n = 101
    feat = np.zeros((3 + 2 + n, 4), np.float32)
    feat[0:3] = [[7.5, -2.0, 0.0, 1e6]] * 3                      # constant group
    feat[3:5] = [[1.0, -4.0, 10.0, 0.0], [3.0, 6.0, 10.0, 2e6]]   # two values
    feat[5:] = np.arange(n, dtype=np.float32)[:, None]            # 0..n-1 in every column
    off = np.array([0, 3, 3, 5, 5 + n], np.int64)                  # group 1 is empty
    cnt, mean, std = oracle.aggregate(feat, off)
    assert list(cnt) == [3, 0, 2, n]
    assert np.array_equal(mean[0], [7.5, -2.0, 0.0, 1e6]) and np.array_equal(std[0], [0, 0, 0, 0])
    assert np.isnan(mean[1]).all() and np.isnan(std[1]).all()
    assert np.array_equal(mean[2], [2.0, 1.0, 10.0, 1e6])
    assert np.array_equal(std[2], [1.0, 5.0, 0.0, 1e6])
    assert np.allclose(mean[3], (n - 1) / 2, rtol=0, atol=1e-12)
    assert np.allclose(std[3], np.sqrt((n * n - 1) / 12.0), rtol=1e-14, atol=0)


def test_matches_numpy():
    rng = np.random.default_rng(3)
    sizes = [5, 1, 0, 400, 33]
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    feat = (rng.standard_normal((off[-1], 36)) * rng.uniform(0.1, 1e4, 36) + 1e3).astype(np.float32)
    cnt, mean, std = oracle.aggregate(feat, off)
    for g, n in enumerate(sizes):
        assert cnt[g] == n
        if n:
            f = feat[off[g]:off[g + 1]].astype(np.float64)
            assert np.allclose(mean[g], f.mean(axis=0), rtol=1e-13, atol=0)
            assert np.allclose(std[g], f.std(axis=0), rtol=1e-11, atol=1e-9)


def test_no_rows():
    cnt, mean, std = oracle.aggregate(np.zeros((0, 36), np.float32), np.zeros(3, np.int64))
    assert list(cnt) == [0, 0] and np.isnan(mean).all() and np.isnan(std).all()
