"""IWPP stress inputs (BASELINE.json configs[4]).

1-px corridors separated by 1-px walls, either a boustrophedon serpentine or a square
spiral, so that the corridor is one dependency chain of about 0.5*N pixels.
  binary: mask = 255 on the corridor, 0 on the walls;
  ramp:   mask = 255 - floor(254*k/L) along the path index k (L = path length).
The marker is the mask value at the path start and 0 elsewhere, so the expected
reconstruction equals the mask (a property every correct MR must reproduce).
"""
from __future__ import annotations

import numpy as np


def _serpentine_path(h, w):
    ys, xs = [], []
    for i, y in enumerate(range(0, h, 2)):
        row = np.arange(w) if i % 2 == 0 else np.arange(w - 1, -1, -1)
        ys.append(np.full(w, y))
        xs.append(row)
        if y + 2 < h:  # connector through the wall at the row end
            ys.append(np.array([y + 1]))
            xs.append(np.array([row[-1]]))
    return np.concatenate(ys), np.concatenate(xs)


def _spiral_path(h, w):
    ys, xs = [np.array([0])], [np.array([0])]
    y = x = 0
    top, bottom, left, right = 0, h - 1, 0, w - 1
    while True:
        moved = False
        if x < right:
            xs.append(np.arange(x + 1, right + 1)); ys.append(np.full(right - x, y))
            x = right; moved = True
        top += 2
        if y < bottom:
            ys.append(np.arange(y + 1, bottom + 1)); xs.append(np.full(bottom - y, x))
            y = bottom; moved = True
        right -= 2
        if x > left:
            xs.append(np.arange(x - 1, left - 1, -1)); ys.append(np.full(x - left, y))
            x = left; moved = True
        bottom -= 2
        if y > top:
            ys.append(np.arange(y - 1, top - 1, -1)); xs.append(np.full(y - top, x))
            y = top; moved = True
        left += 2
        if not moved or top > bottom or left > right:
            break
    return np.concatenate(ys), np.concatenate(xs)


def make_stress(kind: str, size: int = 4096, ramp: bool = False):
    """Return (marker u8[size,size], mask u8[size,size], path_len)."""
    if kind == "serpentine":
        py, px = _serpentine_path(size, size)
    elif kind == "spiral":
        py, px = _spiral_path(size, size)
    else:
        raise ValueError(kind)
    L = py.size
    mask = np.zeros((size, size), dtype=np.uint8)
    if ramp:
        k = np.arange(L, dtype=np.int64)
        mask[py, px] = (255 - (254 * k) // L).astype(np.uint8)
    else:
        mask[py, px] = 255
    marker = np.zeros_like(mask)
    marker[py[0], px[0]] = mask[py[0], px[0]]
    return marker, mask, L
