"""Seeded synthetic H&E-like RGB tissue tiles (input recipe).

The recipe follows SURVEY.md §8(d) "Synthetic H&E-like generator":
  1. tissue mask: smooth noise thresholded to a tissue fraction t;
  2. stroma: smooth eosin/haematoxylin density fields;
  3. nuclei: Poisson count (density rho per tissue pixel), ellipses with semi-axes
     U[3,8] px, 15% overlapping pairs, 10% vesicular (pale core), chromatin noise;
  4. red blood cells: small discs of saturated red;
  5. composition by Beer-Lambert absorption plus sensor noise N(0, 2), rounded to u8.

This is a PAINTER, not part of the method: its stain colours are its own physical
model (generic haematoxylin / eosin absorbances), deliberately not the deconvolution
matrix either side of the parity tests uses.  Everything is drawn from
numpy.random.default_rng(seed); the same seed gives the same bytes on any host.
"""
from __future__ import annotations

import dataclasses
import hashlib

import numpy as np

# Painter absorbances (optical density per unit stain) for the R, G, B channels.
_PAINT_H = np.array([0.65, 0.70, 0.29], dtype=np.float64)
_PAINT_E = np.array([0.07, 0.99, 0.11], dtype=np.float64)


@dataclasses.dataclass(frozen=True)
class TileSpec:
    height: int = 4096
    width: int = 4096
    tissue_frac: float = 1.0
    density: float = 1.15e-4      # nuclei per tissue pixel (~30 on 512^2, ~1900 on 4K)
    pair_frac: float = 0.15
    vesicular_frac: float = 0.10
    rbc_rel_density: float = 0.10
    noise_sigma: float = 2.0


def make_pool_seed(slide: int, idx: int) -> int:
    """Tile id -> 63-bit seed (stable across hosts/Python versions)."""
    h = hashlib.blake2b(f"{slide}:{idx}".encode(), digest_size=8).digest()
    return int.from_bytes(h, "little") & ((1 << 63) - 1)


def _smooth_field(rng, h, w, scale):
    """Uniform noise at 1/scale resolution, bilinearly upsampled and normalised to [0,1]."""
    import cv2
    lh, lw = max(2, h // scale + 2), max(2, w // scale + 2)
    low = rng.random((lh, lw), dtype=np.float32)
    f = cv2.resize(low, (w, h), interpolation=cv2.INTER_LINEAR)
    lo, hi = float(f.min()), float(f.max())
    return (f - lo) * np.float32(1.0 / max(hi - lo, 1e-12))


def _paint_ellipse(ch, cx, cy, a, b, theta, value, noise_rng, noise_sigma, mode="max"):
    h, w = ch.shape
    r = int(np.ceil(max(a, b))) + 1
    x0, x1 = max(0, int(cx) - r), min(w, int(cx) + r + 1)
    y0, y1 = max(0, int(cy) - r), min(h, int(cy) + r + 1)
    if x0 >= x1 or y0 >= y1:
        return None
    yy, xx = np.mgrid[y0:y1, x0:x1]
    dx = xx - cx
    dy = yy - cy
    ct, st = np.cos(theta), np.sin(theta)
    u = (dx * ct + dy * st) / a
    v = (-dx * st + dy * ct) / b
    inside = (u * u + v * v) <= 1.0
    if not inside.any():
        return None
    sub = ch[y0:y1, x0:x1]
    vals = value + noise_rng.normal(0.0, noise_sigma, size=inside.sum())
    if mode == "max":
        sub[inside] = np.maximum(sub[inside], vals)
    else:
        sub[inside] = vals
    return (y0, y1, x0, x1, inside)


def make_tile(seed: int, spec: TileSpec = TileSpec()) -> dict:
    """Return {'rgb': uint8[H, W, 3] (C-contiguous, R,G,B interleaved), 'nuclei': [...]}."""
    rng = np.random.default_rng(seed)
    h, w = spec.height, spec.width

    # 1. tissue mask
    if spec.tissue_frac >= 1.0:
        tissue = np.ones((h, w), dtype=bool)
    else:
        f = _smooth_field(rng, h, w, 64)
        thr = np.quantile(f, 1.0 - spec.tissue_frac)
        tissue = f >= thr

    # 2. stroma
    s1 = _smooth_field(rng, h, w, 8)
    s2 = _smooth_field(rng, h, w, 8)
    c_e = np.where(tissue, np.float32(0.25) + np.float32(0.25) * s1, np.float32(0.0))
    c_h = np.where(tissue, np.float32(0.04) + np.float32(0.04) * s2, np.float32(0.0))

    # 3. nuclei
    n_tissue = int(tissue.sum())
    n_nuc = int(rng.poisson(spec.density * n_tissue)) if n_tissue else 0
    nuclei = []
    if n_nuc:
        ty, tx = np.nonzero(tissue) if spec.tissue_frac < 1.0 else (None, None)
        for _ in range(n_nuc):
            if ty is None:
                cy, cx = rng.uniform(0, h), rng.uniform(0, w)
            else:
                k = rng.integers(0, n_tissue)
                cy, cx = ty[k] + rng.uniform(), tx[k] + rng.uniform()
            a, b = rng.uniform(3, 8), rng.uniform(3, 8)
            theta = rng.uniform(0, np.pi)
            shapes = [(cx, cy, a, b, theta)]
            if rng.random() < spec.pair_frac:
                a2, b2 = rng.uniform(3, 8), rng.uniform(3, 8)
                dist = rng.uniform(0.6, 0.9) * (max(a, b) + max(a2, b2))
                phi = rng.uniform(0, 2 * np.pi)
                shapes.append((cx + dist * np.cos(phi), cy + dist * np.sin(phi), a2, b2,
                               rng.uniform(0, np.pi)))
            for (ex, ey, ea, eb, et) in shapes:
                val = rng.uniform(0.6, 1.1)
                _paint_ellipse(c_h, ex, ey, ea, eb, et, val, rng, 0.05, "max")
                # nuclei carry little eosin
                _paint_ellipse(c_e, ex, ey, ea, eb, et, 0.08, rng, 0.0, "set")
                if rng.random() < spec.vesicular_frac:
                    _paint_ellipse(c_h, ex, ey, 0.4 * ea, 0.4 * eb, et, 0.3 * val, rng, 0.0, "set")
                nuclei.append((ex, ey, ea, eb, et))

    # 5. compose (Beer-Lambert) + sensor noise
    od = c_h[..., None] * _PAINT_H.astype(np.float32) + c_e[..., None] * _PAINT_E.astype(np.float32)
    img = np.float32(255.0) * np.exp(od * np.float32(-np.log(10.0)))
    del od
    img += np.float32(spec.noise_sigma) * rng.standard_normal(size=img.shape, dtype=np.float32)

    # 4. red blood cells (painted over, saturated red)
    n_rbc = int(rng.poisson(spec.rbc_rel_density * spec.density * n_tissue)) if n_tissue else 0
    for _ in range(n_rbc):
        cy, cx = rng.uniform(0, h), rng.uniform(0, w)
        rad = rng.uniform(3, 4)
        col = (rng.normal(200, 10 / 3), rng.normal(30, 5 / 3), rng.normal(40, 5 / 3))
        r = int(np.ceil(rad)) + 1
        x0, x1 = max(0, int(cx) - r), min(w, int(cx) + r + 1)
        y0, y1 = max(0, int(cy) - r), min(h, int(cy) + r + 1)
        if x0 >= x1 or y0 >= y1:
            continue
        yy, xx = np.mgrid[y0:y1, x0:x1]
        inside = (xx - cx) ** 2 + (yy - cy) ** 2 <= rad * rad
        for ch in range(3):
            sub = img[y0:y1, x0:x1, ch]
            sub[inside] = col[ch] + rng.normal(0, 2.0, size=inside.sum())

    rgb = np.clip(np.rint(img), 0, 255).astype(np.uint8)
    return {"rgb": np.ascontiguousarray(rgb), "nuclei": nuclei, "n_rbc": n_rbc}


def make_config_tile(config: int, index: int = 0) -> np.ndarray:
    """The seeded inputs of BASELINE.json configs."""
    if config == 1:
        return make_tile(1, TileSpec(512, 512))["rgb"]
    if config == 2:
        return make_tile(2, TileSpec())["rgb"]
    if config == 3:
        return make_tile(1000 + (index % 64), TileSpec())["rgb"]
    if config == 4:
        slide, k = divmod(index, 108)
        srng = np.random.default_rng(make_pool_seed(slide, -1))
        dens = 1.15e-4 * srng.uniform(0.5, 2.0)
        trng = np.random.default_rng(make_pool_seed(slide, k))
        t = trng.uniform(0.3, 1.0)
        return make_tile(make_pool_seed(slide, k), TileSpec(tissue_frac=t, density=dens))["rgb"]
    raise ValueError(config)
