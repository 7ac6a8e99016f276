"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This package holds NO arithmetic of the method (no deconvolution, no thresholds, no
morphology).  It only paints H&E-like RGB tiles from a physical stain-absorption model
and draws IWPP stress masks.  Both sides of every parity test consume its output.
"""
from .hne import make_tile, make_pool_seed, TileSpec  # noqa: F401
from .stress import make_stress  # noqa: F401
