"""End-to-end sanity of the oracle on the config-1 tile (not parity: a plausibility check
that the segmentation finds the painted nuclei, "a set of features for
each segmented nucleus"), plus determinism (SPEC.md:316 pattern: byte-identical reruns)."""
import numpy as np

import oracle
from synth.hne import TileSpec, make_tile


def test_object_count_near_ground_truth():
    d = make_tile(1, TileSpec(512, 512))
    lab, rl, rf, ft = oracle.process_tile(d["rgb"])
    gt = len(d["nuclei"])
    assert abs(len(rl) - gt) <= max(3, 0.15 * gt), (len(rl), gt)
    assert np.all(ft[:, 0] >= 21) and np.all(ft[:, 0] <= 1000)   # S10 area bounds (C10)


def test_deterministic(tile512):
    a = oracle.process_tile(tile512)
    b = oracle.process_tile(tile512)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_background_tile_and_skip():
    white = np.full((64, 64, 3), 250, np.uint8)
    lab, rl, rf, ft = oracle.process_tile(white)
    assert len(rl) == 0 and not lab.any()
    p = oracle.default_params()
    p.bg_skip_frac = 0.5
    lab, n = oracle.segment_tile(white, p)
    assert n == 0
