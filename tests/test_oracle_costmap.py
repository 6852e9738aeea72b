"""Pins for the costmap ("each of the
output maps get some weight assigned to them and the resulting per pixel sum
is the cost in that pixel").  Closed form on hand-made layers, including the
reading B5 rules (NaN layers contribute 0; 'unknown' = undefined height that
is not a negative obstacle) and linearity in the weights."""
import math

import numpy as np

from oracle import oracle as O


def _layers():
    nan = math.nan
    f = lambda v: np.array([v], np.float32)  # noqa: E731
    u = lambda v: np.array([v], np.uint8)  # noqa: E731
    # cells: defined flat / hard obstacle / soft obstacle / undefined unknown / negative
    height = np.array([[1.0, 1.5, 0.5, nan, nan]], np.float32)
    density = np.array([[0.0, 0.9, 0.2, nan, nan]], np.float32)
    hard = np.array([[0, 1, 0, 0, 0]], np.uint8)
    soft = np.array([[0, 0, 1, 0, 0]], np.uint8)
    neg = np.array([[0, 0, 0, 0, 1]], np.uint8)
    slope = np.array([[0.1, 0.5, nan, nan, nan]], np.float32)
    rough = np.array([[0.01, nan, 0.02, nan, nan]], np.float32)
    del f, u
    return O.Layers(height, density, hard, soft, neg, slope, rough, None, None)


def test_costmap_closed_form():
    L = _layers()
    w = [10.0, 3.0, 2.0, 7.0, 1.0, 5.0, 0.5]
    c = O.costmap(L, w)[0]
    exp = [
        2.0 * 0.0 + 1.0 * 0.1 + 5.0 * 0.01,
        10.0 + 2.0 * 0.9 + 1.0 * 0.5,
        3.0 + 2.0 * 0.2 + 5.0 * 0.02,
        0.5,
        7.0,
    ]
    assert np.allclose(c, np.array(exp, np.float32), rtol=1e-6, atol=1e-6)


def test_costmap_linear_in_weights_and_zero():
    L = _layers()
    rs = np.random.default_rng(0)
    w1 = rs.uniform(0, 5, 7)
    w2 = rs.uniform(0, 5, 7)
    c1, c2, c12 = O.costmap(L, w1), O.costmap(L, w2), O.costmap(L, w1 + w2)
    assert np.allclose(c12, c1 + c2, rtol=1e-5, atol=1e-5)
    assert np.all(O.costmap(L, np.zeros(7)) == 0)
    # one-hot weights pick single layers (NaN -> 0)
    for i, name in enumerate(["hard", "soft", "density", "neg", "slope", "roughness"]):
        e = np.zeros(7)
        e[i] = 1.0
        ref = np.nan_to_num(getattr(L, name).astype(np.float32), nan=0.0)
        assert np.array_equal(O.costmap(L, e), ref)
