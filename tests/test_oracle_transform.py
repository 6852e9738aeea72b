"""Pins for oracle steps O0-O3 (thresholds, origin snap, affine, transform).

PAPER.md P:81 (origin an integer multiple of the resolution), P:75 (map
centred on the vehicle), P:105 (transform into the map frame).  Pins are
closed forms with exactly representable values (SURVEY.md 8(c) "Pins").
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_thresholds_G3():
    g = json.load(open(os.path.join(GOLD, "G3_column.json")))
    d = g["defaults"]
    T = O.thresholds(g["res"], d["min_obstacle_height"], d["max_obstacle_height"],
                     d["density_threshold"], d["neg_obs_threshold"])
    t = g["thresholds"]
    assert list(T) == [t["T_lo"], t["T_hi"], t["tau"], t["T_neg"]]


@pytest.mark.parametrize("p,expect", [
    # vehicle at 0 -> origin (-51.2, -51.2, -12.8) m = (-128, -128, -32) voxels
    ((0.0, 0.0, 0.0), (-128, -128, -32)),
    # 0.13 m rounds to the same multiple of 0.4
    ((0.13, 0.0, 0.0), (-128, -128, -32)),
    # ties (x.5) round up (reading A3): -3/0.4 = -7.5 -> -7
    ((10.0, -3.0, 1.0), (25 - 128, -7 - 128, 3 - 32)),
])
def test_snap_origin_examples(p, expect):
    o = O.snap_origin(256, 256, 64, 0.4, 0.5, p)
    assert tuple(o) == expect


def test_snap_origin_centres_vehicle():
    # property: the vehicle is within half a voxel of the grid centre
    rs = np.random.default_rng(3)
    for _ in range(500):
        p = rs.uniform(-1000, 1000, size=3)
        res = float(rs.choice([0.1, 0.2, 0.25, 0.4]))
        dims = (int(rs.choice([64, 256, 512])), int(rs.choice([64, 256])), int(rs.choice([16, 64])))
        o = O.snap_origin(*dims, res, 0.5, p)
        centre = o + np.array([dims[0] // 2, dims[1] // 2, dims[2] // 2])
        assert np.all(np.abs(p / res - centre) <= 0.5 + 1e-9)


def _pose(R, t):
    P = np.zeros((3, 4))
    P[:, :3] = R
    P[:, 3] = t
    return P


def test_affine_identity_translation():
    A, b = O.affine(_pose(np.eye(3), (1.0, 2.0, 3.0)), 1.0, np.zeros(3, np.int64))
    assert np.array_equal(A, np.eye(3, dtype=np.float32).reshape(9))
    assert np.array_equal(b, np.array([1, 2, 3], np.float32))
    # translation (1,2,3) of a point -> +(1,2,3); (0,0,0) itself is a no-return
    ok, g = O.transform_point(A, b, 0.5, 0.0, 0.0)
    assert ok and np.array_equal(g, np.array([1.5, 2.0, 3.0], np.float32))
    ok, _ = O.transform_point(A, b, 0.0, 0.0, 0.0)
    assert not ok


def test_affine_folds_resolution_and_origin():
    # b = t/res - o, A = R/res (reading A4) with exactly representable values
    o = np.array([-128, -100, -32], np.int64)
    A, b = O.affine(_pose(np.eye(3), (2.5, -1.25, 0.75)), 0.25, o)
    assert np.array_equal(A, (4 * np.eye(3, dtype=np.float32)).reshape(9))
    assert np.array_equal(b, np.array([10 + 128, -5 + 100, 3 + 32], np.float32))


def test_yaw90_is_exact_permutation():
    # 90 deg yaw maps (1,0,0) -> (0,1,0); with exact 0/+-1 entries the
    # result is a bit-exact permutation of the scaled inputs.
    R = np.array([[0.0, -1.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 1.0]])
    A, b = O.affine(_pose(R, (0.0, 0.0, 0.0)), 0.25, np.zeros(3, np.int64))
    ok, g = O.transform_point(A, b, 1.0, 0.0, 0.0)
    assert ok and np.array_equal(g, np.array([0.0, 4.0, 0.0], np.float32))
    rs = np.random.default_rng(0)
    for _ in range(1000):
        x, y, z = rs.uniform(-50, 50, size=3).astype(np.float32)
        ok, g = O.transform_point(A, b, x, y, z)
        assert ok
        assert g[0] == np.float32(-4) * y and g[1] == np.float32(4) * x and g[2] == np.float32(4) * z


def test_transform_matches_exact_rational_when_representable():
    # Points on a 1/8 lattice, entries powers of two: every f32 op is exact, so
    # g equals the exact affine map computed in float64.
    rs = np.random.default_rng(1)
    R = np.eye(3)[[1, 2, 0]] * np.array([1, -1, 1])[:, None]
    t = np.array([3.5, -2.25, 1.0])
    o = np.array([-40, -30, -8], np.int64)
    A, b = O.affine(_pose(R, t), 0.5, o)
    for _ in range(500):
        p = rs.integers(-400, 400, size=3) / 8.0
        if not p.any():
            continue
        ok, g = O.transform_point(A, b, *p.astype(np.float32))
        exact = R @ p / 0.5 + t / 0.5 - o
        assert ok and np.array_equal(g.astype(np.float64), exact)


@pytest.mark.parametrize("pt", [(math.nan, 0, 0), (math.inf, 1, 1), (1, -math.inf, 0),
                                (0.0, 0.0, 0.0)])
def test_invalid_points(pt):
    A, b = O.affine(_pose(np.eye(3), (0.5, 0.5, 0.5)), 1.0, np.zeros(3, np.int64))
    ok, _ = O.transform_point(A, b, *pt)
    assert not ok


def test_out_of_range_points_invalid():
    # reading A5: |g_i| >= 2^22 voxels is dropped
    A, b = O.affine(_pose(np.eye(3), (0.0, 0.0, 0.0)), 1.0, np.zeros(3, np.int64))
    ok, _ = O.transform_point(A, b, 4194303.0, 0.0, 1.0)
    assert ok
    ok, _ = O.transform_point(A, b, 4194304.0, 0.0, 1.0)
    assert not ok
    ok, _ = O.transform_point(A, b, 1.0, -4194304.0, 1.0)
    assert not ok
