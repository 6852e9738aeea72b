"""Pins for oracle step O5 (ray traversal, "the lidar rays are
traced"; miss definition P:81 "passed though the voxel but did not end in it").

- brute force: exact segment/voxel interval intersection on tiny grids
  (tests/brute.py), near-ties (crossing gap < 1e-5) excluded;
- special case: the axis-aligned 10-voxel ray of SPEC S:151;
- invariants on long rays in a 1024x1024x128 grid: 6-connected, monotone per
  axis, length = sum |E - S| when E is in the grid, never leaves bbox(S, E);
- golden G1 walks.
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests import brute

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_axis_aligned_ten_voxels():
    w = O.traverse((16, 4, 4), (0.5, 0.5, 0.5), (10.5, 0.5, 0.5))
    assert w.tolist() == [[x, 0, 0] for x in range(10)]


def test_same_voxel_no_miss():
    w = O.traverse((8, 8, 8), (0.5, 0.5, 0.5), (0.75, 0.25, 0.9))
    assert w.shape[0] == 0


def test_golden_G1_walks():
    g = json.load(open(os.path.join(GOLD, "G1_integrate.json")))
    for p, walk in zip(g["points_world"], g["walks"]):
        w = O.traverse(tuple(g["dims"]), g["sensor"], p)
        assert w.tolist() == walk


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_dda_matches_exact_geometry(seed):
    rs = np.random.default_rng(seed)
    dims = (8, 8, 8)
    checked = 0
    for _ in range(1000):
        s = rs.uniform(0.0, 8.0, size=3).astype(np.float32)
        g = rs.uniform(-4.0, 12.0, size=3).astype(np.float32)
        if brute.near_tie(s, g):
            continue
        walk = O.traverse(dims, s, g)
        got = {tuple(v) for v in walk.tolist()}
        assert len(got) == walk.shape[0], "a voxel was visited twice"
        assert got == brute.misses_of_ray(dims, s, g)
        checked += 1
    assert checked > 900


def test_dda_exact_corner_and_face_rays_consistent():
    # rays through exact voxel corners: deterministic tie order x < y < z (A10)
    w = O.traverse((8, 8, 8), (0.5, 0.5, 0.5), (2.5, 2.5, 0.5))
    assert w.tolist() == [[0, 0, 0], [1, 0, 0], [1, 1, 0], [2, 1, 0]]


def _check_walk(walk, S, E, dims):
    V = np.asarray(walk, dtype=np.int64)
    if V.shape[0] == 0:
        return
    assert tuple(V[0]) == tuple(S)
    step = np.sign(np.asarray(E) - np.asarray(S))
    dv = np.diff(V, axis=0)
    # 6-connected, one axis per step, in the step direction
    assert np.all(np.abs(dv).sum(1) == 1)
    assert np.all((dv * step[None, :]) >= 0)
    lo = np.minimum(S, E)
    hi = np.maximum(S, E)
    assert np.all(V >= lo) and np.all(V <= hi)
    assert np.all(V >= 0) and np.all(V < np.asarray(dims))


def test_long_ray_invariants():
    rs = np.random.default_rng(7)
    dims = (1024, 1024, 128)
    for _ in range(300):
        s = rs.uniform([400, 400, 50], [624, 624, 78]).astype(np.float32)
        g = (s + rs.normal(0, 300, size=3)).astype(np.float32)
        walk = O.traverse(dims, s, g, cap=1 << 14)
        S = np.floor(s).astype(np.int64)
        E = np.floor(g).astype(np.int64)
        _check_walk(walk, S, E, dims)
        inside = np.all(E >= 0) and np.all(E < np.asarray(dims))
        if inside:
            assert walk.shape[0] == int(np.abs(E - S).sum())
            last = walk[-1].astype(np.int64)
            assert int(np.abs(E - last).sum()) == 1
        else:
            # stopped at the grid boundary: one more step leaves the grid
            last = walk[-1].astype(np.int64)
            assert np.any(last == 0) or np.any(last == np.asarray(dims) - 1)


def test_exit_walk_matches_brute_force_on_small_grid():
    # endpoints far outside: walk must equal the in-grid part of the segment
    rs = np.random.default_rng(11)
    dims = (6, 5, 4)
    n = 0
    for _ in range(600):
        s = rs.uniform([0, 0, 0], dims).astype(np.float32)
        g = rs.uniform(-30, 30, size=3).astype(np.float32)
        if brute.near_tie(s, g):
            continue
        walk = O.traverse(dims, s, g)
        assert {tuple(v) for v in walk.tolist()} == brute.misses_of_ray(dims, s, g)
        n += 1
    assert n > 500
