"""Pins of the 8-cone negative-obstacle oracle (or_negative8; SURVEY 8(f) NEXT-3,
SPEC S:327 "D = 8 directions at half-angle 22.5 deg ... Chebyshev rings";
DESIGN.md reading B8), against things other than its own integer cone rule:

- the cone of an offset equals the nearest multiple of 45 degrees of its
  float64 atan2 angle (tan 22.5 is irrational: no offset sits on a boundary);
- small random maps agree with a pure-Python search that assigns cones by
  atan2 and walks each Chebyshev ring explicitly;
- a hand-checked scene where 8 cones see a second height that 4 cones miss;
- a fully defined map has no flags; flags never grow with the threshold.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O


def atan_cone(u, v):
    a = math.atan2(v, u) / (math.pi / 4)
    j = int(math.floor(a + 0.5)) % 8
    # distance to the nearest cone boundary (odd multiples of 22.5 deg), in units of 45 deg
    margin = 0.5 - abs(a - math.floor(a + 0.5))
    return j, margin


def test_cone8_partition_matches_atan2():
    for u in range(-40, 41):
        for v in range(-40, 41):
            if u == 0 and v == 0:
                assert O.cone8_of(0, 0) == -1
                continue
            j, margin = atan_cone(u, v)
            assert margin > 1e-6  # never on a boundary
            assert O.cone8_of(u, v) == j, (u, v)


def brute_negative8(qs, defined, K, T):
    ny, nx = qs.shape
    neg = np.zeros((ny, nx), dtype=np.uint8)
    for y in range(ny):
        for x in range(nx):
            if defined[y, x]:
                continue
            F = []
            for cone in range(8):
                for k in range(1, K + 1):
                    ring = [(x + u, y + v) for u in range(-k, k + 1) for v in range(-k, k + 1)
                            if max(abs(u), abs(v)) == k and atan_cone(u, v)[0] == cone]
                    hits = [qs[yy, xx] for xx, yy in ring
                            if 0 <= xx < nx and 0 <= yy < ny and defined[yy, xx]]
                    if hits:
                        F += hits
                        break
            neg[y, x] = 1 if len(F) >= 2 and max(F) - min(F) > T else 0
    return neg


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_negative8_matches_brute_force(seed):
    rs = np.random.default_rng(seed)
    ny, nx, K = 18, 23, 6
    defined = (rs.random((ny, nx)) < 0.3).astype(np.uint8)
    qs = np.where(defined, rs.integers(0, 40 * 65536, (ny, nx)), np.iinfo(np.int32).min)
    qs = qs.astype(np.int32)
    T = 5 * 65536
    got = O.negative8(qs, defined, K, T)
    assert np.array_equal(got, brute_negative8(qs, defined, K, T))
    assert got.sum() > 0  # the case is not vacuous


def test_negative8_sees_what_four_cones_miss():
    # apex at (10, 10); defined cells at offsets (2, 2) (45-deg cone, ring 2) and
    # (4, 0) (+x cone, ring 4).  4 axis cones: +x and +y both stop at ring 2 on
    # (2, 2) alone -> F = {h1}.  8 cones: (4, 0) is the first ring of the +x cone
    # -> F = {h1, h2}.
    nx = ny = 21
    defined = np.zeros((ny, nx), np.uint8)
    qs = np.full((ny, nx), np.iinfo(np.int32).min, np.int32)
    defined[12, 12], qs[12, 12] = 1, 10 * 65536
    defined[10, 14], qs[10, 14] = 1, 2 * 65536
    T = 1 * 65536
    n4 = O.negative(qs, defined, 8, T)
    n8 = O.negative8(qs, defined, 8, T)
    assert n4[10, 10] == 0
    assert n8[10, 10] == 1


def test_negative8_fully_defined_and_monotone():
    rs = np.random.default_rng(7)
    ny, nx, K = 16, 16, 5
    qs = rs.integers(0, 30 * 65536, (ny, nx)).astype(np.int32)
    assert O.negative8(qs, np.ones((ny, nx), np.uint8), K, 0).sum() == 0
    defined = (rs.random((ny, nx)) < 0.35).astype(np.uint8)
    prev = None
    for T in (0, 65536, 4 * 65536, 16 * 65536, 64 * 65536):
        cur = O.negative8(qs, defined, K, T)
        if prev is not None:
            assert np.all(cur <= prev)
        prev = cur
