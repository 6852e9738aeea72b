"""Pins of the contract edges G1-G5 leave open: readings A18, A19, A22, A24, A25.

Golden cases in tests/golden/G6_contract_edges.json, each derived by hand in
its "derivation" field (PAPER.md P:114 band and weighted density, P:116 plane
fit, P:133 / fig:neg_obs_search P:142 cones and "larger than").  Each case is
chosen so that the plausible misreading listed beside it gives a different
answer; tests/test_oracle_mutants.py checks that the oracle's misread
variants fail here.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                   "G6_contract_edges.json")))
RES = GOLD["res"]


def _thr():
    t = GOLD["thresholds"]
    T = np.array([t["T_lo"], t["T_hi"], t["tau"], t["T_neg"]])
    # the golden thresholds are O0 of the defaults (derivation field)
    assert np.array_equal(T, O.thresholds(RES, 0.3, 2.0, 0.5, 0.5))
    return T


def _column(nz, voxels, o_z=0):
    H = np.zeros(nz, np.uint64)
    Mi = np.zeros(nz, np.uint64)
    mn = np.full(nz, 0xFFFFFFFF, np.uint32)
    for v in voxels:
        H[v["z"]], Mi[v["z"]], mn[v["z"]] = v["hits"], v["misses"], v["min_dz"]
    height, dens, hard, soft, qs, dfn = O.columns((1, 1, nz), RES, o_z, _thr(), H, Mi, mn)
    return dens[0, 0], hard[0, 0], soft[0, 0], qs[0, 0], dfn[0, 0]


# ------------------------------------------------------------------ A19
def test_A19_weighted_density_two_band_voxels():
    g = GOLD["A19_weighted_density"]
    dens, hard, soft, qs, dfn = _column(g["nz"], g["column"], g["o_z"])
    assert dfn == 1 and qs == g["q_s"]
    assert dens == np.float32(g["density"])
    assert dens == np.float32(2.0 / 11.0)
    assert (hard, soft) == (g["hard"], g["soft"])


# ------------------------------------------------------------------ A18
@pytest.mark.parametrize("case", GOLD["A18_band_edges"]["cases"], ids=lambda c: c["name"])
def test_A18_band_edges(case):
    g = GOLD["A18_band_edges"]
    dens, hard, soft, _, dfn = _column(g["nz"], case["column"], g["o_z"])
    assert dfn == 1
    assert dens == np.float32(case["density"])
    assert (hard, soft) == (case["hard"], case["soft"])


# ------------------------------------------------------------------ A22
def _window(case):
    g = GOLD["A22_min_plane_points"]
    n = g["size"]
    q = np.zeros((n, n), np.int32)
    dfn = np.zeros((n, n), np.uint8)
    for x, y in g["defined_xy"]:
        dfn[y, x] = 1
    for x, y, v in case["q_xy"]:
        q[y, x] = v
    return q, dfn


def test_A22_exactly_min_plane_points_is_enough():
    g = GOLD["A22_min_plane_points"]
    cx, cy = g["centre"]
    c = g["planar"]
    q, dfn = _window(c)
    sl, ro = O.slope_roughness(q, dfn, RES, g["N"], c["min_plane_points"])
    assert int(dfn.sum()) == c["min_plane_points"]
    assert sl[cy, cx] == np.float32(c["slope"])
    assert ro[cy, cx] == 0.0


def test_A22_four_point_residual_closed_form():
    g = GOLD["A22_min_plane_points"]
    cx, cy = g["centre"]
    c = g["one_off"]
    q, dfn = _window(c)
    sl, ro = O.slope_roughness(q, dfn, RES, g["N"], c["min_plane_points"])
    assert sl[cy, cx] == pytest.approx(c["slope"], rel=1e-6)
    assert sl[cy, cx] == pytest.approx(math.atan(math.sqrt(2.0) / 3.0), rel=1e-6)
    assert ro[cy, cx] == pytest.approx(c["roughness"], rel=1e-6)
    assert ro[cy, cx] == pytest.approx(RES * RES / 48.0, rel=1e-6)


def test_A22_one_point_short_is_nodata():
    g = GOLD["A22_min_plane_points"]
    cx, cy = g["centre"]
    q, dfn = _window(g["planar"])
    sl, ro = O.slope_roughness(q, dfn, RES, g["N"], g["too_few"]["min_plane_points"])
    assert math.isnan(sl[cy, cx]) and math.isnan(ro[cy, cx])


# ------------------------------------------------------------- A24
@pytest.mark.parametrize("case", GOLD["A24_ring_corners"]["cases"], ids=lambda c: c["name"])
def test_A24_ring_corners_shared(case):
    g = GOLD["A24_ring_corners"]
    n = case["size"]
    q = np.full((n, n), case.get("default_q", 0), np.int32)
    if case.get("undefined_all"):
        dfn = np.zeros((n, n), np.uint8)
    else:
        dfn = np.ones((n, n), np.uint8)
        for x, y in case["undefined_xy"]:
            dfn[y, x] = 0
    for x, y, v in case["q_xy"]:
        q[y, x] = v
        dfn[y, x] = 1
    neg = O.negative(q, dfn, g["K_neg"], _thr()[3])
    x, y = case["neg_at"]
    assert neg[y, x] == case["flag"]


# ------------------------------------------------------------------ A25
def test_A25_delta_h_equal_to_threshold_is_not_an_obstacle():
    g = GOLD["A25_strict_greater"]
    n = g["size"]
    for low, flag in g["flag_cases"]:
        q = np.zeros((n, n), np.int32)
        dfn = np.ones((n, n), np.uint8)
        dfn[n // 2, n // 2] = 0
        x, y = g["low_cell"]
        q[y, x] = low
        neg = O.negative(q, dfn, g["K_neg"], _thr()[3])
        assert neg[n // 2, n // 2] == flag
