"""Pins for oracle steps O8 (columns), O9 (slope/roughness), O10 (negative).

PAPER.md P:112 (height = min return of the lowest voxel), P:114 (positive
obstacles, weighted density, hard/soft), P:116 (N x N least-squares plane,
roughness = average squared error), P:118 / P:133 / P:142 (negative obstacles
by cone search and Delta-H).  Pins: golden G3-G5, closed-form planes,
numpy.linalg.lstsq brute force, brute-force column minima, invariants and
scenario worlds from the seeded generator (wall -> hard, sparse vegetation ->
soft, 1.5 m step -> negative, 0.3 m dip -> none).
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2109_13176_b200 import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# --------------------------------------------------------------------------- O8
def test_golden_G3_column():
    g = json.load(open(os.path.join(GOLD, "G3_column.json")))
    nz = g["nz"]
    dims = (1, 1, nz)
    H = np.zeros(nz, np.uint64)
    Mi = np.zeros(nz, np.uint64)
    mn = np.full(nz, 0xFFFFFFFF, np.uint32)
    for c in g["column"]:
        H[c["z"]], Mi[c["z"]], mn[c["z"]] = c["hits"], c["misses"], c["min_dz"]
    t = g["thresholds"]
    T = np.array([t["T_lo"], t["T_hi"], t["tau"], t["T_neg"]])
    height, dens, hard, soft, qs, dfn = O.columns(dims, g["res"], g["o_z"], T, H, Mi, mn)
    assert qs[0, 0] == g["q_s"] and dfn[0, 0] == 1
    assert height[0, 0] == np.float32(g["height"])
    assert dens[0, 0] == np.float32(g["density"])
    assert (hard[0, 0], soft[0, 0]) == (g["hard"], g["soft"])


def test_columns_empty_and_no_band():
    dims = (2, 1, 8)
    H = np.zeros(16, np.uint64)
    Mi = np.zeros(16, np.uint64)
    mn = np.full(16, 0xFFFFFFFF, np.uint32)
    H[3], mn[3] = 4, 100  # column 0: single ground voxel, nothing in the band
    T = O.thresholds(0.25, 0.3, 2.0, 0.5, 0.5)
    height, dens, hard, soft, qs, dfn = O.columns(dims, 0.25, 0, T, H, Mi, mn)
    assert dfn[0, 0] == 1 and dens[0, 0] == 0.0 and hard[0, 0] == 0 and soft[0, 0] == 0
    assert dfn[0, 1] == 0 and math.isnan(height[0, 1]) and math.isnan(dens[0, 1])


def test_hard_at_equality():
    # A20: density == threshold counts as hard
    dims = (1, 1, 8)
    H = np.zeros(8, np.uint64)
    Mi = np.zeros(8, np.uint64)
    mn = np.full(8, 0xFFFFFFFF, np.uint32)
    H[0], mn[0] = 1, 0
    H[2], Mi[2], mn[2] = 5, 5, 0
    T = O.thresholds(0.25, 0.3, 2.0, 0.5, 0.5)
    _, dens, hard, soft, _, _ = O.columns(dims, 0.25, 0, T, H, Mi, mn)
    assert dens[0, 0] == 0.5 and hard[0, 0] == 1 and soft[0, 0] == 0


def _run(world, grid, **scan_kw):
    scan = synth.scenario_scan(world, **scan_kw)
    om = O.OracleMap(grid)
    om.shift((scan.pose[0, 3], scan.pose[1, 3], scan.pose[2, 3] - scan_kw.get("sensor_z", 1.5)))
    fm = om.integrate([(scan.points, scan.pose)])
    return om, fm, om.compute_maps(), scan


def test_height_is_brute_force_column_min():
    # each defined cell equals the min return of its lowest occupied voxel
    w = synth.workload(0)
    om = O.OracleMap(w.grid)
    f = w.frames[0]
    om.shift(f.vehicle_xyz)
    om.integrate([(s.points, s.pose) for s in f.scans])
    L = om.compute_maps()
    s = f.scans[0]
    A, b = O.affine(s.pose, om.res, om.origin)
    g = np.array([O.transform_point(A, b, *p[:3])[1] for p in s.points])
    v = np.floor(g).astype(np.int64)
    nx, ny, nz = om.dims
    inb = np.all((v >= 0) & (v < np.array([nx, ny, nz])), axis=1)
    q = np.floor(g[inb, 2].astype(np.float32) * np.float32(65536)).astype(np.int64)
    col = v[inb, 0] + nx * v[inb, 1]
    exp = np.full(nx * ny, np.iinfo(np.int64).max)
    np.minimum.at(exp, col, q)
    defined = exp != np.iinfo(np.int64).max
    assert np.array_equal(L.defined.reshape(-1).astype(bool), defined)
    assert np.array_equal(L.qs.reshape(-1)[defined].astype(np.int64), exp[defined])
    # invariants: hard XOR soft on defined cells, nothing on undefined
    assert not np.any(L.hard & L.soft)
    assert not np.any((L.hard | L.soft) & (L.defined == 0))
    assert not np.any(L.neg & L.defined)


def _scen_grid(n=128, nz=32, res=0.25):
    return synth.grid_cfg(n, n, nz, res)


def test_wall_is_hard_obstacle():
    # north_star: "a wall as a hard one"; P:114 hard = density above threshold
    w = synth.World()
    w.boxes.append((4.1, 4.3, -1.5, 1.5, 0.0, 1.2))
    om, fm, L, _ = _run(w, _scen_grid(), rings=64, columns=1440, vfov=(-30.0, 10.0))
    o = om.buffer[-1].origin
    res = om.res
    xs = (np.arange(om.dims[0]) + o[0] + 0.5) * res
    ys = (np.arange(om.dims[1]) + o[1] + 0.5) * res
    X, Y = np.meshgrid(xs, ys)
    foot = (np.abs(X - 4.125) < 0.126) & (np.abs(Y) < 1.4)
    assert foot.sum() >= 8
    assert L.hard[foot].mean() >= 0.9
    near = (np.abs(X - 4.2) < 0.5) & (np.abs(Y) < 1.75)
    assert L.hard[~near].sum() == 0
    assert L.soft[~near].sum() == 0


def test_sparse_vegetation_is_soft_obstacle():
    # north_star: "sparse vegetation is classed as a soft obstacle"
    w = synth.World()
    w.veg_boxes.append((4.0, 6.0, -1.0, 1.0, 0.0, 1.5, 0.1))
    om, fm, L, _ = _run(w, _scen_grid(), rings=64, columns=1440, vfov=(-30.0, 10.0))
    o = om.buffer[-1].origin
    res = om.res
    xs = (np.arange(om.dims[0]) + o[0] + 0.5) * res
    ys = (np.arange(om.dims[1]) + o[1] + 0.5) * res
    X, Y = np.meshgrid(xs, ys)
    foot = (X > 4.3) & (X < 5.7) & (np.abs(Y) < 0.7) & (L.defined == 1)
    assert foot.sum() >= 10
    flagged = foot & ((L.soft == 1) | (L.hard == 1))
    assert flagged.sum() >= 0.8 * foot.sum()
    assert L.soft[flagged].mean() >= 0.9
    d = L.density[flagged]
    assert 0.02 <= float(np.median(d)) <= 0.3


def test_flat_ground_no_flags():
    w = synth.World()
    om, fm, L, _ = _run(w, _scen_grid(64, 16), rings=32, columns=720)
    assert L.hard.sum() == 0 and L.soft.sum() == 0 and L.neg.sum() == 0
    d = L.defined == 1
    assert np.nanmax(np.abs(L.slope[d])) < 0.05


# --------------------------------------------------------------------------- O9
def _window_case(q, res=0.25, N=5, minp=4):
    qs = np.asarray(q, np.int32)
    dfn = np.ones_like(qs, dtype=np.uint8)
    return O.slope_roughness(qs, dfn, res, N, minp)


def test_flat_plane_zero():
    sl, ro = _window_case(np.full((7, 7), 12345))
    assert np.all(sl == 0) and np.all(ro == 0)


def test_golden_G4_plane_and_checkerboard():
    g = json.load(open(os.path.join(GOLD, "G4_G5_layers.json")))["G4"]
    u, v = np.meshgrid(np.arange(-2, 3), np.arange(-2, 3))
    q = g["plane_q"]["a"] * u + g["plane_q"]["b"] * v + 500000
    sl, ro = _window_case(q, g["res"], g["N"])
    assert sl[2, 2] == np.float32(g["slope"])
    # closed form: atan of the exact fixed-point gradient norm
    assert sl[2, 2] == np.float32(math.atan(math.hypot(19661, 26214) / 65536))
    assert ro[2, 2] == 0.0
    cb = np.where((u + v) % 2 == 0, 1000, -1000)
    sl2, ro2 = _window_case(q + cb, g["res"], g["N"])
    assert ro2[2, 2] == pytest.approx(g["checkerboard_roughness"], rel=1e-6)
    assert sl2[2, 2] == pytest.approx(g["slope"], abs=1e-12)


def test_spec_plane_03_04():
    # z = 0.3x + 0.4y + 1 -> atan(0.5), roughness 0 (up to fixed point)
    res = 0.25
    u, v = np.meshgrid(np.arange(9), np.arange(9))
    z_vox = (0.3 * u * res + 0.4 * v * res + 1.0) / res
    q = np.round(z_vox * 65536).astype(np.int64)
    sl, ro = _window_case(q, res)
    inner = sl[2:-2, 2:-2]
    assert np.all(np.abs(inner - math.atan(0.5)) < 1e-5)
    assert np.all(ro[2:-2, 2:-2] < 1e-9)


def test_slope_matches_lstsq_brute_force():
    rs = np.random.default_rng(12)
    res = 0.2
    for N in (3, 5, 7, 9):
        r = (N - 1) // 2
        for _ in range(40):
            n = N + 6
            q = rs.integers(0, 2 ** 24, size=(n, n))
            dfn = (rs.random((n, n)) > 0.25).astype(np.uint8)
            dfn[n // 2, n // 2] = 1
            sl, ro = O.slope_roughness(q.astype(np.int32), dfn, res, N, 4)
            cy = cx = n // 2
            uu, vv, zz = [], [], []
            for dv in range(-r, r + 1):
                for du in range(-r, r + 1):
                    if dfn[cy + dv, cx + du]:
                        uu.append(du)
                        vv.append(dv)
                        zz.append(q[cy + dv, cx + du] - q[cy, cx])
            Am = np.stack([uu, vv, np.ones(len(uu))], 1).astype(np.float64)
            if len(uu) < 4 or np.linalg.matrix_rank(Am) < 3:
                assert math.isnan(sl[cy, cx])
                continue
            coef, *_ = np.linalg.lstsq(Am, np.asarray(zz, np.float64), rcond=None)
            a, b = coef[0] / 65536, coef[1] / 65536
            resid = np.asarray(zz) - Am @ coef
            exp_ro = float(np.mean(resid ** 2)) * (res / 65536) ** 2
            assert sl[cy, cx] == pytest.approx(math.atan(math.hypot(a, b)), rel=1e-6, abs=1e-9)
            assert ro[cy, cx] == pytest.approx(exp_ro, rel=1e-5, abs=1e-12)


def test_slope_rotation_consistency():
    # rotating the height grid by 90 deg rotates the layers
    rs = np.random.default_rng(13)
    q = rs.integers(0, 2 ** 22, size=(20, 20)).astype(np.int32)
    dfn = (rs.random((20, 20)) > 0.2).astype(np.uint8)
    sl, ro = O.slope_roughness(q, dfn, 0.25, 5, 4)
    sl2, ro2 = O.slope_roughness(np.ascontiguousarray(np.rot90(q)),
                                 np.ascontiguousarray(np.rot90(dfn)), 0.25, 5, 4)
    a, b = np.rot90(sl), sl2
    assert np.array_equal(np.isnan(a), np.isnan(b))
    m = ~np.isnan(a)
    assert np.allclose(a[m], b[m], rtol=1e-6, atol=1e-9)
    assert np.allclose(np.rot90(ro)[m], ro2[m], rtol=1e-5, atol=1e-12)


def test_slope_nodata_cases():
    q = np.zeros((5, 5), np.int32)
    dfn = np.zeros((5, 5), np.uint8)
    dfn[2, :] = 1  # collinear defined cells -> singular -> NaN
    sl, ro = O.slope_roughness(q, dfn, 0.25, 5, 4)
    assert np.all(np.isnan(sl)) and np.all(np.isnan(ro))
    dfn2 = np.zeros((5, 5), np.uint8)
    dfn2[2, 2] = dfn2[1, 1] = dfn2[3, 1] = 1  # only 3 points < min_plane_points
    sl, _ = O.slope_roughness(q, dfn2, 0.25, 5, 4)
    assert np.all(np.isnan(sl))
    dfn3 = np.ones((5, 5), np.uint8)
    dfn3[2, 2] = 0  # undefined centre -> NaN there only
    sl, _ = O.slope_roughness(q, dfn3, 0.25, 5, 4)
    assert math.isnan(sl[2, 2]) and sl[0, 0] == 0.0


# -------------------------------------------------------------------------- O10
def test_golden_G5():
    g = json.load(open(os.path.join(GOLD, "G4_G5_layers.json")))["G5"]
    n = g["size"]
    for low, flag in g["flag_cases"]:
        q = np.zeros((n, n), np.int32)
        dfn = np.ones((n, n), np.uint8)
        dfn[2, 2] = 0
        x, y = g["low_cell"]
        q[y, x] = low
        neg = O.negative(q, dfn, g["K_neg"], g["T_neg"])
        assert neg[2, 2] == flag
        assert neg.sum() == flag


def test_negative_fully_defined_none():
    q = np.random.default_rng(0).integers(-10 ** 6, 10 ** 6, size=(16, 16)).astype(np.int32)
    assert O.negative(q, np.ones((16, 16), np.uint8), 8, 1).sum() == 0


def test_negative_first_ring_only():
    # a cone stops at its first ring holding a defined cell ("until a
    # defined surface has been found"): the deeper cell behind is never used
    n = 11
    q = np.zeros((n, n), np.int32)
    dfn = np.zeros((n, n), np.uint8)
    c = 5
    dfn[c, c + 2] = 1  # +x ring 2 (first defined), q = 0
    dfn[c, c + 4] = 1
    q[c, c + 4] = -10 ** 6  # behind it, ring 4
    dfn[c, c - 3] = 1  # -x ring 3, q = 0
    assert O.negative(q, dfn, 6, 1000)[c, c] == 0
    q[c, c - 3] = -5000  # now the two found heights differ by 5000
    assert O.negative(q, dfn, 6, 1000)[c, c] == 1
    assert O.negative(q, dfn, 2, 1000)[c, c] == 0  # -x ring 3 beyond K_neg = 2


def _step_world(drop):
    w = synth.World()
    w.steps.append((1.0, 0.0, 5.0, -drop))
    return w


def test_negative_step_scenario():
    # P:266-279 (1.5 m step seen from above)
    om, fm, L, _ = _run(_step_world(1.5), _scen_grid(128, 32), rings=64, columns=1440,
                        vfov=(-30.0, 10.0))
    o = om.buffer[-1].origin
    xs = (np.arange(om.dims[0]) + o[0] + 0.5) * om.res
    ys = (np.arange(om.dims[1]) + o[1] + 0.5) * om.res
    X, Y = np.meshgrid(xs, ys)
    shadow = (X > 5.6) & (X < 9.4) & (np.abs(Y) < 2.0) & (L.defined == 0)
    assert shadow.sum() > 50
    assert L.neg[shadow].mean() >= 0.95
    # well-sampled upper ground before the edge is never flagged
    assert L.neg[(X < 4.5) & (np.abs(Y) < 6.0)].sum() == 0


def test_negative_shallow_dip_none():
    w = synth.World()
    w.pits.append((5.0, 7.0, -8.0, 8.0, 0.3))
    om, fm, L, _ = _run(w, _scen_grid(128, 32), rings=64, columns=1440, vfov=(-30.0, 10.0))
    assert L.neg.sum() == 0


def test_negative_monotone_in_threshold():
    # raising Delta-H never adds flags
    om, fm, L, _ = _run(_step_world(1.5), _scen_grid(128, 32), rings=32, columns=720,
                        vfov=(-30.0, 10.0))
    prev = None
    for thr in np.linspace(0.1, 2.0, 12):
        T = O.thresholds(om.res, 0.3, 2.0, 0.5, float(thr))
        neg = O.negative(L.qs, L.defined, int(om.g["neg_obs_search_cells"]), T[3])
        if prev is not None:
            assert np.all(neg <= prev)
        prev = neg
    assert prev.sum() == 0


# ------------------------------------------------------------ NEXT-3 variants
def test_spread_closed_form():
    # point spread of the surface voxel = population variance of its return
    # heights (numpy.var of the fixed-point values), times (res/65536)^2
    res = 0.25
    rs = np.random.default_rng(5)
    for n in (1, 2, 5, 40):
        dz = rs.integers(0, 65536, size=n).astype(np.uint64)
        nz = 6
        H = np.zeros(nz, np.uint64)
        M1 = np.zeros(nz, np.uint64)
        M2 = np.zeros(nz, np.uint64)
        H[2], M1[2], M2[2] = n, dz.sum(), (dz * dz).sum()
        H[4], M1[4], M2[4] = 3, 10, 1000  # a higher voxel is ignored
        sp = O.spread((1, 1, nz), res, H, M1, M2)[0, 0]
        exp = np.var(dz.astype(np.float64)) * (res / 65536) ** 2
        assert sp == pytest.approx(exp, rel=1e-6, abs=1e-15)
    assert math.isnan(O.spread((1, 1, 3), res, np.zeros(3, np.uint64), np.zeros(3, np.uint64),
                               np.zeros(3, np.uint64))[0, 0])


def test_slope_excluding_obstacle_cells():
    # SPEC S:338 variant: excluded cells leave every window and get NaN
    rs = np.random.default_rng(6)
    q = rs.integers(0, 2 ** 20, size=(12, 12)).astype(np.int32)
    dfn = np.ones((12, 12), np.uint8)
    ex = (rs.random((12, 12)) < 0.2).astype(np.uint8)
    sl, ro = O.slope_roughness(q, dfn, 0.25, 5, 4, ex)
    sl2, ro2 = O.slope_roughness(q, (dfn & (1 - ex)).astype(np.uint8), 0.25, 5, 4)
    assert np.array_equal(np.isnan(sl), np.isnan(sl2))
    m = ~np.isnan(sl)
    assert np.array_equal(sl[m], sl2[m]) and np.array_equal(ro[m], ro2[m])
    assert np.all(np.isnan(sl[ex == 1]))
