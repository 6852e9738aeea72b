"""Pins for oracle step O7 (combine / shift) and O1+O7 map shifts.

PAPER.md P:110: "offsetting each of the map indices by the offset between the
buffer map and the combined map.  The combined map uses the location of the
most recent buffer map as it's origin.  Voxel metrics are then combined with
number of hits and misses being added together and minimum return heights
compared and the minimum taken."
"""
import numpy as np
import pytest

from oracle import oracle as O


def _pose_t(t):
    P = np.zeros((3, 4))
    P[:, :3] = np.eye(3)
    P[:, 3] = t
    return P


def _fm_from_dense(h, m, mn, m1, m2, o):
    return O.frame_map(h.astype(np.uint32), m.astype(np.uint32), mn.astype(np.uint32),
                       m1.astype(np.uint64), m2.astype(np.uint64), np.asarray(o, np.int64))


def _g1_map(o=(0, 0, 0)):
    dims = (4, 4, 2)
    s = np.array([0.5, 0.5, 0.5])
    pw = np.array([[3.5, 0.5, 0.5], [2.5, 2.25, 0.5], [1.5, 0.5, 0.5], [6.5, 0.5, 0.5]])
    pts = np.zeros((4, 4), np.float32)
    pts[:, :3] = pw - s
    h, m, mn, m1, m2, st = O.integrate_dense(dims, [(pts, _pose_t(s))], 1.0, np.zeros(3, np.int64))
    return dims, O.frame_map(h, m, mn, m1, m2, np.asarray(o, np.int64), st)


def test_single_slot_identity():
    # single-map buffer -> output equals input field for field
    dims, fm = _g1_map()
    H, Mi, mn, M1, M2 = O.combine(dims, [fm], fm.origin)
    out = _fm_from_dense(H, Mi, mn, M1, M2, fm.origin)
    for f in ("lut", "hits", "misses", "min_dz", "m1", "m2"):
        assert np.array_equal(getattr(out, f), getattr(fm, f)), f


def test_two_map_arithmetic():
    # same voxel with hits 2/3, misses 1/4, min 0.9/0.7 -> 5, 5, min
    dims = (2, 2, 2)
    V = 8
    maps = []
    for hits, miss, mnv in ((2, 1, 58982), (3, 4, 45875)):
        h = np.zeros(V)
        m = np.zeros(V)
        mn = np.full(V, 0xFFFFFFFF)
        h[3], m[3], mn[3] = hits, miss, mnv
        maps.append(_fm_from_dense(h, m, mn, h * mnv, h * mnv * mnv, (0, 0, 0)))
    H, Mi, mn, M1, M2 = O.combine(dims, maps, np.zeros(3, np.int64))
    assert H[3] == 5 and Mi[3] == 5 and mn[3] == 45875
    assert M1[3] == 2 * 58982 + 3 * 45875


def test_empty_misses_carried():
    # empty-voxel N_m of one map adds to an occupied voxel of another
    dims = (2, 2, 2)
    V = 8
    h0 = np.zeros(V)
    m0 = np.zeros(V)
    m0[5] = 7
    h1 = np.zeros(V)
    h1[5] = 2
    m1 = np.zeros(V)
    m1[5] = 1
    mn1 = np.full(V, 0xFFFFFFFF)
    mn1[5] = 10
    a = _fm_from_dense(h0, m0, np.full(V, 0xFFFFFFFF), h0, h0, (0, 0, 0))
    b = _fm_from_dense(h1, m1, mn1, h1 * 10, h1 * 100, (0, 0, 0))
    H, Mi, mn, M1, M2 = O.combine(dims, [a, b], np.zeros(3, np.int64))
    assert (H[5], Mi[5], mn[5]) == (2, 8, 10)


def test_golden_G2_shift():
    dims, fm = _g1_map()
    o1 = np.array([1, 0, 0], np.int64)
    H, Mi, mn, M1, M2 = O.combine(dims, [fm], o1)
    L = lambda x, y, z: z + 2 * (x + 4 * y)  # noqa: E731
    # output (0,0,0) <- source (1,0,0): occupied, hits 1, misses 3
    assert (H[L(0, 0, 0)], Mi[L(0, 0, 0)]) == (1, 3)
    # column x = 3 is newly exposed: empty with 0 misses
    for y in range(4):
        for z in range(2):
            assert H[L(3, y, z)] == 0 and Mi[L(3, y, z)] == 0
    # shift back by -(1,0,0): x in [1,3] restored, x = 0 empty
    shifted = _fm_from_dense(H, Mi, mn, M1, M2, o1)
    H2, Mi2, mn2, _, _ = O.combine(dims, [shifted], np.zeros(3, np.int64))
    Hr, Mir, mnr, _, _ = O.combine(dims, [fm], np.zeros(3, np.int64))
    for y in range(4):
        for z in range(2):
            assert H2[L(0, y, z)] == 0 and Mi2[L(0, y, z)] == 0
            for x in range(1, 4):
                assert (H2[L(x, y, z)], Mi2[L(x, y, z)], mn2[L(x, y, z)]) == (
                    Hr[L(x, y, z)], Mir[L(x, y, z)], mnr[L(x, y, z)])


def test_shift_preserves_counts_on_overlap():
    # BASELINE.json north_star: "map shifts preserve counts"
    from paper_2109_13176_b200 import synth
    w = synth.workload(0)
    om = O.OracleMap(w.grid)
    f = w.frames[0]
    om.shift(f.vehicle_xyz)
    fm = om.integrate([(s.points, s.pose) for s in f.scans])
    dims = om.dims
    rs = np.random.default_rng(4)
    for _ in range(4):
        d = rs.integers(-6, 7, size=3)
        o2 = fm.origin + d
        H, Mi, mn, M1, M2 = O.combine(dims, [fm], o2)
        H0, Mi0, mn0, M10, M20 = O.combine(dims, [fm], fm.origin)
        g0 = H0.reshape(dims[1], dims[0], dims[2])  # [y][x][z]
        g1 = H.reshape(dims[1], dims[0], dims[2])
        m0 = Mi0.reshape(g0.shape)
        m1_ = Mi.reshape(g0.shape)
        # output v at o2 equals source v + d at o1 where both are in grid
        sl_src = [slice(max(0, d[i]), dims[i] + min(0, d[i])) for i in range(3)]
        sl_dst = [slice(max(0, -d[i]), dims[i] + min(0, -d[i])) for i in range(3)]
        src = (sl_src[1], sl_src[0], sl_src[2])
        dst = (sl_dst[1], sl_dst[0], sl_dst[2])
        assert np.array_equal(g1[dst], g0[src])
        assert np.array_equal(m1_[dst], m0[src])
        assert int(g1.sum()) == int(g0[src].sum())


def test_union_equality_integer_motion():
    # SPEC S:225/S:228 under the condition that makes it exact:
    # identity rotation, integer-voxel motion, points on a 1/8 lattice, res 1 ->
    # every f32 op exact; combine(buffer) == one integration of the union of
    # rays at the newest origin, on voxels inside both grids.
    dims = (24, 20, 10)
    rs = np.random.default_rng(8)
    grid = dict(nx=dims[0], ny=dims[1], nz=dims[2], res=1.0, z_center_frac=0.5, buffer_frames=4,
                min_obstacle_height=0.3, max_obstacle_height=2.0, density_threshold=0.5,
                slope_window=5, min_plane_points=4, neg_obs_threshold=0.5,
                neg_obs_search_cells=6)
    om = O.OracleMap(grid)
    scans = []
    veh = np.array([0.0, 0.0, 0.0])
    for f in range(3):
        veh = veh + np.array([rs.integers(-2, 3), rs.integers(-2, 3), 0])
        om.shift(veh)
        sensor = veh + np.array([0.5, 0.25, 0.125])
        world = sensor + rs.integers(-160, 160, size=(300, 3)) / 8.0
        pts = np.zeros((300, 4), np.float32)
        pts[:, :3] = world - sensor
        pts = pts[np.any(pts[:, :3] != 0, axis=1)]
        om.integrate([(pts, _pose_t(sensor))])
        scans.append((pts, _pose_t(sensor)))
    om.compute_maps()
    H, Mi, mn, M1, M2, o = om.merged
    hu, mu, mnu, m1u, m2u, _ = O.integrate_dense(dims, scans, 1.0, o)
    # voxels inside every frame's grid
    mask = np.ones((dims[1], dims[0], dims[2]), bool)
    for fm in om.buffer:
        d = fm.origin - o
        yy, xx, zz = np.meshgrid(np.arange(dims[1]), np.arange(dims[0]), np.arange(dims[2]),
                                 indexing="ij")
        mask &= (xx - d[0] >= 0) & (xx - d[0] < dims[0]) & (yy - d[1] >= 0) & (
            yy - d[1] < dims[1]) & (zz - d[2] >= 0) & (zz - d[2] < dims[2])
    mk = mask.reshape(-1)
    assert mk.sum() > 0.5 * mk.size
    for a, b in ((H, hu), (Mi, mu), (mn, mnu), (M1, m1u), (M2, m2u)):
        assert np.array_equal(a[mk].astype(np.int64), b[mk].astype(np.int64))


def test_buffer_eviction_and_newest_origin():
    from paper_2109_13176_b200 import synth
    w = synth.workload(0)
    g = dict(w.grid)
    g["buffer_frames"] = 2
    om = O.OracleMap(g)
    f = w.frames[0]
    with pytest.raises(RuntimeError):
        om.compute_maps()
    for i in range(3):
        om.shift((0.25 * i, 0.0, 0.0))
        om.integrate([(s.points, s.pose) for s in f.scans])
    assert len(om.buffer) == 2
    om.shift((5.0, 0.0, 0.0))  # a shift after the last integrate does not move the map
    om.compute_maps()
    assert np.array_equal(om.merged[5], om.buffer[-1].origin)
