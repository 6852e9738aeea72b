"""Pins of the rolling-map oracle (NEXT-3 "rolling in-place map (K = inf)";
DESIGN.md reading B9) against the pinned K-buffer combine (O7) and a per-voxel
definition of the window move:

- roll_window keeps exactly the voxels whose world coordinates stay inside
  the window (brute force over world coordinates);
- with the vehicle standing still, the rolling map after n scans equals the
  K >= n buffer combine (same origin: the combine is a plain sum);
- with motion monotone in every axis the windows nest, so the rolling map
  still equals the K >= n combine;
- leaving the window entirely and coming back drops the old scans: the
  rolling map equals the last scan alone, unlike the K = 3 combine.
"""
import numpy as np
import torch

from oracle import oracle as O
from paper_2109_13176_b200 import synth


def test_roll_window_matches_world_coordinates():
    rs = np.random.default_rng(3)
    dims = (7, 5, 4)
    nx, ny, nz = dims
    V = nx * ny * nz
    acc = (rs.integers(1, 9, V).astype(np.uint64), rs.integers(1, 9, V).astype(np.uint64),
           rs.integers(1, 9, V).astype(np.uint32), rs.integers(1, 9, V).astype(np.uint64),
           rs.integers(1, 9, V).astype(np.uint64))
    for d in [(1, 0, 0), (-2, 3, 1), (0, 0, -3), (7, 0, 0), (-3, -4, 2)]:
        out = O.roll_window(dims, acc, np.array(d))
        for L in range(V):
            z, x, y = L % nz, (L // nz) % nx, L // (nz * nx)
            ox, oy, oz = x + d[0], y + d[1], z + d[2]  # old logical coordinates
            inside = 0 <= ox < nx and 0 <= oy < ny and 0 <= oz < nz
            Lo = oz + nz * (ox + nx * oy)
            for a, b, empty in zip(out, acc, (0, 0, 0xFFFFFFFF, 0, 0)):
                assert a[L] == (b[Lo] if inside else empty), (d, L)


def _frames(xs, seed=5):
    w = synth.World()
    w.waves.append((0.3, 9.0, 0.2, 0.0))
    w.boxes.append((1.5, 2.1, -1.0, 0.4, 0.0, 0.8))
    w.pits.append((-1.2, 0.2, -3.5, -2.0, 0.7))
    lid = synth.Lidar(16, 240, (-35.0, 10.0))
    frames = []
    for f, x in enumerate(xs):
        g = float(w.height(torch.tensor([x], dtype=torch.float64),
                           torch.tensor([0.1 * x], dtype=torch.float64))[0])
        pose = synth.pose_matrix(synth.rot_zyx(0.05 * f, 0.01, 0.0), (x, 0.1 * x, g + 1.1))
        pts = synth.cast_scan(w, lid, pose, seed=seed, frame=f, sensor=0)
        frames.append(synth.Frame((x, 0.1 * x, g), [synth.Scan(pts, pose, 16)]))
    return frames


def _run(grid, frames):
    om = O.OracleMap(grid)
    for f in frames:
        om.shift(f.vehicle_xyz)
        om.integrate([(s.points, s.pose) for s in f.scans])
    L = om.compute_maps()
    return om, L


def _same(a, b):
    ma, mb = a[0].merged, b[0].merged
    for x, y in zip(ma, mb):
        assert np.array_equal(x, y)
    for k in ("height", "density", "slope", "roughness", "spread"):
        assert np.array_equal(np.nan_to_num(getattr(a[1], k), nan=-7),
                              np.nan_to_num(getattr(b[1], k), nan=-7)), k
    for k in ("hard", "soft", "neg"):
        assert np.array_equal(getattr(a[1], k), getattr(b[1], k)), k


def _grid(K, rolling):
    g = synth.grid_cfg(48, 40, 16, 0.3, buffer_frames=K)
    g["rolling"] = rolling
    return g


def test_rolling_equals_combine_when_standing_still():
    frames = _frames([0.0] * 4)
    _same(_run(_grid(1, True), frames), _run(_grid(4, False), frames))


def test_rolling_equals_combine_for_monotone_motion():
    frames = _frames([0.0, 0.45, 1.1, 1.6, 2.4])
    a = _run(_grid(1, True), frames)
    _same(a, _run(_grid(5, False), frames))
    assert int(a[0].merged[0].sum()) > 0


def test_rolling_forgets_a_window_it_left():
    far = 48 * 0.3 + 3.0
    frames = _frames([0.0, far, 0.0])
    roll = _run(_grid(1, True), frames)
    last = _run(_grid(1, False), frames)  # the last scan alone
    buf3 = _run(_grid(3, False), frames)
    _same(roll, last)
    assert not np.array_equal(roll[0].merged[0], buf3[0].merged[0])
