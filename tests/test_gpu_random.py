"""Randomised GPU parity: seeded random grids (odd sizes), buffer depths,
thresholds, variant flags (8 cones, obstacle-free slope windows, rolling
map), one or two sensors with ordered or unordered clouds, random motion,
driven through the separate calls or gvom_step -- every frame against the
oracle (frame map, layers, merged or window map)."""
import numpy as np
import pytest
import torch

from paper_2109_13176_b200 import synth
from tests.gpu_helpers import run_sequence

pytestmark = pytest.mark.gpu


def _case(seed):
    rs = np.random.default_rng(1000 + seed)
    res = float(rs.choice([0.2, 0.25, 0.3]))
    nx, ny = int(rs.integers(20, 90)), int(rs.integers(20, 90))
    nz = int(rs.integers(int(3.2 / res) + 1, 70))  # the sensors (<= 1.2 m up) stay inside
    rolling = bool(rs.random() < 0.3)
    K = 1 if rolling else int(rs.integers(1, 5))
    grid = synth.grid_cfg(nx, ny, nz, res, buffer_frames=K)
    grid["slope_window"] = int(rs.choice([3, 5, 7]))
    grid["min_plane_points"] = int(rs.integers(3, 7))
    grid["min_obstacle_height"] = float(rs.uniform(0.1, 0.5))
    grid["max_obstacle_height"] = float(rs.uniform(0.8, 3.0))
    grid["density_threshold"] = float(rs.uniform(0.2, 0.8))
    grid["neg_obs_threshold"] = float(rs.uniform(0.2, 0.8))
    grid["neg_obs_search_cells"] = int(rs.integers(2, 14))
    grid["neg_8cone"] = bool(rs.random() < 0.4)
    grid["slope_skip_obstacles"] = bool(rs.random() < 0.4)
    grid["rolling"] = rolling
    w = synth.World()
    w.waves.append((float(rs.uniform(0.1, 0.5)), float(rs.uniform(5, 15)), 0.2, 0.0))
    w.boxes.append((1.5, 2.2, -1.0, 0.6, 0.0, float(rs.uniform(0.4, 1.5))))
    w.veg_boxes.append((-3.0, -1.4, 0.8, 2.8, 0.0, 1.2, float(rs.uniform(0.05, 0.3))))
    w.pits.append((-1.4, 0.1, -3.8, -2.2, float(rs.uniform(0.4, 1.2))))
    n_sensors = int(rs.integers(1, 3))
    rings = [int(rs.choice([12, 16, 24])) for _ in range(n_sensors)]
    lids = [synth.Lidar(r, int(rs.integers(120, 300)), (-35.0, 12.0)) for r in rings]
    frames = []
    x = y = 0.0
    for f in range(int(rs.integers(2, 5))):
        x += float(rs.uniform(-0.6, 0.9))
        y += float(rs.uniform(-0.5, 0.5))
        g = float(w.height(torch.tensor([x], dtype=torch.float64),
                           torch.tensor([y], dtype=torch.float64))[0])
        scans = []
        for i, lid in enumerate(lids):
            pose = synth.pose_matrix(synth.rot_zyx(float(rs.uniform(-3, 3)), 0.02, -0.01),
                                     (x + 0.3 * i, y - 0.2 * i, g + 1.0 + 0.2 * i))
            pts = synth.cast_scan(w, lid, pose, seed=seed, frame=f, sensor=i)
            # ordered (rings) or an unordered cloud (rings = 0)
            scans.append(synth.Scan(pts, pose, rings[i] if rs.random() < 0.7 else 0))
        frames.append(synth.Frame((x, y, g), scans))
    return synth.Workload(f"random{seed}", grid, frames, w), bool(rs.random() < 0.5)


@pytest.mark.parametrize("seed", range(40))
def test_random_configuration(seed):
    wl, use_step = _case(seed)
    run_sequence(wl, use_step=use_step)
