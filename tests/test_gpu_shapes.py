"""GPU parity across grid shapes and layer parameters the shipped configs do
not exercise: nz not a multiple of 32 (columns straddle bitmask words), nx
not a multiple of 32, non-square maps, K = 1 and K = 3 buffers with motion,
slope windows N = 3 / 7 / 9, other band / density / Delta-H thresholds and
cone distances.  Every case runs the full update through the C ABI and
compares LUT, data rows, merged map and all layers with the oracle."""
import math

import numpy as np
import pytest

from paper_2109_13176_b200 import synth
from tests.gpu_helpers import run_sequence

pytestmark = pytest.mark.gpu


def _world_frames(n_frames, step, seed, rings=24, columns=360):
    w = synth.World()
    w.waves.append((0.4, 12.0, 0.3, 0.0))
    w.boxes.append((2.0, 2.6, -1.0, 0.5, 0.0, 0.9))
    w.veg_boxes.append((-3.0, -1.5, 1.0, 3.0, 0.0, 1.2, 0.15))
    w.pits.append((-1.0, 0.5, -4.0, -2.5, 0.8))
    lid = synth.Lidar(rings, columns, (-35.0, 10.0))
    frames = []
    for f in range(n_frames):
        x = step * f
        g = float(w.height(*[__import__("torch").tensor([v], dtype=__import__("torch").float64)
                              for v in (x, 0.2 * x)])[0])
        pose = synth.pose_matrix(synth.rot_zyx(0.1 * f, 0.02, -0.01), (x, 0.2 * x, g + 1.2))
        pts = synth.cast_scan(w, lid, pose, seed=seed, frame=f, sensor=0)
        frames.append(synth.Frame((x, 0.2 * x, g), [synth.Scan(pts, pose, rings)]))
    return w, frames


CASES = [
    # (nx, ny, nz, res, K, overrides)
    (48, 40, 20, 0.3, 1, {}),
    (70, 33, 12, 0.25, 3, {"slope_window": 3}),
    (64, 96, 40, 0.2, 3, {"slope_window": 7, "min_plane_points": 6}),
    (37, 37, 7, 0.5, 1, {"slope_window": 9, "neg_obs_search_cells": 3}),
    (96, 64, 33, 0.2, 2, {"min_obstacle_height": 0.1, "max_obstacle_height": 1.0,
                          "density_threshold": 0.3, "neg_obs_threshold": 0.2}),
    # obstacle band of 70 voxels: reaches past k_columns' 64-z occupancy window
    (40, 40, 96, 0.2, 2, {"max_obstacle_height": 14.0}),
    # 1600-wide lines: the cone sweep's temporally blocked kernel with 3-4
    # segments per warp (k_negative_tb<4>)
    (1600, 40, 16, 0.25, 1, {}),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_shapes_and_parameters(case):
    nx, ny, nz, res, K, over = CASES[case]
    grid = synth.grid_cfg(nx, ny, nz, res, buffer_frames=K)
    grid.update(over)
    w, frames = _world_frames(4, 0.37 + 0.1 * case, 100 + case)
    wl = synth.Workload(f"shape{case}", grid, frames, w)
    run_sequence(wl, check_every=1)


def test_slope_skip_obstacles_flag():
    # GVOM_FLAG_SLOPE_SKIP_OBSTACLES (SPEC S:338 variant) against the oracle
    grid = synth.grid_cfg(64, 64, 24, 0.25, buffer_frames=2)
    grid["slope_skip_obstacles"] = True
    w, frames = _world_frames(3, 0.3, 77)
    run_sequence(synth.Workload("skip_obstacles", grid, frames, w))


@pytest.mark.parametrize("case", [0, 1, 3])
def test_neg_8cone_flag_shapes(case):
    # GVOM_FLAG_NEG_8CONE (SPEC S:327 / NEXT-3 variant, reading B8) against
    # or_negative8: odd shapes, K = 3 .. 24 cone distances, tiles straddling edges
    nx, ny, nz, res, K, over = CASES[case]
    grid = synth.grid_cfg(nx, ny, nz, res, buffer_frames=K)
    grid.update(over)
    grid["neg_8cone"] = True
    w, frames = _world_frames(3, 0.41 + 0.1 * case, 300 + case)
    run_sequence(synth.Workload(f"neg8_{case}", grid, frames, w))


def test_neg_8cone_flag_c2_and_c4():
    # the shipped workloads (K = 24 and 30 cone cells) with the 8-cone search
    for i in (1, 3):
        wl = synth.workload(i)
        grid = dict(wl.grid)
        grid["neg_8cone"] = True
        run_sequence(synth.Workload(wl.name + "_neg8", grid, wl.frames, wl.world),
                     check_merged=False)
