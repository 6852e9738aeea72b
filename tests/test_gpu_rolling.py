"""GVOM_FLAG_ROLLING (NEXT-3 rolling map, reading B9) against the oracle's
rolling map, frame by frame: the scan's frame map, the dense window map
(u64 counts, min_dz) and every layer, under standing still, monotone motion,
back-and-forth motion that leaves and re-enters the window, vertical motion,
and jumps larger than the window; through the separate calls and gvom_step."""
import dataclasses

import numpy as np
import pytest
import torch

from paper_2109_13176_b200 import synth
from tests.gpu_helpers import run_sequence

pytestmark = pytest.mark.gpu


def _frames(path, seed=11, rings=16, columns=300):
    w = synth.World()
    w.waves.append((0.3, 9.0, 0.2, 0.0))
    w.boxes.append((1.5, 2.1, -1.0, 0.4, 0.0, 0.8))
    w.veg_boxes.append((-2.5, -1.2, 0.8, 2.5, 0.0, 1.1, 0.15))
    w.pits.append((-1.2, 0.2, -3.5, -2.0, 0.7))
    lid = synth.Lidar(rings, columns, (-35.0, 10.0))
    frames = []
    for f, (x, y, dz) in enumerate(path):
        g = float(w.height(torch.tensor([x], dtype=torch.float64),
                           torch.tensor([y], dtype=torch.float64))[0]) + dz
        pose = synth.pose_matrix(synth.rot_zyx(0.07 * f, 0.01, 0.0), (x, y, g + 1.1))
        pts = synth.cast_scan(w, lid, pose, seed=seed, frame=f, sensor=0)
        frames.append(synth.Frame((x, y, g), [synth.Scan(pts, pose, rings)]))
    return w, frames


def _grid(nz=20):
    g = synth.grid_cfg(48, 40, nz, 0.3, buffer_frames=1)
    g["rolling"] = True
    return g


PATHS = {
    "still": [(0.0, 0.0, 0.0)] * 4,
    "forward": [(0.4 * i, 0.1 * i, 0.0) for i in range(6)],
    "back_and_forth": [(0.0, 0.0, 0.0), (1.3, 0.2, 0.0), (0.2, -0.5, 0.0), (-1.1, 0.0, 0.0),
                       (0.6, 0.7, 0.0)],
    "vertical": [(0.0, 0.0, 0.0), (0.2, 0.0, 0.7), (0.4, 0.0, -0.5), (0.6, 0.0, 1.4)],
    "jumps": [(0.0, 0.0, 0.0), (20.0, 0.0, 0.0), (20.3, 1.0, 0.0), (0.0, 0.0, 0.0)],
}


@pytest.mark.parametrize("name", list(PATHS))
def test_rolling_matches_oracle(name):
    w, frames = _frames(PATHS[name])
    run_sequence(synth.Workload("roll_" + name, _grid(), frames, w))


@pytest.mark.parametrize("name", ["back_and_forth", "jumps"])
def test_rolling_through_gvom_step(name):
    w, frames = _frames(PATHS[name], seed=12)
    m, _ = run_sequence(synth.Workload("roll_step_" + name, _grid(), frames, w), use_step=True)
    assert m.graph_stats()["graph_launches"] == len(frames)


def test_rolling_c3_motion_sequence():
    wl = synth.config3(speed=12.0, n_frames=8, columns=1024)
    grid = dict(wl.grid)
    grid["buffer_frames"] = 1
    grid["rolling"] = True
    run_sequence(synth.Workload(wl.name + "_roll", grid, wl.frames, wl.world), check_every=4)


def test_rolling_odd_nz_scalar_path():
    # nz not a multiple of 4: the accumulate kernel's one-voxel-per-thread path
    w, frames = _frames(PATHS["vertical"] + PATHS["back_and_forth"], seed=13)
    run_sequence(synth.Workload("roll_nz21", _grid(21), frames, w))
