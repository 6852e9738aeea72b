"""Integrate one frame of a BASELINE config and run compute_maps `reps`
times (a small driver for ncu captures of the map kernels).
  python tools/run_maps.py [config_index] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_13176_b200 import GvomMap, synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = synth.workload(cfg)
f = w.frames[0]
m = GvomMap(w.grid, max_points_per_frame=f.n_points)
scans = [(torch.from_numpy(s.points).cuda(), s.pose, s.rings) for s in f.scans]
m.shift(f.vehicle_xyz)
m.integrate_scan(scans)
for _ in range(reps):
    m.compute_maps()
torch.cuda.synchronize()
print("ok", w.name)
