"""c5 (1024x1024x128, 4.2M points, 8 sensors): GPU vs oracle at full size."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2109_13176_b200 import GvomMap, synth  # noqa: E402
from tests.gpu_helpers import compare_frame, compare_layers, layers_np  # noqa: E402

t = time.time()
w = synth.workload(4)
print("gen", time.time() - t, flush=True)
f = w.frames[0]
m = GvomMap(w.grid, max_points_per_frame=f.n_points)
m.shift(f.vehicle_xyz)
scans = [(torch.from_numpy(s.points).cuda(), s.pose, s.rings) for s in f.scans]
for _ in range(3):
    m.integrate_scan(scans)
    m.compute_maps()
m.synchronize()
m.set_timing(True)
m.stage_times()
for _ in range(10):
    m.integrate_scan(scans)
    m.compute_maps()
st = m.stage_times()
print("gpu stages us/step", {k: round(v[0] / 10 * 1000, 1) for k, v in st.items() if v[1]}, flush=True)
t = time.time()
om = O.OracleMap(w.grid)
om.shift(f.vehicle_xyz)
fm = om.integrate([(s.points, s.pose) for s in f.scans])
print("oracle integrate", time.time() - t, fm.k, fm.stats, flush=True)
t = time.time()
L = om.compute_maps()
print("oracle maps", time.time() - t, om.times, flush=True)
compare_frame(m, fm)
print("frame map bit-exact", flush=True)
compare_layers(layers_np(m), L)
print("layers ok", flush=True)
