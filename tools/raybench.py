"""Micro-benchmark of the integrate stages on one workload (stage event times)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_13176_b200 import GvomMap, synth  # noqa: E402


def main(cfg=1, steps=50):
    w = [synth.config1, synth.config2, None, synth.config4, synth.config5][cfg]()
    f = w.frames[0]
    m = GvomMap(w.grid, max_points_per_frame=f.n_points)
    scans = [(torch.from_numpy(s.points).cuda(), s.pose, s.rings) for s in f.scans]
    m.shift(f.vehicle_xyz)
    for _ in range(5):
        m.integrate_scan(scans)
        m.compute_maps()
    m.synchronize()
    m.set_timing(True)
    m.stage_times()
    for _ in range(steps):
        m.integrate_scan(scans)
        m.compute_maps()
    st = m.stage_times()
    print(os.environ.get("GVOM_RAY_BLOCK", "default"),
          {k: round(v[0] / steps * 1000, 2) for k, v in st.items() if v[1]})


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
