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




def cpu_submit(cfg=1, steps=200):
    """CPU time to enqueue a full update (no synchronisation) vs GPU time."""
    import time
    w = [synth.config1, synth.config2, None, synth.config4, synth.config5][cfg]()
    f = w.frames[0]
    m = GvomMap(w.grid, max_points_per_frame=f.n_points)
    scans = [(torch.from_numpy(s.points).cuda(), s.pose, s.rings) for s in f.scans]
    m.shift(f.vehicle_xyz); m.integrate_scan(scans); m.compute_maps()
    out = m.export_layers()
    for _ in range(10):
        m.shift(f.vehicle_xyz); m.integrate_scan(scans); m.compute_maps(); m.export_layers(out)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(steps):
        m.shift(f.vehicle_xyz); m.integrate_scan(scans); m.compute_maps(); m.export_layers(out)
    t1 = time.perf_counter()
    ev1.record(); torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"cpu submit {1e6*(t1-t0)/steps:.1f} us/step, wall {1e6*(t2-t0)/steps:.1f} us/step, "
          f"gpu events {1000*ev0.elapsed_time(ev1)/steps:.1f} us/step")
    # per-call CPU cost
    for name, fn in (("shift", lambda: m.shift(f.vehicle_xyz)), ("integrate", lambda: m.integrate_scan(scans)),
                     ("compute_maps", lambda: m.compute_maps()), ("export", lambda: m.export_layers(out))):
        torch.cuda.synchronize(); t = time.perf_counter()
        for _ in range(50):
            fn()
        torch.cuda.synchronize()
        print(f"  {name}: {1e6*(time.perf_counter()-t)/50:.1f} us/call (incl. GPU)")


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "cpu":
        cpu_submit(int(sys.argv[1]))
    else:
        main(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
