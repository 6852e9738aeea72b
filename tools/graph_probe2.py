"""Probe: gvom_step GPU time with / without the L2 flush and with / without
captured stage-timing events.  Not part of the product."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2109_13176_b200 import GvomMap, LAYERS, synth  # noqa: E402

w = synth.workload(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
f = w.frames[0]
dev = torch.device("cuda")
s = torch.cuda.Stream()
m = GvomMap(w.grid, max_points_per_frame=w.points_per_frame, stream=s)
scans = [(torch.from_numpy(x.points).to(dev), x.pose, x.rings) for x in f.scans]
out = {k: torch.empty((m.ny, m.nx), dtype=(torch.uint8 if k in ("hard", "soft", "neg")
                                           else torch.float32), device=dev) for k in LAYERS}
flush = torch.empty(256 << 18, dtype=torch.float32, device=dev)
n = 30
with torch.cuda.stream(s):
    for timing in (False, True):
        for fl in (False, True):
            for graph in (False, True):
                m.set_timing(timing, stages=["raycast"])
                m.stage_times()
                evs = []
                for i in range(n + 3):
                    if fl:
                        flush.zero_()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(s)
                    if graph:
                        m.step(f.vehicle_xyz, scans, out)
                    else:
                        m.shift(f.vehicle_xyz); m.integrate_scan(scans); m.compute_maps(); m.export_layers(out)
                    b.record(s)
                    evs.append((a, b))
                s.synchronize()
                t = sum(a.elapsed_time(b) for a, b in evs[3:]) / n
                st = m.stage_times()["raycast"]
                print(f"P2 timing={timing:d} flush={fl:d} graph={graph:d} step_ms={t:.4f} ray_ms={st[0]/max(st[1],1):.4f}")
