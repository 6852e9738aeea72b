"""Probe: how much of a step is launch / host overhead?  Times the c2 step
eagerly and as a replayed CUDA graph captured around the library calls (same
inputs every replay, timing instrumentation off).  Not part of the product."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2109_13176_b200 import GvomMap, LAYERS, synth  # noqa: E402


def main(cfg=1, n=50):
    w = synth.workload(cfg)
    f = w.frames[0]
    dev = torch.device("cuda")
    s = torch.cuda.Stream()
    m = GvomMap(w.grid, max_points_per_frame=w.points_per_frame, stream=s)
    scans = [(torch.from_numpy(x.points).to(dev), x.pose, x.rings) for x in f.scans]
    out = {k: torch.empty((m.ny, m.nx), dtype=(torch.uint8 if k in ("hard", "soft", "neg")
                                               else torch.float32), device=dev) for k in LAYERS}

    def step():
        m.shift(f.vehicle_xyz)
        m.integrate_scan(scans)
        m.compute_maps()
        m.export_layers(out)

    with torch.cuda.stream(s):
        for _ in range(5):
            step()
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(s)
        for _ in range(n):
            step()
        e1.record(s)
        t1 = time.perf_counter()
        s.synchronize()
        eager = e0.elapsed_time(e1) / n
        cpu = (t1 - t0) / n * 1e3
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step()
        for _ in range(3):
            g.replay()
        s.synchronize()
        e0.record(s)
        for _ in range(n):
            g.replay()
        e1.record(s)
        s.synchronize()
        graph = e0.elapsed_time(e1) / n
        # the library's own graph path (capture + exec update + launch per step)
        for _ in range(3):
            m.step(f.vehicle_xyz, scans, out)
        s.synchronize()
        t0 = time.perf_counter()
        e0.record(s)
        for _ in range(n):
            m.step(f.vehicle_xyz, scans, out)
        e1.record(s)
        t1 = time.perf_counter()
        s.synchronize()
        gstep = e0.elapsed_time(e1) / n
        gcpu = (t1 - t0) / n * 1e3
    print(f"GRAPH cfg={w.name} eager_ms={eager:.4f} cpu_submit_ms={cpu:.4f} graph_ms={graph:.4f} "
          f"gvom_step_ms={gstep:.4f} gvom_step_cpu_ms={gcpu:.4f} {m.graph_stats()}")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
