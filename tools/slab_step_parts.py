"""Where a partitioned (ray-segment) step's time goes at N = 1 on c5: CUDA
events around the points all-gather, integrate_slab, the two map phases and
the row gathers, per step.   torchrun --nproc-per-node 1 tools/slab_step_parts.py"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_13176_b200 import GvomMap, parallel, synth  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    w = synth.workload(4)
    f = w.frames[0]
    grid = dict(w.grid)
    grid["buffer_frames"] = 1
    mine = [(torch.from_numpy(s.points).to(dev), s.pose, s.rings) for s in f.scans]
    meta = [(0, s.points.shape[0], s.pose, s.rings) for s in f.scans]
    stream = torch.cuda.Stream(device=dev)
    m = GvomMap(grid, max_points_per_frame=f.n_points, device=dev, stream=stream)
    sm = parallel.SegmentMapper(m)
    flush = torch.empty((256 << 20) // 4, dtype=torch.float32, device=dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    rows = []
    with torch.cuda.stream(stream):
        for it in range(8):
            flush.zero_()
            e = [ev() for _ in range(6)]
            e[0].record(stream)
            m.shift(f.vehicle_xyz)
            scans = parallel.all_gather_points(mine, meta)
            e[1].record(stream)
            m.integrate_slab(scans, sm.y0, sm.y1)
            e[2].record(stream)
            m.compute_maps_slab(sm.y0, sm.y1, 0)
            e[3].record(stream)
            parallel.gather_rows(m.surface(), sm.y0, sm.y1, None, sm.ys)
            e[4].record(stream)
            m.compute_maps_slab(sm.y0, sm.y1, 1)
            e[5].record(stream)
            e[5].synchronize()
            rows.append([round(e[i].elapsed_time(e[i + 1]), 3) for i in range(5)])
    print(json.dumps({"parts_ms": ["gather_points", "integrate_slab", "maps0", "gather_rows",
                                   "maps1"], "steps": rows}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
