"""Stage times (CUDA events per launch, gvom_set_timing) of single ranks of
the ray-segment partition at c5, P ranks emulated on one GPU: where a rank's
fixed cost goes.   python tools/slab_rank_stages.py [P] [ranks...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_13176_b200 import GvomMap, parallel, synth  # noqa: E402


def main():
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    ranks = [int(a) for a in sys.argv[2:]] or [0, P // 2]
    w = synth.workload(4)
    f = w.frames[0]
    grid = dict(w.grid)
    grid["buffer_frames"] = 1
    scans = [(torch.from_numpy(s.points).cuda(), s.pose, s.rings) for s in f.scans]
    ys = parallel.slab_rows(grid["ny"], P)
    out = {}
    for r in ranks:
        m = GvomMap(grid, max_points_per_frame=f.n_points)
        m.shift(f.vehicle_xyz)

        def once():
            m.integrate_slab(scans, ys[r], ys[r + 1])
            m.compute_maps_slab(ys[r], ys[r + 1], 0)
            m.compute_maps_slab(ys[r], ys[r + 1], 1)

        once()
        torch.cuda.synchronize()
        m.set_timing(True)
        t0 = m.stage_times()
        reps = 5
        for _ in range(reps):
            once()
        torch.cuda.synchronize()
        t1 = m.stage_times()
        out[r] = {k: round((t1[k][0] - t0[k][0]) / reps * 1000, 1) for k in t1
                  if t1[k][1] > t0[k][1]}
        out[r]["launches_per_rep"] = sum(t1[k][1] - t0[k][1] for k in t1
                                         if k not in ("integrate", "maps")) / reps
        del m
        torch.cuda.empty_cache()
    print(json.dumps({"P": P, "slabs": ys, "us_per_rank_call": out}))


if __name__ == "__main__":
    main()
