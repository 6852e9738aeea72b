"""Per-rank work of the partitioned path, P ranks emulated on ONE GPU (no
rank waits on another: each rank's calls run alone, back to back), for P = 1,
2, 4, 8 on BASELINE configs[4] (c5).  For every rank: CUDA events around its
own calls -- ray segments: gvom_integrate_slab (all sensors, its rows) +
compute_maps_slab phase 0 + phase 1; reduce-scatter: gvom_partial_scan of its
sensors + slab_occupancy + slab_finalize (the NCCL exchange itself is not
emulated) + phase 0 + phase 1.  Reports the max and mean over ranks: the
compute part of a strong-scaling step (collectives come on top: the segment
path's points all-gather moves 16 B per point, the reduce-scatter path's
exchange (P-1)/P * 4V bytes per rank).  Ray segments twice: equal-row slabs
and slabs balanced on the frame's per-row work (gvom_row_work +
parallel.balanced_slab_rows, as SegmentMapper.rebalance does).

  python tools/slab_scaling.py [config_index] [frames]   -> one JSON line
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_13176_b200 import GvomMap, parallel, synth  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def segments_rank_times(grid, f, scans, npts, ys, reps):
    """Each rank's integrate_slab + compute_maps_slab (phase 0 + 1), alone."""
    times = []
    for r in range(len(ys) - 1):
        m = GvomMap(grid, max_points_per_frame=npts)
        m.shift(f.vehicle_xyz)
        m.integrate_slab(scans, ys[r], ys[r + 1])  # warm-up
        m.compute_maps_slab(ys[r], ys[r + 1], 0)
        m.compute_maps_slab(ys[r], ys[r + 1], 1)
        torch.cuda.synchronize()
        best = None
        for _ in range(reps):
            a, b = ev(), ev()
            a.record(m.stream)
            m.integrate_slab(scans, ys[r], ys[r + 1])
            m.compute_maps_slab(ys[r], ys[r + 1], 0)
            m.compute_maps_slab(ys[r], ys[r + 1], 1)
            b.record(m.stream)
            b.synchronize()
            t = a.elapsed_time(b)
            best = t if best is None else min(best, t)
        times.append(best)
        del m
        torch.cuda.empty_cache()
    return times


def reduce_scatter_rank_times(grid, f, scans, npts, ys, reps):
    """Each rank's compute of the reduce-scatter path (no exchange), alone."""
    P = len(ys) - 1
    V = grid["nx"] * grid["ny"] * grid["nz"]
    row = grid["nx"] * grid["nz"]
    times = []
    for r in range(P):
        m = GvomMap(grid, max_points_per_frame=npts)
        m.shift(f.vehicle_xyz)
        mine = [s for i, s in enumerate(scans) if i % P == r]
        miss = torch.zeros(V, dtype=torch.int32, device="cuda")
        rec = torch.empty(npts + 1, dtype=torch.int64, device="cuda")
        best = None
        for it in range(reps + 1):
            a, b = ev(), ev()
            a.record(m.stream)
            counts = m.partial_scan(mine, miss, rec, ys)
            # this rank's slab from its own grid / records only: the kernels
            # an exchange would feed, on the same sizes
            o0 = int(sum(counts[:r]))
            mr = rec[o0:o0 + counts[r]]  # this rank's own returns in its slab
            m.slab_occupancy(ys[r], ys[r + 1], mr, counts[r])
            m.slab_finalize(ys[r], ys[r + 1], miss[ys[r] * row:ys[r + 1] * row].contiguous(),
                            mr, counts[r], 0)
            m.compute_maps_slab(ys[r], ys[r + 1], 0)
            m.compute_maps_slab(ys[r], ys[r + 1], 1)
            b.record(m.stream)
            b.synchronize()
            t = a.elapsed_time(b)
            if it > 0:
                best = t if best is None else min(best, t)
        times.append(best)
        del m, miss, rec
        torch.cuda.empty_cache()
    return times


def summary(times, ys, **extra):
    return {"max_ms": max(times), "mean_ms": float(np.mean(times)), "ranks_ms": times,
            "slabs": list(ys), **extra}


def run(cfg=4, reps=3):
    w = synth.workload(cfg)
    f = w.frames[0]
    grid = dict(w.grid)
    grid["buffer_frames"] = 1
    scans = [(torch.from_numpy(s.points).cuda(), s.pose, s.rings) for s in f.scans]
    npts = f.n_points
    V = grid["nx"] * grid["ny"] * grid["nz"]
    out = {"workload": w.name, "points": npts, "emulated": "P ranks on one GPU, each rank's "
           "calls timed alone (no collective)", "segments": {}, "segments_balanced": {},
           "reduce_scatter": {}}
    # the frame's per-row work (gvom_row_work on one GPU) -> balanced bounds
    one = GvomMap(grid, max_points_per_frame=npts)
    one.shift(f.vehicle_xyz)
    one.integrate_scan(scans)
    row_work = one.row_work().cpu().numpy()
    del one
    for P in (1, 2, 4, 8):
        ys = parallel.slab_rows(grid["ny"], P)
        out["segments"][P] = summary(segments_rank_times(grid, f, scans, npts, ys, reps), ys)
        yb = parallel.balanced_slab_rows(row_work, P)
        out["segments_balanced"][P] = summary(
            segments_rank_times(grid, f, scans, npts, yb, reps), yb)
        out["reduce_scatter"][P] = summary(
            reduce_scatter_rank_times(grid, f, scans, npts, ys, reps), ys,
            exchange_bytes_per_rank=int((P - 1) / P * 4 * V))
    return out


if __name__ == "__main__":
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    print(json.dumps(run(cfg)))
