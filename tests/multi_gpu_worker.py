"""Worker of tests/test_gpu_multiproc.py, run under torchrun with one process
per GPU (NCCL): every slab mode of the partitioned path (ray segments,
reduce-scatter, symmetric-memory fused finalize) on one frame, its layers'
slab rows all-gathered and compared on every rank with a single-GPU map of
the same frame (bit-exact; slope / roughness within the contract tolerance)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_13176_b200 import LAYERS, GvomMap, parallel, synth  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, P = dist.get_rank(), dist.get_world_size()
    w = synth.workload(int(os.environ.get("GVOM_MP_CONFIG", "3")))
    f = w.frames[0]
    grid = dict(w.grid)
    grid["buffer_frames"] = 1
    scans = [(torch.from_numpy(s.points).to(dev), s.pose, s.rings) for s in f.scans]
    ref = GvomMap(grid, max_points_per_frame=f.n_points, device=dev)
    ref.shift(f.vehicle_xyz)
    ref.integrate_scan(scans)
    ref.compute_maps()
    want = {k: v.cpu().numpy() for k, v in ref.export_layers().items()}
    mine = [s for i, s in enumerate(scans) if i % P == rank]
    for mode in ("segments", "segments_balanced", "reduce_scatter", "fused"):
        m = GvomMap(grid, max_points_per_frame=f.n_points, device=dev)
        sm = (parallel.SegmentMapper(m) if mode.startswith("segments") else
              parallel.SlabMapper(m, ep_capacity=f.n_points, fused=(mode == "fused")))
        m.shift(f.vehicle_xyz)
        sm.integrate(mine)
        sm.compute_maps()
        if mode == "segments_balanced":  # bounds from this frame's row work, then again
            sm.rebalance()
            m.shift(f.vehicle_xyz)
            sm.integrate(mine)
            sm.compute_maps()
        lay = m.export_layers()
        m.synchronize()
        for k in LAYERS:
            t = lay[k].contiguous()
            parallel.gather_rows(t, sm.y0, sm.y1, None, sm.ys)
            got = t.cpu().numpy()
            if k in ("slope", "roughness", "spread"):
                ok = np.array_equal(np.isnan(got), np.isnan(want[k]))
                fin = ~np.isnan(want[k])
                ok = ok and np.all(np.abs(got[fin] - want[k][fin]) <= 1e-4 + 1e-5 * np.abs(
                    want[k][fin]))
            else:
                ok = np.array_equal(np.nan_to_num(got, nan=-7), np.nan_to_num(want[k], nan=-7))
            assert ok, (mode, k, rank)
        if rank == 0:
            print(f"MULTI-GPU {mode} P={P} ok", flush=True)
        del sm, m
    # ray segments with motion: K = 8 buffered maps in symmetric memory, the
    # shifted rows of other slabs read from their owners over NVLink
    w3 = synth.config3(speed=12.0, n_frames=6, columns=512)
    g3 = dict(w3.grid)
    npts = w3.points_per_frame
    ref = GvomMap(g3, max_points_per_frame=npts, device=dev)
    m, sm = parallel.segment_map(g3, npts, dev)
    for f in w3.frames:
        sc = [(torch.from_numpy(s.points).to(dev), s.pose, s.rings) for s in f.scans]
        ref.shift(f.vehicle_xyz)
        ref.integrate_scan(sc)
        m.shift(f.vehicle_xyz)
        sm.integrate(sc, gathered=True)
    ref.compute_maps()
    want = {k: v.cpu().numpy() for k, v in ref.export_layers().items()}
    sm.compute_maps()
    lay = m.export_layers()
    m.synchronize()
    sl = slice(sm.y0, sm.y1)
    for k in LAYERS:
        got = lay[k].cpu().numpy()[sl]
        assert np.array_equal(np.nan_to_num(got, nan=-7), np.nan_to_num(want[k][sl], nan=-7)), (
            "segments_motion", k, rank)
    if rank == 0:
        print(f"MULTI-GPU segments_motion P={P} ok", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
