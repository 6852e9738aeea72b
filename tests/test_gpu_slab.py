"""GPU test of the multi-GPU slab partition's kernels with P
ranks emulated in one process on one GPU: every rank has its own handle and
its share of the sensors; the collectives (reduce-scatter of miss grids,
all-to-all of return records, all-gather of slab counts and surface rows) are
played with torch ops on the device.  The slabs must reproduce the single-GPU
frame bit for bit: LUT (global ranks = slab base + local rank), data rows,
height / density / hard / soft of the slab rows, and slope / roughness /
negative obstacles of the whole map.  (No rank waits on another inside a
kernel, so this emulation is faithful.)
"""
import numpy as np
import pytest
import torch

from paper_2109_13176_b200 import GvomMap, parallel, synth
from tests.gpu_helpers import layers_np

pytestmark = pytest.mark.gpu


def _run(w, P):
    grid = dict(w.grid)
    grid["buffer_frames"] = 1
    f = w.frames[0]
    scans = [(torch.from_numpy(s.points).cuda(), s.pose, s.rings) for s in f.scans]
    # single GPU reference
    ref = GvomMap(grid, max_points_per_frame=f.n_points)
    ref.shift(f.vehicle_xyz)
    ref.integrate_scan(scans)
    ref.compute_maps()
    ref_lut, ref_data, _ = ref.export_frame(0)
    ref_layers = layers_np(ref)
    nx, ny, nz = ref.nx, ref.ny, ref.nz
    ys = parallel.slab_rows(ny, P)
    row = nx * nz
    # ranks: sensors dealt round-robin (some ranks may hold none)
    ranks = []
    for r in range(P):
        m = GvomMap(grid, max_points_per_frame=f.n_points)
        m.shift(f.vehicle_xyz)
        miss = torch.empty(nx * ny * nz, dtype=torch.int32, device="cuda")
        rec = torch.empty(f.n_points + 1, dtype=torch.int64, device="cuda")
        mine = [s for i, s in enumerate(scans) if i % P == r]
        counts = m.partial_scan(mine, miss, rec, ys)
        ranks.append((m, miss, rec, counts))
    # emulated reduce-scatter + all-to-all
    total_miss = sum(x[1] for x in ranks)
    offs = [np.concatenate([[0], np.cumsum(x[3])]) for x in ranks]
    ks, states = [], []
    for r in range(P):
        miss_slab = total_miss[ys[r] * row:ys[r + 1] * row].contiguous()
        recv = torch.cat([x[2][int(o[r]):int(o[r + 1])] for x, o in zip(ranks, offs)]).contiguous()
        m = ranks[r][0]
        k = m.slab_occupancy(ys[r], ys[r + 1], recv, recv.numel())
        ks.append(k)
        states.append((miss_slab, recv))
    assert sum(ks) == ref_data["hits"].shape[0]
    bases = np.concatenate([[0], np.cumsum(ks)])
    for r in range(P):
        m = ranks[r][0]
        miss_slab, recv = states[r]
        m.slab_finalize(ys[r], ys[r + 1], miss_slab, recv, recv.numel())
        m.compute_maps_slab(ys[r], ys[r + 1], 0)
    # emulated all-gather of the surface rows
    surf = torch.cat([ranks[r][0].surface()[ys[r]:ys[r + 1]] for r in range(P)])
    for r in range(P):
        m = ranks[r][0]
        m.surface().copy_(surf)
        m.compute_maps_slab(ys[r], ys[r + 1], 1)
    torch.cuda.synchronize()
    for r in range(P):
        m = ranks[r][0]
        lut, data, _ = m.export_frame(0)
        v0, v1 = ys[r] * row, ys[r + 1] * row
        got = lut[v0:v1].astype(np.int64)
        got = np.where(got >= 0, got + bases[r], got)
        assert np.array_equal(got, ref_lut[v0:v1].astype(np.int64)), f"rank {r} LUT"
        for k_ in ("hits", "misses", "min_dz", "m1", "m2"):
            assert np.array_equal(data[k_], ref_data[k_][bases[r]:bases[r + 1]]), (r, k_)
        lay = layers_np(m)
        sl = slice(ys[r], ys[r + 1])
        for k_ in ("height", "density", "hard", "soft"):
            a, b = lay[k_][sl], ref_layers[k_][sl]
            assert np.array_equal(np.nan_to_num(a, nan=-7), np.nan_to_num(b, nan=-7)), (r, k_)
        for k_ in ("slope", "roughness", "neg"):
            a, b = lay[k_], ref_layers[k_]
            assert np.array_equal(np.nan_to_num(a, nan=-7), np.nan_to_num(b, nan=-7)), (r, k_)


@pytest.mark.parametrize("P", [2, 4])
def test_slab_partition_c4_matches_single_gpu(P):
    _run(synth.workload(3), P)


def test_slab_partition_c1_eight_ranks():
    _run(synth.workload(0), 8)


@pytest.mark.slow
def test_slab_partition_c5_eight_ranks():
    _run(synth.workload(4), 8)
