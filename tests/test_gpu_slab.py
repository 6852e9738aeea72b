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
import dataclasses

import numpy as np
import pytest
import torch

from paper_2109_13176_b200 import GvomMap, parallel, synth
from tests.gpu_helpers import layers_np

pytestmark = pytest.mark.gpu


def _run(w, P, peers=False, **over):
    grid = dict(w.grid)
    grid["buffer_frames"] = 1
    grid.update(over)
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
    grid_ptrs = [x[1].data_ptr() for x in ranks]  # the ranks' partial miss grids
    for r in range(P):
        m = ranks[r][0]
        miss_slab, recv = states[r]
        if peers:  # fused: the finalize sums the P grids itself (no reduce-scatter)
            m.slab_finalize_peers(ys[r], ys[r + 1], grid_ptrs, recv, recv.numel(), int(bases[r]))
        else:
            m.slab_finalize(ys[r], ys[r + 1], miss_slab, recv, recv.numel(), int(bases[r]))
        m.compute_maps_slab(ys[r], ys[r + 1], 0)
    # emulated all-gather of the surface rows (+ obstacle rows when slope
    # windows skip obstacles, as parallel.SlabMapper does)
    surf = torch.cat([ranks[r][0].surface()[ys[r]:ys[r + 1]] for r in range(P)])
    obst = None
    if grid.get("slope_skip_obstacles", False):
        obst = [torch.cat([ranks[r][0].obstacles()[i][ys[r]:ys[r + 1]] for r in range(P)])
                for i in range(2)]
    for r in range(P):
        m = ranks[r][0]
        m.surface().copy_(surf)
        if obst is not None:
            for t, full in zip(m.obstacles(), obst):
                t.copy_(full)
        m.compute_maps_slab(ys[r], ys[r + 1], 1)
    torch.cuda.synchronize()
    for r in range(P):
        m = ranks[r][0]
        lut, data, _ = m.export_frame(0)
        v0, v1 = ys[r] * row, ys[r + 1] * row
        # global ranks: the slab's LUT rows and its data rows [base, base + k)
        assert np.array_equal(lut[v0:v1], ref_lut[v0:v1]), f"rank {r} LUT"
        for k_ in ("hits", "misses", "min_dz", "m1", "m2"):
            assert np.array_equal(data[k_][bases[r]:bases[r + 1]],
                                  ref_data[k_][bases[r]:bases[r + 1]]), (r, k_)
        lay = layers_np(m)
        sl = slice(ys[r], ys[r + 1])
        for k_ in ("height", "density", "hard", "soft"):
            a, b = lay[k_][sl], ref_layers[k_][sl]
            assert np.array_equal(np.nan_to_num(a, nan=-7), np.nan_to_num(b, nan=-7)), (r, k_)
        for k_ in ("slope", "roughness", "neg"):  # phase 1 is slab-local
            a, b = lay[k_][sl], ref_layers[k_][sl]
            assert np.array_equal(np.nan_to_num(a, nan=-7), np.nan_to_num(b, nan=-7)), (r, k_)


@pytest.mark.parametrize("P", [2, 4])
def test_slab_partition_c4_matches_single_gpu(P):
    _run(synth.workload(3), P)


@pytest.mark.parametrize("P", [2, 4])
def test_slab_finalize_peers_fused_reduction(P):
    # NEXT-2 fused collective: gvom_slab_finalize_peers reads the P partial
    # grids (here P buffers on one GPU standing in for peer memory) and sums
    # them while encoding the slab -- bit-identical to reduce-scatter + finalize
    _run(synth.workload(3), P, peers=True)


def test_slab_partition_with_variants():
    # the slab path with the 8-cone search and obstacle-free slope windows:
    # phase 1 runs the same surface kernels on the gathered surface
    _run(synth.workload(3), 2, neg_8cone=True, slope_skip_obstacles=True)


def test_slab_partition_c1_eight_ranks():
    _run(synth.workload(0), 8)


@pytest.mark.slow
def test_slab_partition_c5_eight_ranks():
    _run(synth.workload(4), 8)


def _run_sequence(w, P, K, frames):
    """NEXT-2: motion with a K-map buffer.  Every frame: the slab steps on P
    emulated ranks, the frame-map gather (LUT slabs + data rows into every
    rank's newest slot, then gvom_slab_complete), the slab column pass and the
    surface gather; compared with one GPU after every frame."""
    grid = dict(w.grid)
    grid["buffer_frames"] = K
    npts = max(f.n_points for f in frames)
    ref = GvomMap(grid, max_points_per_frame=npts)
    ms = [GvomMap(grid, max_points_per_frame=npts) for _ in range(P)]
    nx, ny, nz = ref.nx, ref.ny, ref.nz
    ys = parallel.slab_rows(ny, P)
    row = nx * nz
    V = nx * ny * nz
    for f in frames:
        scans = [(torch.from_numpy(s.points).cuda(), s.pose, s.rings) for s in f.scans]
        ref.shift(f.vehicle_xyz)
        ref.integrate_scan(scans)
        ref.compute_maps()
        ref_layers = layers_np(ref)
        st = []
        for r, m in enumerate(ms):
            m.shift(f.vehicle_xyz)
            miss = torch.empty(V, dtype=torch.int32, device="cuda")
            rec = torch.empty(npts + 1, dtype=torch.int64, device="cuda")
            mine = [s for i, s in enumerate(scans) if i % P == r]
            st.append((miss, rec, m.partial_scan(mine, miss, rec, ys)))
        total_miss = sum(x[0] for x in st)
        offs = [np.concatenate([[0], np.cumsum(x[2])]) for x in st]
        recvs, ks = [], []
        for r, m in enumerate(ms):
            recv = torch.cat([x[1][int(o[r]):int(o[r + 1])] for x, o in zip(st, offs)]).contiguous()
            ks.append(m.slab_occupancy(ys[r], ys[r + 1], recv, recv.numel()))
            recvs.append(recv)
        bases = np.concatenate([[0], np.cumsum(ks)])
        for r, m in enumerate(ms):
            miss_slab = total_miss[ys[r] * row:ys[r + 1] * row].contiguous()
            m.slab_finalize(ys[r], ys[r + 1], miss_slab, recvs[r], recvs[r].numel(),
                            int(bases[r]))
        torch.cuda.synchronize()
        # emulated gather_frame: every rank's newest slot gets every slab
        bufs = [m.slot_buffers(0) for m in ms]
        for r in range(P):
            for q in range(P):
                if q == r:
                    continue
                bufs[r][0][ys[q] * row:ys[q + 1] * row] = bufs[q][0][ys[q] * row:ys[q + 1] * row]
                bufs[r][1][int(bases[q]):int(bases[q + 1])] = \
                    bufs[q][1][int(bases[q]):int(bases[q + 1])]
        torch.cuda.synchronize()
        for m in ms:
            m.slab_complete(int(bases[-1]))
        ref_lut, ref_data, _ = ref.export_frame(0)
        for r, m in enumerate(ms):
            lut, data, _ = m.export_frame(0)
            assert np.array_equal(lut, ref_lut), f"rank {r} frame LUT"
            for k_ in ("hits", "misses", "min_dz", "m1", "m2"):
                assert np.array_equal(data[k_], ref_data[k_]), (r, k_)
            m.compute_maps_slab(ys[r], ys[r + 1], 0)
        surf = torch.cat([ms[r].surface()[ys[r]:ys[r + 1]] for r in range(P)])
        for r, m in enumerate(ms):
            m.surface().copy_(surf)
            m.compute_maps_slab(ys[r], ys[r + 1], 1)
        torch.cuda.synchronize()
        for r, m in enumerate(ms):
            lay = layers_np(m)
            sl = slice(ys[r], ys[r + 1])
            for k_ in ("height", "density", "hard", "soft"):
                a, b = lay[k_][sl], ref_layers[k_][sl]
                assert np.array_equal(np.nan_to_num(a, nan=-7), np.nan_to_num(b, nan=-7)), (r, k_)
            for k_ in ("slope", "roughness", "neg"):  # phase 1 is slab-local
                a, b = lay[k_][sl], ref_layers[k_][sl]
                assert np.array_equal(np.nan_to_num(a, nan=-7), np.nan_to_num(b, nan=-7)), (r, k_)


@pytest.mark.parametrize("P", [2, 4])
def test_slab_partition_with_motion_k8(P):
    # BASELINE configs[2] (c3, OS1-128, 12 m/s): shift + merge of 8 maps, slabbed
    w = synth.config3(speed=12.0, n_frames=10, columns=512)
    _run_sequence(w, P, 8, w.frames)


def test_slab_partition_with_motion_multi_sensor():
    # c4's three lidars over a moving sequence (sensors dealt round-robin), K = 3
    w = synth.workload(3)
    f0 = w.frames[0]
    frames = []
    for i in range(4):
        dx = 0.7 * i
        scans = [dataclasses.replace(s, pose=_moved(s.pose, dx)) for s in f0.scans]
        x, y, z = f0.vehicle_xyz
        frames.append(dataclasses.replace(f0, vehicle_xyz=(x + dx, y, z), scans=scans))
    _run_sequence(w, 2, 3, frames)


def _moved(pose, dx):
    p = np.array(pose, dtype=np.float64).reshape(3, 4).copy()
    p[0, 3] += dx
    return p


def _run_segments(w, P, ys=None):
    """The ray-segment slab partition (gvom_integrate_slab): every rank sees
    every sensor and traces only the part of each ray inside its rows; its
    buffer map holds the slab with LOCAL ranks (global = the k of the slabs
    before + local).  No exchange of counts at all; the surface rows are
    all-gathered for the plane fits and the cone search as before."""
    grid = dict(w.grid)
    grid["buffer_frames"] = 1
    f = w.frames[0]
    scans = [(torch.from_numpy(s.points).cuda(), s.pose, s.rings) for s in f.scans]
    ref = GvomMap(grid, max_points_per_frame=f.n_points)
    ref.shift(f.vehicle_xyz)
    ref.integrate_scan(scans)
    ref.compute_maps()
    ref_lut, ref_data, _ = ref.export_frame(0)
    ref_layers = layers_np(ref)
    nx, ny, nz = ref.nx, ref.ny, ref.nz
    ys = parallel.slab_rows(ny, P) if ys is None else ys
    row = nx * nz
    ranks = []
    for r in range(P):
        m = GvomMap(grid, max_points_per_frame=f.n_points)
        m.shift(f.vehicle_xyz)
        m.integrate_slab(scans, ys[r], ys[r + 1])
        m.compute_maps_slab(ys[r], ys[r + 1], 0)
        ranks.append(m)
    surf = torch.cat([ranks[r].surface()[ys[r]:ys[r + 1]] for r in range(P)])
    for r in range(P):
        ranks[r].surface().copy_(surf)
        ranks[r].compute_maps_slab(ys[r], ys[r + 1], 1)
    torch.cuda.synchronize()
    base = 0
    for r in range(P):
        m = ranks[r]
        lut, data, _ = m.export_frame(0)
        k = data["hits"].shape[0]
        v0, v1 = ys[r] * row, ys[r + 1] * row
        got = lut[v0:v1].astype(np.int64)
        got[got >= 0] += base  # local -> global ranks
        assert np.array_equal(got, ref_lut[v0:v1].astype(np.int64)), f"rank {r} LUT"
        for k_ in ("hits", "misses", "min_dz", "m1", "m2"):
            assert np.array_equal(data[k_], ref_data[k_][base:base + k]), (r, k_)
        base += k
        lay = layers_np(m)
        sl = slice(ys[r], ys[r + 1])
        for k_ in ("height", "density", "hard", "soft"):
            a, b = lay[k_][sl], ref_layers[k_][sl]
            assert np.array_equal(np.nan_to_num(a, nan=-7), np.nan_to_num(b, nan=-7)), (r, k_)
        for k_ in ("slope", "roughness", "neg"):  # phase 1 is slab-local
            a, b = lay[k_][sl], ref_layers[k_][sl]
            assert np.array_equal(np.nan_to_num(a, nan=-7), np.nan_to_num(b, nan=-7)), (r, k_)
    assert base == ref_data["hits"].shape[0]


@pytest.mark.parametrize("P", [2, 4])
def test_ray_segment_slabs_c4(P):
    _run_segments(synth.workload(3), P)


@pytest.mark.parametrize("P", [8, 16])
def test_ray_segment_slabs_c1(P):
    # c1: 64 x 64 x 16 -- a finalize tile holds 8 rows: P = 16 gives 4-row
    # slabs, so neighbouring slabs share boundary tiles
    _run_segments(synth.workload(0), P)


def test_ray_segment_slabs_c2_and_c3():
    _run_segments(synth.workload(1), 4)
    _run_segments(synth.config3(speed=12.0, n_frames=1), 8)


def _oracle_row_work(w):
    """Per-row pass-throughs + returns of frame 0 from the oracle's dense
    counts (integrate_dense: H and M per voxel)."""
    from oracle import oracle as O
    om = O.OracleMap(w.grid)
    f = w.frames[0]
    om.shift(f.vehicle_xyz)
    H, M, _, _, _, _ = O.integrate_dense(om.dims, [(s.points, s.pose) for s in f.scans],
                                         om.res, om.origin)
    nx, ny, nz = om.dims
    return (H.astype(np.int64) + M).reshape(ny, nx * nz).sum(axis=1)


@pytest.mark.parametrize("cfg", [0, 1, 3])
def test_row_work_matches_oracle(cfg):
    # gvom_row_work (slab balancing) = sum over each row's voxels of the
    # oracle's hits + misses; on a slab handle only its rows are written
    w = synth.workload(cfg)
    want = _oracle_row_work(w)
    grid = dict(w.grid)
    grid["buffer_frames"] = 1
    f = w.frames[0]
    scans = [(torch.from_numpy(s.points).cuda(), s.pose, s.rings) for s in f.scans]
    m = GvomMap(grid, max_points_per_frame=f.n_points)
    m.shift(f.vehicle_xyz)
    m.integrate_scan(scans)
    got = m.row_work()
    torch.cuda.synchronize()
    assert np.array_equal(got.cpu().numpy(), want)
    ny = m.ny
    y0, y1 = ny // 3, ny // 3 + 5
    s = GvomMap(grid, max_points_per_frame=f.n_points)
    s.shift(f.vehicle_xyz)
    s.integrate_slab(scans, y0, y1)
    out = torch.full((ny,), -7, dtype=torch.int64, device="cuda")
    s.row_work(y0, y1, out)
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    assert np.array_equal(o[y0:y1], want[y0:y1]) and (np.delete(o, np.s_[y0:y1]) == -7).all()


@pytest.mark.parametrize("cfg,P", [(3, 4), (1, 8), (0, 5)])
def test_ray_segment_slabs_balanced(cfg, P):
    # uneven slab bounds from the measured row work (SegmentMapper.rebalance):
    # the partition stays exact whatever the bounds (c1 at P = 5: slabs that
    # do not divide the rows, several sharing finalize tiles)
    w = synth.workload(cfg)
    ys = parallel.balanced_slab_rows(_oracle_row_work(w), P)
    assert ys != parallel.slab_rows(w.grid["ny"], P) if w.grid["ny"] % P == 0 else True
    _run_segments(w, P, ys)


@pytest.mark.slow
def test_ray_segment_slabs_c5_eight_ranks():
    _run_segments(synth.workload(4), 8)


def _run_segments_motion(w, P, K, frames, check_every=3):
    """Ray segments with motion (K > 1): each rank's buffer maps hold only its
    slab; a shifted older map's rows of other slabs are read from their
    owner's workspace (gvom_set_peers: here the P handles' workspaces on one
    GPU stand in for peer memory).  Compared with one GPU every few frames."""
    grid = dict(w.grid)
    grid["buffer_frames"] = K
    npts = max(f.n_points for f in frames)
    ref = GvomMap(grid, max_points_per_frame=npts)
    ms = [GvomMap(grid, max_points_per_frame=npts) for _ in range(P)]
    ny = ref.ny
    ys = parallel.slab_rows(ny, P)
    ptrs = [m.workspace.data_ptr() for m in ms]
    for r, m in enumerate(ms):
        m.set_peers(ptrs, ys, r)
    for i, f in enumerate(frames):
        scans = [(torch.from_numpy(s.points).cuda(), s.pose, s.rings) for s in f.scans]
        ref.shift(f.vehicle_xyz)
        ref.integrate_scan(scans)
        for r, m in enumerate(ms):
            m.shift(f.vehicle_xyz)
            m.integrate_slab(scans, ys[r], ys[r + 1])
        if (i + 1) % check_every and i != len(frames) - 1:
            continue
        ref.compute_maps()
        ref_layers = layers_np(ref)
        for r, m in enumerate(ms):
            m.compute_maps_slab(ys[r], ys[r + 1], 0)
        surf = torch.cat([ms[r].surface()[ys[r]:ys[r + 1]] for r in range(P)])
        for r, m in enumerate(ms):
            m.surface().copy_(surf)
            m.compute_maps_slab(ys[r], ys[r + 1], 1)
        torch.cuda.synchronize()
        for r, m in enumerate(ms):
            lay = layers_np(m)
            sl = slice(ys[r], ys[r + 1])
            for k_ in ("height", "density", "hard", "soft", "spread", "slope", "roughness",
                       "neg"):
                a, b = lay[k_][sl], ref_layers[k_][sl]
                assert np.array_equal(np.nan_to_num(a, nan=-7), np.nan_to_num(b, nan=-7)), \
                    (i, r, k_)


@pytest.mark.parametrize("P", [2, 4])
def test_ray_segments_with_motion_k8(P):
    # BASELINE configs[2] (c3, OS1-128, 12 m/s): 8 buffered maps, slabbed, the
    # shifted rows read over "peer" memory
    w = synth.config3(speed=12.0, n_frames=12, columns=512)
    _run_segments_motion(w, P, 8, w.frames)
