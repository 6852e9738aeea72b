"""Multi-rank (world size 2, gloo, CPU) test of the slab partition's exchange
(paper_2109_13176_b200/parallel.py).

Each rank owns one sensor of a two-lidar frame.  The compute steps are played
by the oracle (dense miss grid and (L, dz) return records of its own sensor);
the exchange is the product's code: reduce-scatter of the miss grids by
y-slab, all-to-all routing of the records to the slab owner, all-gather of the
slab occupancy counts into global rank offsets, all-gather of surface rows.
Each rank then encodes its slab and checks it against the single-process
oracle frame of both sensors: LUT (ranks shifted by the slab's base), data
rows and surface rows must be identical -- the partition algebra is exact.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _frame():
    from paper_2109_13176_b200 import synth
    w = synth.config1(noise=True)
    lid = synth.Lidar(16, 400, (-40.0, 15.0))
    pose_b = synth.pose_matrix(synth.rot_zyx(0.7), (1.5, -1.0, 0.8))
    pts_b = synth.cast_scan(w.world, lid, pose_b, seed=5, frame=0, sensor=1, device="cpu")
    s_a = w.frames[0].scans[0]
    return w.grid, [(s_a.points, s_a.pose), (pts_b, pose_b)]


def _records(om_dims, res, origin, pts, pose):
    """(L, dz) of the in-grid returns, computed with the oracle's O3/O4 steps."""
    from oracle import oracle as O
    nx, ny, nz = om_dims
    A, b = O.affine(pose, res, origin)
    recs = []
    for p in pts:
        ok, g = O.transform_point(A, b, *p[:3])
        if not ok:
            continue
        v = np.floor(g.astype(np.float64)).astype(np.int64)
        if np.all(v >= 0) and np.all(v < np.array([nx, ny, nz])):
            qz = int(np.floor(np.float32(g[2]) * np.float32(65536)))
            dz = qz - 65536 * int(v[2])
            L = int(v[2] + nz * (v[0] + nx * v[1]))
            recs.append((L, dz, int(v[1])))
    return recs


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import sys
        sys.path.insert(0, ROOT)
        from oracle import oracle as O
        from paper_2109_13176_b200 import parallel
        dist.init_process_group("gloo", rank=rank, world_size=world)
        grid, scans = _frame()
        dims = (grid["nx"], grid["ny"], grid["nz"])
        nx, ny, nz = dims
        V = nx * ny * nz
        res = grid["res"]
        origin = O.snap_origin(nx, ny, nz, res, 0.5, (0.0, 0.0, 0.0))
        ys = parallel.slab_rows(ny, world)
        y0, y1 = ys[rank], ys[rank + 1]
        # --- this rank's compute (oracle stands in for gvom_partial_scan) ---
        pts, pose = scans[rank]
        h, m, mn, m1, m2, st = O.integrate_dense(dims, [(pts, pose)], res, origin)
        recs = _records(dims, res, origin, pts, pose)
        by_dest = [[(L, dz) for (L, dz, y) in recs if ys[r] <= y < ys[r + 1]] for r in range(world)]
        counts = [len(b) for b in by_dest]
        flat = [L | (dz << 32) for b in by_dest for (L, dz) in b]
        records = torch.tensor(flat + [0], dtype=torch.int64)
        miss = torch.from_numpy(m.astype(np.int32))
        # --- the product's exchange ---
        miss_slab = parallel.exchange_misses(miss)
        recv = parallel.route_records(records, counts)
        # slab owner: occupancy + stats from the routed records (oracle O4/O6)
        L = (recv & 0xFFFFFFFF).numpy().astype(np.int64)
        dz = (recv >> 32).numpy().astype(np.int64)
        v0, v1 = y0 * nx * nz, y1 * nx * nz
        assert np.all((L >= v0) & (L < v1))
        sl = L - v0
        n = v1 - v0
        hits = np.bincount(sl, minlength=n).astype(np.uint32)
        mind = np.full(n, 0xFFFFFFFF, np.uint32)
        np.minimum.at(mind, sl, dz.astype(np.uint32))
        mm1 = np.zeros(n, np.uint64)
        np.add.at(mm1, sl, dz.astype(np.uint64))
        mm2 = np.zeros(n, np.uint64)
        np.add.at(mm2, sl, (dz * dz).astype(np.uint64))
        fm = O.frame_map(hits, miss_slab.numpy().astype(np.uint32), mind, mm1, mm2, origin)
        base, k_total, ks = parallel.rank_base(fm.k, "cpu")
        # --- reference: both sensors in one oracle frame -----------------
        H, M, MN, M1, M2, _ = O.integrate_dense(dims, scans, res, origin)
        ref = O.frame_map(H, M, MN, M1, M2, origin)
        assert k_total == ref.k
        lut_ref = ref.lut[v0:v1].astype(np.int64)
        lut_got = fm.lut.astype(np.int64)
        lut_got = np.where(lut_got >= 0, lut_got + base, lut_got)
        assert np.array_equal(lut_got, lut_ref)
        for f in ("hits", "misses", "min_dz", "m1", "m2"):
            assert np.array_equal(getattr(fm, f), getattr(ref, f)[base:base + fm.k]), f
        # --- NEXT-2 frame gather (K > 1): every rank ends with the whole map -
        def rows_of(x, lo, n):  # gvom_voxel rows as int64 words [n, 4]
            w = np.zeros((n, 4), np.uint64)
            w[:, 0] = x.hits[lo:lo + n].astype(np.uint64) | (
                x.misses[lo:lo + n].astype(np.uint64) << np.uint64(32))
            w[:, 1] = x.min_dz[lo:lo + n].astype(np.uint64)
            w[:, 2] = x.m1[lo:lo + n]
            w[:, 3] = x.m2[lo:lo + n]
            return w.view(np.int64)
        lut_full = torch.full((V,), -7, dtype=torch.int32)
        lut_full[v0:v1] = torch.from_numpy(np.where(fm.lut >= 0, fm.lut + base, fm.lut)
                                           .astype(np.int32))
        data = torch.full((k_total + 3, 4), -9, dtype=torch.int64)
        data[base:base + fm.k] = torch.from_numpy(rows_of(fm, 0, fm.k))
        bases = [sum(ks[:r]) for r in range(world)]
        parallel.gather_frame(lut_full, data, nx * nz, y0, y1, bases, ks)
        assert np.array_equal(lut_full.numpy(), ref.lut)
        assert np.array_equal(data[:k_total].numpy(), rows_of(ref, 0, ref.k))
        # --- surface rows: columns of the slab, then all-gather ------------
        T = O.thresholds(res, grid["min_obstacle_height"], grid["max_obstacle_height"],
                         grid["density_threshold"], grid["neg_obs_threshold"])
        Hs, Mis, mns, _, _ = O.combine((nx, y1 - y0, nz), [fm], origin)
        _, _, _, _, qs_slab, dfn_slab = O.columns((nx, y1 - y0, nz), res, origin[2], T, Hs, Mis,
                                                  mns)
        qs_full = torch.zeros((ny, nx), dtype=torch.int32)
        qs_full[y0:y1] = torch.from_numpy(np.where(dfn_slab == 1, qs_slab, np.int32(-2 ** 31)))
        parallel.gather_rows(qs_full, y0, y1)
        Hr, Mir, mnr, _, _ = O.combine(dims, [ref], origin)
        _, _, _, _, qs_r, dfn_r = O.columns(dims, res, origin[2], T, Hr, Mir, mnr)
        want = np.where(dfn_r == 1, qs_r, np.int32(-2 ** 31))
        assert np.array_equal(qs_full.numpy(), want)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok", fm.k, base))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, "fail", traceback.format_exc(), None))


def test_slab_exchange_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + (os.getpid() % 200)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, status, info, base in res:
        assert status == "ok", info
    bases = sorted((r[0], r[3]) for r in res)
    assert bases[0][1] == 0


def test_slab_rows():
    from paper_2109_13176_b200 import parallel
    assert parallel.slab_rows(1024, 8) == [0, 128, 256, 384, 512, 640, 768, 896, 1024]
    with pytest.raises(ValueError):
        parallel.slab_rows(100, 8)


def test_balanced_slab_rows():
    from paper_2109_13176_b200 import parallel
    # uniform work: equal slabs
    assert parallel.balanced_slab_rows([5] * 64, 4) == [0, 16, 32, 48, 64]
    # all work in the middle rows: the middle slabs get narrow
    w = np.zeros(64)
    w[24:40] = 100.0
    ys = parallel.balanced_slab_rows(w, 4, row_share=0.0)
    assert ys[0] == 0 and ys[-1] == 64 and 24 <= ys[1] < ys[2] < ys[3] <= 40
    # property on random work: monotone, >= 1 row each, every bound within
    # half a row weight of its target (unless clamped), all ranks agree
    rng = np.random.default_rng(3)
    for trial in range(50):
        ny = int(rng.integers(8, 300))
        P = int(rng.integers(1, min(ny, 16) + 1))
        w = rng.gamma(0.5, 100.0, ny) * (rng.random(ny) < 0.8)
        ys = parallel.balanced_slab_rows(w, P, row_share=0.1)
        assert len(ys) == P + 1 and ys[0] == 0 and ys[-1] == ny
        assert all(b > a for a, b in zip(ys, ys[1:]))
        ww = w + 0.1 * w.sum() / ny if w.sum() > 0 else w + 1.0
        cum = np.concatenate([[0.0], np.cumsum(ww)])
        for k in range(1, P):
            t = cum[-1] * k / P
            y = ys[k]
            clamped = y == ys[k - 1] + 1 or y == ny - (P - k)
            assert clamped or (abs(cum[y] - t) <= ww[y - 1] / 2 + 1e-9 * cum[-1] or
                               abs(cum[y] - t) <= ww[min(y, ny - 1)] / 2 + 1e-9 * cum[-1]), \
                (trial, k, y)
        assert parallel.balanced_slab_rows(w, P, row_share=0.1) == ys
    with pytest.raises(ValueError):
        parallel.balanced_slab_rows([1.0] * 4, 5)


def _worker_segments(rank, world, port, q):
    """The ray-segment partition's exchange: all_gather_scans must hand every
    rank every sensor (bit-identical points, poses, ring counts, rank order),
    and global_rank_base must turn the slabs' occupied counts -- here the
    oracle's, per slab of the two-sensor frame -- into the global ranks of
    the single-process frame map."""
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import sys
        sys.path.insert(0, ROOT)
        from oracle import oracle as O
        from paper_2109_13176_b200 import parallel
        dist.init_process_group("gloo", rank=rank, world_size=world)
        grid, scans = _frame()
        mine = [(torch.from_numpy(scans[rank][0]), scans[rank][1], 16)]
        got = parallel.all_gather_scans(mine)
        assert len(got) == len(scans)
        for (p, pose, rings), (pr, poser) in zip(got, scans):
            assert np.array_equal(p.numpy(), pr) and np.array_equal(pose, poser) and rings == 16
        # with every sensor's (rank, n, pose, rings) known on every rank, only
        # the points move
        meta = [(r, scans[r][0].shape[0], scans[r][1], 16) for r in range(world)]
        got2 = parallel.all_gather_points(mine, meta)
        for (p, pose, rings), (pr, poser) in zip(got2, scans):
            assert np.array_equal(p.numpy(), pr) and np.array_equal(pose, poser) and rings == 16
        # with buffers kept across frames (SegmentMapper): a second frame with
        # other points reuses them and still gathers exactly
        bufs = {}
        parallel.all_gather_points(mine, meta, None, bufs)
        mine2 = [(torch.from_numpy(scans[rank][0] * 2.0), scans[rank][1], 16)]
        got3 = parallel.all_gather_points(mine2, meta, None, bufs)
        assert bufs["cap"] >= max(s[0].shape[0] for s in scans)
        for (p, pose, rings), (pr, poser) in zip(got3, scans):
            assert np.array_equal(p.numpy(), pr * 2.0) and rings == 16
        dims = (grid["nx"], grid["ny"], grid["nz"])
        nx, ny, nz = dims
        res = grid["res"]
        origin = O.snap_origin(nx, ny, nz, res, 0.5, (0.0, 0.0, 0.0))
        H, M, MN, M1, M2, _ = O.integrate_dense(dims, scans, res, origin)
        ref = O.frame_map(H, M, MN, M1, M2, origin)
        ys = parallel.slab_rows(ny, world)
        v0, v1 = ys[rank] * nx * nz, ys[rank + 1] * nx * nz
        k_local = int((H[v0:v1] >= 1).sum())
        base, total = parallel.global_rank_base(torch.tensor(k_local, dtype=torch.int64))
        assert int(total) == ref.k
        occ = ref.lut[v0:v1] >= 0
        if occ.any():  # the slab's first occupied voxel has global rank = base
            assert int(ref.lut[v0:v1][occ][0]) == int(base)
        # balanced slabs (SegmentMapper.rebalance's arithmetic): each rank's
        # rows of the oracle's per-row pass-throughs + returns, all-reduced,
        # give the same uneven bounds on both ranks; the surface rows then
        # travel through the padded all-gather and the global ranks still
        # line up with the single-process frame
        work = (H + M).reshape(ny, nx * nz).sum(axis=1).astype(np.int64)
        mine_w = np.zeros(ny, np.int64)
        mine_w[ys[rank]:ys[rank + 1]] = work[ys[rank]:ys[rank + 1]]
        wt = torch.from_numpy(mine_w)
        dist.all_reduce(wt)
        assert np.array_equal(wt.numpy(), work)
        yb = parallel.balanced_slab_rows(wt.numpy(), world)
        allyb = [None] * world
        dist.all_gather_object(allyb, yb)
        assert all(a == yb for a in allyb) and yb != ys, (yb, ys)
        full = torch.full((ny, 3), -1.0)
        full[yb[rank]:yb[rank + 1]] = torch.arange(yb[rank], yb[rank + 1]).float()[:, None]
        parallel.gather_rows(full, yb[rank], yb[rank + 1], None, yb)
        assert torch.equal(full, torch.arange(ny).float()[:, None].expand(ny, 3))
        v0, v1 = yb[rank] * nx * nz, yb[rank + 1] * nx * nz
        k_b = int((H[v0:v1] >= 1).sum())
        base_b, total_b = parallel.global_rank_base(torch.tensor(k_b, dtype=torch.int64))
        assert int(total_b) == ref.k
        occ = ref.lut[v0:v1] >= 0
        if occ.any():
            assert int(ref.lut[v0:v1][occ][0]) == int(base_b)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok", k_local, int(base)))
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, "fail", traceback.format_exc(), None))


def test_segment_exchange_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29400 + (os.getpid() % 200)
    procs = [ctx.Process(target=_worker_segments, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, status, info, base in res:
        assert status == "ok", info


def _worker_gather3(rank, world, port, q):
    """Three ranks, uneven slab bounds (balanced_slab_rows of a skewed work
    profile): gather_rows must assemble every rank's rows in place on every
    rank, for 1-D and 2-D row payloads, and all ranks must agree on the bounds."""
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import sys
        sys.path.insert(0, ROOT)
        from paper_2109_13176_b200 import parallel
        dist.init_process_group("gloo", rank=rank, world_size=world)
        ny = 37
        work = np.zeros(ny)
        work[10:20] = 50.0  # skewed: most work in a few rows
        mine = np.zeros(ny, np.int64)
        ys0 = [0, 12, 24, ny]  # the frame's (equal-ish) slabs that measured the work
        mine[ys0[rank]:ys0[rank + 1]] = work[ys0[rank]:ys0[rank + 1]]
        t = torch.from_numpy(mine)
        dist.all_reduce(t)
        yb = parallel.balanced_slab_rows(t.numpy(), world)
        allyb = [None] * world
        dist.all_gather_object(allyb, yb)
        assert all(a == yb for a in allyb)
        rows = [yb[r + 1] - yb[r] for r in range(world)]
        assert len(set(rows)) > 1, yb  # uneven
        for shape in ((ny,), (ny, 5)):
            full = torch.full(shape, -1, dtype=torch.int32)
            full[yb[rank]:yb[rank + 1]] = rank * 1000 + torch.arange(yb[rank], yb[rank + 1],
                                                                    dtype=torch.int32).view(
                -1, *([1] * (len(shape) - 1)))
            parallel.gather_rows(full, yb[rank], yb[rank + 1], None, yb)
            for r in range(world):
                want = r * 1000 + torch.arange(yb[r], yb[r + 1], dtype=torch.int32)
                got = full[yb[r]:yb[r + 1]]
                assert torch.equal(got, want.view(-1, *([1] * (len(shape) - 1))).expand_as(got))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok", yb, None))
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, "fail", traceback.format_exc(), None))


def test_uneven_slab_gather_three_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29200 + (os.getpid() % 200)
    procs = [ctx.Process(target=_worker_gather3, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, status, info, _ in res:
        assert status == "ok", info
