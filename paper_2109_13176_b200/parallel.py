"""Multi-GPU slab partition of one frame, collectives only.

Two partitions of the same frame, both exact (identical to one GPU):

* ray segments (SegmentMapper, the default of bench.py): every rank receives
  every sensor's points (all_gather_scans: 16 bytes per point) and
  gvom_integrate_slab traces only the part of each ray inside its own rows --
  no dense count grid leaves a GPU, nothing is reduced; the surface rows are
  all-gathered for the plane fits and the cone search.  A rank's work is the
  steps inside its rows, which crowd around the vehicle, so the slab bounds
  can be rebalanced from a frame's per-row work (SegmentMapper.rebalance:
  gvom_row_work, all_reduce, balanced_slab_rows); uneven slabs gather
  through one padded all-gather.
* reduce-scatter (SlabMapper, the north_star's design): every rank traces its
  own sensors' rays whole into a dense partial miss grid, and the grids are
  combined by slab as below.

One process per GPU (torch.distributed, NCCL over NVLink; gloo on CPU for the
tests).  Rank r of P owns the y-rows [y_r, y_{r+1}) of the map; in L order
(z + nz*(x + nx*y)) that is one contiguous voxel range, so the exchange is:

  miss grids   -> reduce_scatter_tensor(SUM): integer sums, exact  ("hits
                  and misses being added together"); or, fused (NEXT-2), the
                  grids in symmetric memory and the slab finalize summing every
                  rank's grid over peer memory (gvom_slab_finalize_peers)
  returns      -> all_to_all_single of 8-byte (L, dz) records to the slab owner
  slab k       -> all_gather: global rank of a slab's voxel = sum of the k of the
                  slabs before it + its local rank (ranks stay in L order)
  frame map    -> (buffer_frames > 1, motion; NEXT-2) all_gather of the LUT
                  slabs + one broadcast of data rows per rank: every rank holds
                  every buffered frame whole, so shifted maps read any row
  surface rows -> all_gather_into_tensor of q_s rows (slope / cone-search halos)

The compute steps are the C-ABI slab calls (gvom_partial_scan,
gvom_slab_occupancy, gvom_slab_finalize, gvom_compute_maps_slab).  Because
every reduction is an exact integer sum or min, the result is identical to the
single-GPU map; tests/test_multi_rank_cpu.py checks the exchange with gloo and
the oracle, tests/test_gpu_slab.py checks the kernels with P emulated ranks.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist


def slab_rows(ny: int, P: int) -> List[int]:
    """Equal y-slabs (reduce_scatter_tensor needs equal chunks)."""
    if ny % P:
        raise ValueError(f"ny={ny} is not divisible by {P} ranks")
    return [r * (ny // P) for r in range(P + 1)]


def balanced_slab_rows(row_work: Sequence[float], P: int, row_share: float = 0.25) -> List[int]:
    """Slab bounds [y_0 = 0, ..., y_P = ny] that split the rows' work evenly
    (ray-segment partition, gvom_row_work: a rank traces only the steps in its
    rows).  Row weight = its pass-throughs + returns + a per-row constant
    carrying `row_share` of the total (the column / plane-fit / cone passes,
    which cost the same on every row); bound k is the row where the running
    weight is nearest k/P of the total, every slab at least one row.  Pure
    host arithmetic on the same all-reduced vector, so every rank agrees."""
    import numpy as np
    w = np.asarray(row_work, dtype=np.float64)
    ny = int(w.shape[0])
    if P < 1 or P > ny:
        raise ValueError(f"{P} slabs over {ny} rows")
    tot = float(w.sum())
    w = w + (row_share * tot / ny if tot > 0 else 1.0)
    cum = np.concatenate([[0.0], np.cumsum(w)])  # cum[y] = weight of rows [0, y)
    ys = [0]
    for k in range(1, P):
        t = cum[-1] * k / P
        y = int(np.searchsorted(cum, t))  # cum[y - 1] < t <= cum[y]
        if y > 0 and t - cum[y - 1] < cum[y] - t:
            y -= 1
        ys.append(min(max(y, ys[-1] + 1), ny - (P - k)))
    ys.append(ny)
    return ys


def exchange_misses(miss_full: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the ranks' dense miss grids and keep this rank's slab (int32 [V/P])."""
    P = dist.get_world_size(group)
    out = torch.empty(miss_full.numel() // P, dtype=miss_full.dtype, device=miss_full.device)
    dist.reduce_scatter_tensor(out, miss_full, op=dist.ReduceOp.SUM, group=group)
    return out


def route_records(records: torch.Tensor, send_counts: Sequence[int], group=None) -> torch.Tensor:
    """all-to-all of the (L, dz) records (int64 each), grouped by destination."""
    dev = records.device
    sc = torch.tensor(list(send_counts), dtype=torch.int64, device=dev)
    rc = torch.empty_like(sc)
    dist.all_to_all_single(rc, sc, group=group)
    rcl = [int(v) for v in rc.tolist()]
    total = int(sum(send_counts))
    out = torch.empty(max(sum(rcl), 1), dtype=records.dtype, device=dev)
    dist.all_to_all_single(out[:sum(rcl)], records[:total].contiguous(),
                           output_split_sizes=rcl, input_split_sizes=list(send_counts),
                           group=group)
    return out[:sum(rcl)]


def rank_base(k_local: int, device, group=None) -> Tuple[int, int, List[int]]:
    """(global rank of this slab's first occupied voxel, total k, all k)."""
    P = dist.get_world_size(group)
    t = torch.tensor([k_local], dtype=torch.int64, device=device)
    allk = torch.empty(P, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(allk, t, group=group)
    ks = [int(v) for v in allk.tolist()]
    r = dist.get_rank(group)
    return sum(ks[:r]), sum(ks), ks


def gather_frame(lut: torch.Tensor, data: torch.Tensor, rows: int, y0: int, y1: int,
                 bases: Sequence[int], ks: Sequence[int], group=None):
    """NEXT-2 (K > 1, motion): make a slab-finalized frame map whole on every
    rank.  lut: int32 [V] with this rank's slab rows [y0, y1) valid (global
    ranks); data: rows [cap, 4] int64 with this rank's rows at [base, base+k).
    All-gather of the equal LUT slabs, then one broadcast per rank of its
    data rows (their counts differ)."""
    P = dist.get_world_size(group)
    mine = lut[y0 * rows:y1 * rows].clone()
    dist.all_gather_into_tensor(lut[:P * mine.numel()], mine, group=group)
    for r in range(P):
        if ks[r] > 0:
            dist.broadcast(data[bases[r]:bases[r] + ks[r]], src=r, group=group)


def gather_rows(full: torch.Tensor, y0: int, y1: int, group=None,
                ys: Optional[Sequence[int]] = None):
    """all-gather the row slabs of a [ny, ...] tensor in place (equal slabs,
    or the bounds `ys`: uneven slabs go through one padded all-gather)."""
    P = dist.get_world_size(group)
    rows = [ys[r + 1] - ys[r] for r in range(P)] if ys is not None else None
    if rows is None or len(set(rows)) == 1:
        mine = full[y0:y1].contiguous().clone()
        dist.all_gather_into_tensor(full.view(-1), mine.view(-1), group=group)
        return
    cap = max(rows)
    per = full[0].numel()
    mine = torch.zeros((cap, per), dtype=full.dtype, device=full.device)
    mine[:y1 - y0] = full[y0:y1].reshape(y1 - y0, per)
    allr = torch.empty((P * cap, per), dtype=full.dtype, device=full.device)
    dist.all_gather_into_tensor(allr, mine, group=group)
    fv = full.view(full.shape[0], per)
    for r in range(P):
        fv[ys[r]:ys[r + 1]] = allr[r * cap:r * cap + rows[r]]


class SlabMapper:
    """Drives one rank's GvomMap through a distributed frame.  With
    buffer_frames > 1 every finalized frame map is made whole on every rank
    (gather_frame) so that the shift of older maps can read any row."""

    def __init__(self, m, group=None, ep_capacity: Optional[int] = None, fused: bool = False):
        self.m = m
        self.group = group
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.ys = slab_rows(m.ny, self.P)
        self.y0, self.y1 = self.ys[self.rank], self.ys[self.rank + 1]
        V = m.nx * m.ny * m.nz
        dev = m.device
        # fused (NEXT-2): the miss grids live in symmetric memory and the slab
        # finalize reads every rank's grid over peer memory
        # (gvom_slab_finalize_peers) instead of a reduce-scatter
        self.fused = fused
        if fused:
            import torch.distributed._symmetric_memory as symm_mem
            self.miss = symm_mem.empty(V, dtype=torch.int32, device=dev)
            grp = group if group is not None else dist.group.WORLD
            self.symm = symm_mem.rendezvous(self.miss, grp.group_name)
            self.grid_ptrs = list(self.symm.buffer_ptrs)
        else:
            self.miss = torch.empty(V, dtype=torch.int32, device=dev)
        cap = ep_capacity or int(m.cfg.max_points_per_frame)
        self.records = torch.empty(max(cap, 1), dtype=torch.int64, device=dev)
        self.base = 0
        self.k_total = 0

    def integrate(self, scans_local):
        cur = torch.cuda.current_stream(self.m.device)
        if self.fused:  # no rank still reads our grid of the previous frame
            cur.wait_stream(self.m.stream)
            self.symm.barrier()
            self.m.stream.wait_stream(cur)
        counts = self.m.partial_scan(scans_local, self.miss, self.records, self.ys)
        if self.fused:  # every rank's grid of this frame is complete
            cur.wait_stream(self.m.stream)
            self.symm.barrier()
            self.m.stream.wait_stream(cur)
        else:
            miss_slab = exchange_misses(self.miss, self.group)
        recv = route_records(self.records, counts, self.group)
        k = self.m.slab_occupancy(self.y0, self.y1, recv, recv.numel())
        self.base, self.k_total, ks = rank_base(k, self.m.device, self.group)
        if self.fused:
            self.m.slab_finalize_peers(self.y0, self.y1, self.grid_ptrs, recv, recv.numel(),
                                       self.base)
        else:
            self.m.slab_finalize(self.y0, self.y1, miss_slab, recv, recv.numel(), self.base)
        if int(self.m.cfg.buffer_frames) > 1:
            lut, data = self.m.slot_buffers(0)
            bases = [sum(ks[:r]) for r in range(self.P)]
            torch.cuda.current_stream(self.m.device).wait_stream(self.m.stream)
            gather_frame(lut, data, self.m.nx * self.m.nz, self.y0, self.y1, bases, ks,
                         self.group)
            self.m.stream.wait_stream(torch.cuda.current_stream(self.m.device))
            self.m.slab_complete(self.k_total)

    def compute_maps(self):
        self.m.compute_maps_slab(self.y0, self.y1, 0)
        gather_rows(self.m.surface(), self.y0, self.y1, self.group)
        if int(self.m.cfg.flags) & 2:  # GVOM_FLAG_SLOPE_SKIP_OBSTACLES: windows read them
            for t in self.m.obstacles():
                gather_rows(t, self.y0, self.y1, self.group)
        self.m.compute_maps_slab(self.y0, self.y1, 1)


# ---------------------------------------------------------------------------
# ray-segment partition
# ---------------------------------------------------------------------------
def all_gather_scans(scans, group=None):
    """Every rank's sensors -> every rank, in (rank, local order): a list of
    (points [n, 4] f32, pose [3, 4], rings) on this rank's device.  Metadata
    with all_gather_object, the points as one padded all_gather_into_tensor."""
    import numpy as np
    P = dist.get_world_size(group)
    dev = scans[0][0].device if scans else (
        torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() and
        dist.get_backend(group) == "nccl" else torch.device("cpu"))
    meta = [(int(p.shape[0]), np.asarray(pose, np.float64).reshape(3, 4).tolist(), int(rings))
            for (p, pose, rings) in scans]
    metas = [None] * P
    dist.all_gather_object(metas, meta, group=group)
    tot = [sum(n for n, _, _ in m) for m in metas]
    cap = max(max(tot), 1)
    mine = torch.zeros((cap, 4), dtype=torch.float32, device=dev)
    if scans:
        flat = torch.cat([p.to(dev, torch.float32).reshape(-1, 4) for (p, _, _) in scans])
        mine[:flat.shape[0]] = flat
    allp = torch.empty((P * cap, 4), dtype=torch.float32, device=dev)
    dist.all_gather_into_tensor(allp, mine, group=group)
    out = []
    for r in range(P):
        off = r * cap
        for n, pose, rings in metas[r]:
            out.append((allp[off:off + n], np.asarray(pose, np.float64), rings))
            off += n
    return out


def all_gather_points(scans, meta, group=None, bufs: Optional[dict] = None):
    """all_gather_scans when every rank already knows every sensor's (n,
    pose, rings) in rank order (`meta`: odometry and sensor geometry are the
    vehicle's state): only the points move, as one padded all_gather on the
    device -- no host synchronisation.  `bufs` (a dict the caller keeps, e.g.
    SegmentMapper's) holds the send / receive buffers across frames: no
    per-frame allocation (a fresh 2 x 67 MB at c5 cost the first frames
    several ms in the caching allocator)."""
    import numpy as np
    P = dist.get_world_size(group)
    me = dist.get_rank(group)
    per_rank = [[] for _ in range(P)]
    for r, n, pose, rings in meta:
        per_rank[r].append((int(n), pose, int(rings)))
    tot = [sum(n for n, _, _ in m) for m in per_rank]
    cap = max(max(tot), 1)
    dev = scans[0][0].device if scans else torch.device("cuda", torch.cuda.current_device())
    bufs = {} if bufs is None else bufs
    if bufs.get("cap", -1) < cap or bufs["mine"].device != dev:
        bufs.update(cap=cap, mine=torch.empty((cap, 4), dtype=torch.float32, device=dev),
                    allp=torch.empty((P * cap, 4), dtype=torch.float32, device=dev))
    cap = bufs["cap"]
    mine, allp = bufs["mine"], bufs["allp"]
    off = 0
    for (p, _, _) in scans:  # this rank's sensors, packed (the padding is never read)
        q = p.reshape(-1, 4)
        mine[off:off + q.shape[0]].copy_(q)
        off += q.shape[0]
    assert off == tot[me], "local scans disagree with meta"
    dist.all_gather_into_tensor(allp, mine, group=group)
    out = []
    for r in range(P):
        off = r * cap
        for n, pose, rings in per_rank[r]:
            out.append((allp[off:off + n], np.asarray(pose, np.float64), rings))
            off += n
    return out


def global_rank_base(k_local: torch.Tensor, group=None):
    """Local data ranks -> global: (this slab's base, total k) from the slabs'
    occupied counts (device scalar in, device scalars out: no host sync)."""
    P = dist.get_world_size(group)
    allk = torch.empty(P, dtype=k_local.dtype, device=k_local.device)
    dist.all_gather_into_tensor(allk, k_local.reshape(1), group=group)
    r = dist.get_rank(group)
    return allk[:r].sum(), allk.sum()


def segment_map(grid: dict, max_points_per_frame: int, device, stream=None, group=None,
                ys: Optional[Sequence[int]] = None):
    """A GvomMap for the ray-segment partition.  With buffer_frames > 1 its
    workspace lives in torch symmetric memory and the handle gets every rank's
    workspace pointer (gvom_set_peers): a shifted older map's rows of other
    slabs are then read from their owners over NVLink.  Returns (map, mapper)."""
    from .gvom import GvomMap, workspace_bytes
    P = dist.get_world_size(group)
    rank = dist.get_rank(group)
    symm = None
    ws = None
    if int(grid.get("buffer_frames", 8)) > 1 and P > 1:
        import torch.distributed._symmetric_memory as symm_mem
        nbytes = workspace_bytes(grid, max_points_per_frame)
        ws = symm_mem.empty(nbytes, dtype=torch.uint8, device=device)
        grp = group if group is not None else dist.group.WORLD
        symm = symm_mem.rendezvous(ws, grp.group_name)
    m = GvomMap(grid, max_points_per_frame=max_points_per_frame, device=device, stream=stream,
                workspace=ws)
    sm = SegmentMapper(m, group, ys)
    if symm is not None:
        m.set_peers(list(symm.buffer_ptrs), sm.ys, rank)
        sm.symm = symm
    return m, sm


class SegmentMapper:
    """Drives one rank's GvomMap through the ray-segment partition: all
    sensors of the frame are gathered, the rank traces and bins only its rows
    (gvom_integrate_slab), computes the columns of its rows, and the surface
    rows are all-gathered for phase 1 (slope / roughness / cone search).  With
    peers (segment_map, K > 1) device barriers order the owners' integrate
    before the readers' column pass and the readers before the next integrate."""

    def __init__(self, m, group=None, ys: Optional[Sequence[int]] = None):
        self.m = m
        self.group = group
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.symm = None
        self._bufs = {}  # the points all-gather's buffers, kept across frames
        self._set_bounds(list(ys) if ys is not None else slab_rows(m.ny, self.P))

    def _set_bounds(self, ys):
        if (len(ys) != self.P + 1 or ys[0] != 0 or ys[-1] != self.m.ny or
                any(b <= a for a, b in zip(ys, ys[1:]))):
            raise ValueError(f"bad slab bounds {ys}")
        self.ys = ys
        self.y0, self.y1 = ys[self.rank], ys[self.rank + 1]

    def rebalance(self, row_share: float = 0.25) -> List[int]:
        """New slab bounds from the last frame's per-row work (gvom_row_work
        of this rank's rows, all-reduced; balanced_slab_rows); the next
        integrate uses them.  One host synchronisation -- call it between
        frames, not every frame.  Not with peers (buffer_frames > 1): the
        older buffer maps' rows stay with the owners that integrated them."""
        if self.symm is not None:
            raise RuntimeError("slab bounds are fixed once peers are set")
        work = self.m.row_work(self.y0, self.y1)
        cur = torch.cuda.current_stream(self.m.device) if work.is_cuda else None
        if cur is not None:
            cur.wait_stream(self.m.stream)
        dist.all_reduce(work, op=dist.ReduceOp.SUM, group=self.group)
        self._set_bounds(balanced_slab_rows(work.cpu().numpy(), self.P, row_share))
        return self.ys

    def _barrier(self):
        cur = torch.cuda.current_stream(self.m.device)
        cur.wait_stream(self.m.stream)
        self.symm.barrier()
        self.m.stream.wait_stream(cur)

    def integrate(self, scans_local, gathered: bool = False, meta=None):
        """scans_local: this rank's sensors (gathered=True: already all of them).
        meta: [(rank, n, pose, rings)] of every sensor in rank order when known
        on every rank (then only the points move, no host sync)."""
        cur = torch.cuda.current_stream(self.m.device)
        cur.wait_stream(self.m.stream)  # the last integrate has read the gather buffers
        if gathered:
            scans = scans_local
        elif meta is not None:
            scans = all_gather_points(scans_local, meta, self.group, self._bufs)
        else:
            scans = all_gather_scans(scans_local, self.group)
        self.m.stream.wait_stream(cur)  # this frame's points are gathered
        if self.symm is not None:  # no peer still reads the slot this frame overwrites
            self._barrier()
        self.m.integrate_slab(scans, self.y0, self.y1)
        if self.symm is not None:  # this frame's slabs complete before peers read them
            self._barrier()

    def compute_maps(self):
        self.m.compute_maps_slab(self.y0, self.y1, 0)
        cur = torch.cuda.current_stream(self.m.device)
        cur.wait_stream(self.m.stream)
        gather_rows(self.m.surface(), self.y0, self.y1, self.group, self.ys)
        if int(self.m.cfg.flags) & 2:  # GVOM_FLAG_SLOPE_SKIP_OBSTACLES: windows read them
            for t in self.m.obstacles():
                gather_rows(t, self.y0, self.y1, self.group, self.ys)
        self.m.stream.wait_stream(cur)
        self.m.compute_maps_slab(self.y0, self.y1, 1)
