"""Multi-GPU slab partition of one frame, collectives only.

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


def gather_rows(full: torch.Tensor, y0: int, y1: int, group=None):
    """all-gather equal row slabs of a [ny, ...] tensor in place."""
    mine = full[y0:y1].contiguous().clone()
    dist.all_gather_into_tensor(full.view(-1), mine.view(-1), group=group)


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
