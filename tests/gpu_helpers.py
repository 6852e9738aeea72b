"""Shared helpers of the GPU parity tests: run the CUDA path (through the
C ABI) and the oracle on the same seeded frames and compare element by element.

Bars (BASELINE.json north_star):
- integer outputs bit-exact: LUT, hits, misses, min_dz, m1, m2, hard, soft, neg,
  nodata masks;
- float layers |gpu - oracle| <= 1e-4 + 1e-5 |oracle| with identical NaNs.
"""
from __future__ import annotations

import numpy as np
import torch

from oracle import oracle as O
from paper_2109_13176_b200 import GvomMap

ATOL, RTOL = 1e-4, 1e-5
FIELDS = ("hits", "misses", "min_dz", "m1", "m2")


def to_dev(scan, device="cuda", host=False):
    t = torch.from_numpy(np.ascontiguousarray(scan.points))
    if host:
        return (t.pin_memory(), scan.pose, scan.rings)
    return (t.to(device), scan.pose, scan.rings)


def compare_frame(m: GvomMap, fm: "O.FrameMap", age: int = 0):
    lut, data, origin = m.export_frame(age)
    assert np.array_equal(origin, fm.origin), (origin, fm.origin)
    bad = np.flatnonzero(lut != fm.lut)
    assert bad.size == 0, f"LUT mismatch at {bad.size} voxels, first {bad[:8]} gpu " \
                          f"{lut[bad[:8]]} oracle {fm.lut[bad[:8]]}"
    for f in FIELDS:
        g, r = data[f], getattr(fm, f)
        assert g.shape == r.shape, (f, g.shape, r.shape)
        bad = np.flatnonzero(g != r)
        assert bad.size == 0, f"data.{f} mismatch at {bad.size} rows, first {bad[:8]}"


def compare_layers(got: dict, L: "O.Layers"):
    for k, ref in (("hard", L.hard), ("soft", L.soft), ("neg", L.neg)):
        g = got[k]
        bad = np.argwhere(g != ref)
        assert bad.size == 0, f"{k} mismatch at {len(bad)} cells, first {bad[:5].tolist()}"
    fl = [("height", L.height), ("density", L.density), ("slope", L.slope),
          ("roughness", L.roughness)]
    if L.spread is not None and "spread" in got:
        fl.append(("spread", L.spread))
    for k, ref in fl:
        g = got[k]
        assert np.array_equal(np.isnan(g), np.isnan(ref)), f"{k} nodata mask differs"
        ok = ~np.isnan(ref)
        err = np.abs(g[ok].astype(np.float64) - ref[ok].astype(np.float64))
        tol = ATOL + RTOL * np.abs(ref[ok].astype(np.float64))
        assert np.all(err <= tol), f"{k} max err {err.max()} "
    # height and density are single rounding of exact integers: bit-exact
    for k, ref in (("height", L.height), ("density", L.density)):
        ok = ~np.isnan(ref)
        assert np.array_equal(got[k][ok], ref[ok]), f"{k} not bit-exact"


def compare_merged(m: GvomMap, om: "O.OracleMap"):
    lut, data = m.export_voxels()
    ref = om.merged_map()
    bad = np.flatnonzero(lut != ref.lut)
    assert bad.size == 0, f"merged LUT mismatch at {bad.size} voxels"
    for f in FIELDS:
        assert np.array_equal(data[f], getattr(ref, f)), f"merged {f}"


def compare_window(m: GvomMap, om: "O.OracleMap"):
    """GVOM_FLAG_ROLLING: the window map against the oracle's accumulators."""
    got = m.export_window()
    H, Mi, mn, M1, M2 = om.roll
    for k, ref in (("hits", H), ("misses", Mi), ("min_dz", mn), ("m1", M1), ("m2", M2)):
        bad = np.flatnonzero(got[k] != ref)
        assert bad.size == 0, f"window {k} mismatch at {bad.size} voxels, first {bad[:8]}"


def layers_np(m: GvomMap) -> dict:
    lay = m.export_layers()
    m.synchronize()  # exports are ordered on the map stream (pipelined mode)
    return {k: v.cpu().numpy() for k, v in lay.items()}


def run_sequence(w, frames=None, *, host=False, check_every=1, check_merged=True,
                 rings_override=None, use_step=False):
    """Integrate frames on GPU and oracle; compare after every `check_every`.
    use_step: drive the GPU with gvom_step (one graph launch per frame)."""
    frames = w.frames if frames is None else frames
    npts = max(f.n_points for f in frames)
    m = GvomMap(w.grid, max_points_per_frame=max(npts, 1))
    om = O.OracleMap(w.grid)
    for i, f in enumerate(frames):
        scans = []
        for s in f.scans:
            pts, pose, rings = to_dev(s, host=host)
            if rings_override is not None:
                rings = rings_override
            scans.append((pts, pose, rings))
        d_ref = om.shift(f.vehicle_xyz)
        if use_step:
            d_gpu, lay = m.step(f.vehicle_xyz, scans)
        else:
            d_gpu = m.shift(f.vehicle_xyz)
            m.integrate_scan(scans)
        assert np.array_equal(d_gpu, d_ref)
        fm = om.integrate([(s.points, s.pose) for s in f.scans])
        if (i + 1) % check_every == 0 or i == len(frames) - 1:
            compare_frame(m, fm)
            if not use_step:
                m.compute_maps()
            L = om.compute_maps()
            assert np.array_equal(m.map_origin(), om.merged[5])
            if use_step:
                m.synchronize()
                compare_layers({k: v.cpu().numpy() for k, v in lay.items()}, L)
            compare_layers(layers_np(m), L)
            if w.grid.get("rolling", False):
                compare_window(m, om)
            elif check_merged:
                compare_merged(m, om)
    return m, om
