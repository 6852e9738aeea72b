"""Independent brute-force references used to pin the oracle (tests only).

segment_voxels(): the set of voxels whose interior the open segment s->g
intersects, by the slab (interval) method evaluated in float64 on the exact
float32 inputs.  This is plain geometry, not a DDA: it never orders crossings
or steps through cells, so it shares no logic with the oracle's O5 walk.
"""
from __future__ import annotations

import numpy as np


def crossing_times(s, g):
    """All axis-plane crossing parameters t in (0,1) of the segment s->g."""
    s = np.asarray(s, dtype=np.float64)
    g = np.asarray(g, dtype=np.float64)
    d = g - s
    out = []
    for a in range(3):
        S, E = np.floor(s[a]), np.floor(g[a])
        if E > S:
            planes = np.arange(S + 1, E + 1)
        elif E < S:
            planes = np.arange(E + 1, S + 1)
        else:
            continue
        for p in planes:
            out.append(((p - s[a]) / d[a], a))
    out.sort()
    return out


def near_tie(s, g, eps=1e-5) -> bool:
    """True if two crossings on different axes are within eps in t."""
    ct = crossing_times(s, g)
    for (t0, a0), (t1, a1) in zip(ct, ct[1:]):
        if a0 != a1 and (t1 - t0) < eps:
            return True
    return False


def segment_voxels(dims, s, g):
    """Voxels (in grid) intersected by the open segment's interior, as a set of tuples."""
    nx, ny, nz = dims
    s = np.asarray(s, dtype=np.float64)
    g = np.asarray(g, dtype=np.float64)
    d = g - s
    lo = np.zeros((nx, ny, nz))
    hi = np.ones((nx, ny, nz))
    idx = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    for a in range(3):
        i = idx[a].astype(np.float64)
        if d[a] != 0:
            t0 = (i - s[a]) / d[a]
            t1 = (i + 1 - s[a]) / d[a]
            lo = np.maximum(lo, np.minimum(t0, t1))
            hi = np.minimum(hi, np.maximum(t0, t1))
        else:
            inside = (i < s[a]) & (s[a] < i + 1)
            hi = np.where(inside, hi, -1.0)
    hit = lo < hi
    return {tuple(int(v) for v in x) for x in np.argwhere(hit)}


def misses_of_ray(dims, s, g):
    """Brute-force miss set of one ray: intersected voxels minus the endpoint voxel."""
    vox = segment_voxels(dims, s, g)
    E = tuple(int(v) for v in np.floor(np.asarray(g, dtype=np.float64)))
    vox.discard(E)
    return vox
