"""Python driver of the C oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module.  It drives oracle/gvom_oracle.c (plain,
single-threaded C, see its header) through ctypes and keeps the map buffer of
PAPER.md section III.B in plain numpy arrays.  It shares no code with
paper_2109_13176_b200/ (the CUDA path); the only module both sides' callers
use is paper_2109_13176_b200/synth.py, the seeded input generator, which
holds none of the method's arithmetic.

Semantics mirror the C-ABI calls (include/gvom.h):
  shift -> or_snap_origin (O1)
  integrate -> or_affine + or_integrate + or_frame_map + buffer push (O2-O6)
  compute_maps -> or_combine + or_columns + or_slope_roughness + or_negative
                  (O7-O10), at the origin of the newest buffer map
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# GVOM_ORACLE_SRC: an alternative source file (tests/test_oracle_mutants.py
# builds deliberately misread copies to check that the pins reject them).
_SRC = os.environ.get("GVOM_ORACLE_SRC") or os.path.join(_HERE, "gvom_oracle.c")
_LIB = os.path.join(os.path.dirname(os.path.abspath(_SRC)), "liboracle.so")

CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
          "-Wall", "-Wno-unused-function"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        i32, i64, f64 = C.c_int32, C.c_int64, C.c_double
        _lib.or_thresholds.argtypes = [f64, f64, f64, f64, f64, P]
        _lib.or_snap_origin.argtypes = [i32, i32, i32, f64, f64, P, P]
        _lib.or_affine.argtypes = [P, f64, P, P, P]
        _lib.or_transform_point.argtypes = [P, P, C.c_float, C.c_float, C.c_float, P]
        _lib.or_transform_point.restype = C.c_int
        _lib.or_traverse.argtypes = [i32, i32, i32, P, P, P, i64]
        _lib.or_traverse.restype = i64
        _lib.or_sensor_inside.argtypes = [i32, i32, i32, P]
        _lib.or_sensor_inside.restype = C.c_int
        _lib.or_integrate.argtypes = [i32, i32, i32, P, P, P, i64, P, P, P, P, P, P]
        _lib.or_integrate.restype = C.c_int
        _lib.or_frame_map.argtypes = [i64, P, P, P, P, P, P, P, P, P, P, P]
        _lib.or_frame_map.restype = i64
        _lib.or_combine.argtypes = [i32, i32, i32, i32, P, P, P, P, P, P, P, P, P, P, P, P, P]
        _lib.or_columns.argtypes = [i32, i32, i32, f64, i64, i64, i64, i64, P, P, P,
                                    P, P, P, P, P, P]
        _lib.or_slope_roughness.argtypes = [i32, i32, f64, i32, i32, P, P, P, P, P]
        _lib.or_spread.argtypes = [i32, i32, i32, f64, P, P, P, P]
        _lib.or_negative.argtypes = [i32, i32, i32, i64, P, P, P]
        _lib.or_negative8.argtypes = [i32, i32, i32, i64, P, P, P]
        _lib.or_cone8_of.argtypes = [i64, i64]
        _lib.or_cone8_of.restype = C.c_int
        _lib.or_costmap.argtypes = [i64, P, P, P, P, P, P, P, P, P]
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(C.c_void_p)


# --------------------------------------------------------------------------
# single steps (each wraps one oracle function)
# --------------------------------------------------------------------------
def thresholds(res, min_h, max_h, dens, neg) -> np.ndarray:
    out = np.zeros(4, dtype=np.int64)
    lib().or_thresholds(res, min_h, max_h, dens, neg, _p(out))
    return out


def snap_origin(nx, ny, nz, res, zfrac, p) -> np.ndarray:
    o = np.zeros(3, dtype=np.int64)
    pp = np.asarray(p, dtype=np.float64).copy()
    lib().or_snap_origin(nx, ny, nz, res, zfrac, _p(pp), _p(o))
    return o


def affine(pose: np.ndarray, res: float, o: np.ndarray):
    A = np.zeros(9, dtype=np.float32)
    b = np.zeros(3, dtype=np.float32)
    ps = np.ascontiguousarray(pose, dtype=np.float64).reshape(12)
    oo = np.ascontiguousarray(o, dtype=np.int64)
    lib().or_affine(_p(ps), res, _p(oo), _p(A), _p(b))
    return A, b


def transform_point(A, b, x, y, z):
    g = np.zeros(3, dtype=np.float32)
    ok = lib().or_transform_point(_p(A), _p(b), C.c_float(x), C.c_float(y), C.c_float(z), _p(g))
    return bool(ok), g


def traverse(dims, s, g, cap: int = 1 << 16) -> np.ndarray:
    """Miss voxels of one ray (O5), [count, 3] int32 in walk order."""
    s = np.asarray(s, dtype=np.float32).copy()
    g = np.asarray(g, dtype=np.float32).copy()
    out = np.zeros((cap, 3), dtype=np.int32)
    n = lib().or_traverse(dims[0], dims[1], dims[2], _p(s), _p(g), _p(out), cap)
    assert n <= cap
    return out[:n].copy()


@dataclass
class FrameMap:
    """One buffer map: LUT [V] int32, data SoA of k rows, origin (voxels)."""
    lut: np.ndarray
    hits: np.ndarray
    misses: np.ndarray
    min_dz: np.ndarray
    m1: np.ndarray
    m2: np.ndarray
    origin: np.ndarray
    stats: Dict[str, int] = field(default_factory=dict)

    @property
    def k(self) -> int:
        return int(self.hits.shape[0])


def integrate_dense(dims, scans, res, origin):
    """O2-O5 into dense grids.  scans: [(points float32 [n,4], pose [3,4])]."""
    nx, ny, nz = dims
    V = nx * ny * nz
    hits = np.zeros(V, dtype=np.uint32)
    misses = np.zeros(V, dtype=np.uint32)
    mind = np.full(V, 0xFFFFFFFF, dtype=np.uint32)
    m1 = np.zeros(V, dtype=np.uint64)
    m2 = np.zeros(V, dtype=np.uint64)
    stats = np.zeros(4, dtype=np.int64)
    for pts, pose in scans:
        A, b = affine(pose, res, origin)
        if not lib().or_sensor_inside(nx, ny, nz, _p(b)):
            raise SensorOutside("sensor voxel outside the grid")
    for pts, pose in scans:
        A, b = affine(pose, res, origin)
        pts = np.ascontiguousarray(pts, dtype=np.float32)
        assert pts.ndim == 2 and pts.shape[1] == 4
        rc = lib().or_integrate(nx, ny, nz, _p(A), _p(b), _p(pts), pts.shape[0], _p(hits),
                                _p(misses), _p(mind), _p(m1), _p(m2), _p(stats))
        assert rc == 0
    return hits, misses, mind, m1, m2, stats


def frame_map(hits, misses, mind, m1, m2, origin, stats=None) -> FrameMap:
    """O6: encode dense grids as LUT + data array."""
    V = hits.shape[0]
    lut = np.zeros(V, dtype=np.int32)
    kmax = int(np.count_nonzero(hits))
    dh = np.zeros(kmax, dtype=np.uint32)
    dm = np.zeros(kmax, dtype=np.uint32)
    dn = np.zeros(kmax, dtype=np.uint32)
    d1 = np.zeros(kmax, dtype=np.uint64)
    d2 = np.zeros(kmax, dtype=np.uint64)
    mi32 = np.ascontiguousarray(np.minimum(misses, 0xFFFFFFFF).astype(np.uint32))
    k = lib().or_frame_map(V, _p(np.ascontiguousarray(hits.astype(np.uint32))), _p(mi32),
                           _p(np.ascontiguousarray(mind.astype(np.uint32))),
                           _p(np.ascontiguousarray(m1)), _p(np.ascontiguousarray(m2)), _p(lut),
                           _p(dh), _p(dm), _p(dn), _p(d1), _p(d2))
    assert k == kmax
    st = {}
    if stats is not None:
        st = dict(valid=int(stats[0]), invalid=int(stats[1]), hits=int(stats[2]),
                  miss_increments=int(stats[3]))
    return FrameMap(lut, dh, dm, dn, d1, d2, np.asarray(origin, dtype=np.int64).copy(), st)


class SensorOutside(Exception):
    pass


@dataclass
class Layers:
    height: np.ndarray
    density: np.ndarray
    hard: np.ndarray
    soft: np.ndarray
    neg: np.ndarray
    slope: np.ndarray
    roughness: np.ndarray
    qs: np.ndarray
    defined: np.ndarray
    spread: Optional[np.ndarray] = None


def combine(dims, slots: Sequence[FrameMap], o):
    """O7 -> dense merged (H, Mi, mn, M1, M2), uint64 sums."""
    nx, ny, nz = dims
    V = nx * ny * nz
    K = len(slots)
    H = np.zeros(V, dtype=np.uint64)
    Mi = np.zeros(V, dtype=np.uint64)
    mn = np.zeros(V, dtype=np.uint32)
    M1 = np.zeros(V, dtype=np.uint64)
    M2 = np.zeros(V, dtype=np.uint64)
    keep = []

    def parr(arrs):
        a = (C.c_void_p * K)(*[x.ctypes.data for x in arrs])
        keep.append(a)
        return C.cast(a, C.c_void_p)

    # zero-length data arrays still need a valid pointer
    def nz_(a):
        return a if a.size else np.zeros(1, dtype=a.dtype)

    luts = [s.lut for s in slots]
    dh = [nz_(s.hits) for s in slots]
    dm = [nz_(s.misses) for s in slots]
    dn = [nz_(s.min_dz) for s in slots]
    d1 = [nz_(s.m1) for s in slots]
    d2 = [nz_(s.m2) for s in slots]
    keep.extend([dh, dm, dn, d1, d2])
    origins = np.ascontiguousarray(np.stack([s.origin for s in slots]).astype(np.int64))
    oo = np.asarray(o, dtype=np.int64).copy()
    lib().or_combine(nx, ny, nz, K, parr(luts), parr(dh), parr(dm), parr(dn), parr(d1), parr(d2),
                     _p(origins), _p(oo), _p(H), _p(Mi), _p(mn), _p(M1), _p(M2))
    return H, Mi, mn, M1, M2


def columns(dims, res, o_z, T, H, Mi, mn):
    """O8 -> height, density, hard, soft, qs, defined ([ny, nx])."""
    nx, ny, nz = dims
    n2 = nx * ny
    height = np.zeros(n2, dtype=np.float32)
    density = np.zeros(n2, dtype=np.float32)
    hard = np.zeros(n2, dtype=np.uint8)
    soft = np.zeros(n2, dtype=np.uint8)
    qs = np.zeros(n2, dtype=np.int32)
    defined = np.zeros(n2, dtype=np.uint8)
    lib().or_columns(nx, ny, nz, res, int(o_z), int(T[0]), int(T[1]), int(T[2]), _p(H), _p(Mi),
                     _p(mn), _p(height), _p(density), _p(hard), _p(soft), _p(qs), _p(defined))
    sh = (ny, nx)
    return (height.reshape(sh), density.reshape(sh), hard.reshape(sh), soft.reshape(sh),
            qs.reshape(sh), defined.reshape(sh))


def slope_roughness(qs, defined, res, N, min_pts, exclude=None):
    """O9 on [ny, nx] fixed-point heights (exclude: cells left out, NEXT-3)."""
    ny, nx = qs.shape
    sl = np.zeros(nx * ny, dtype=np.float32)
    ro = np.zeros(nx * ny, dtype=np.float32)
    ex = None if exclude is None else np.ascontiguousarray(exclude, dtype=np.uint8)
    lib().or_slope_roughness(nx, ny, res, N, min_pts, _p(np.ascontiguousarray(qs, dtype=np.int32)),
                             _p(np.ascontiguousarray(defined, dtype=np.uint8)),
                             None if ex is None else _p(ex), _p(sl), _p(ro))
    return sl.reshape(ny, nx), ro.reshape(ny, nx)


def spread(dims, res, H, M1, M2):
    """NEXT-3 point spread of the surface voxel, [ny, nx] f32 m^2."""
    nx, ny, nz = dims
    out = np.zeros(nx * ny, dtype=np.float32)
    lib().or_spread(nx, ny, nz, res, _p(H), _p(M1), _p(M2), _p(out))
    return out.reshape(ny, nx)


def negative(qs, defined, K, T_neg):
    """O10 on [ny, nx] fixed-point heights."""
    ny, nx = qs.shape
    neg = np.zeros(nx * ny, dtype=np.uint8)
    lib().or_negative(nx, ny, K, int(T_neg), _p(np.ascontiguousarray(qs, dtype=np.int32)),
                      _p(np.ascontiguousarray(defined, dtype=np.uint8)), _p(neg))
    return neg.reshape(ny, nx)


def negative8(qs, defined, K, T_neg):
    """O10 with 8 cones of half-angle 22.5 degrees (NEXT-3, reading B8)."""
    ny, nx = qs.shape
    neg = np.zeros(nx * ny, dtype=np.uint8)
    lib().or_negative8(nx, ny, K, int(T_neg), _p(np.ascontiguousarray(qs, dtype=np.int32)),
                       _p(np.ascontiguousarray(defined, dtype=np.uint8)), _p(neg))
    return neg.reshape(ny, nx)


def cone8_of(u: int, v: int) -> int:
    """Index of the 8-cone holding offset (u, v); -1 if none or several."""
    return int(lib().or_cone8_of(int(u), int(v)))


def costmap(L: "Layers", weights) -> np.ndarray:
    """NEXT-4 costmap: weighted per-pixel sum of the layers (reading B5)."""
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float32).reshape(7))
    shp = L.height.shape
    out = np.zeros(shp, dtype=np.float32)
    c = lambda a, dt: np.ascontiguousarray(a, dtype=dt)  # noqa: E731
    lib().or_costmap(out.size, _p(w), _p(c(L.height, np.float32)), _p(c(L.density, np.float32)),
                     _p(c(L.hard, np.uint8)), _p(c(L.soft, np.uint8)), _p(c(L.neg, np.uint8)),
                     _p(c(L.slope, np.float32)), _p(c(L.roughness, np.float32)), _p(out))
    return out


def roll_window(dims, acc, d):
    """NEXT-3 rolling map (reading B9): re-centre the accumulated dense map
    (H, Mi, mn, M1, M2 over the window, L order) on an origin moved by d
    voxels.  World voxel o_new + l was o_old + (l + d): the overlap is kept,
    voxels that left the window are dropped, entering voxels start empty."""
    nx, ny, nz = dims
    out = []
    for a, empty in zip(acc, (0, 0, 0xFFFFFFFF, 0, 0)):
        src = a.reshape(ny, nx, nz)
        dst = np.full_like(src, empty)
        sl_new, sl_old = [], []
        for dd, n in ((int(d[1]), ny), (int(d[0]), nx), (int(d[2]), nz)):
            lo, hi = max(0, -dd), min(n, n - dd)  # new logical range that was inside
            if lo >= hi:
                lo = hi = 0
            sl_new.append(slice(lo, hi))
            sl_old.append(slice(lo + dd, hi + dd))
        dst[tuple(sl_new)] = src[tuple(sl_old)]
        out.append(dst.reshape(-1))
    return tuple(out)


# --------------------------------------------------------------------------
# the whole update, same call sequence as the C-ABI
# --------------------------------------------------------------------------
class OracleMap:
    def __init__(self, grid: dict):
        self.g = dict(grid)
        self.dims = (int(grid["nx"]), int(grid["ny"]), int(grid["nz"]))
        self.res = float(grid["res"])
        self.K = int(grid.get("buffer_frames", 8))
        self.T = thresholds(self.res, grid["min_obstacle_height"], grid["max_obstacle_height"],
                            grid["density_threshold"], grid["neg_obs_threshold"])
        self.origin = snap_origin(*self.dims, self.res, grid.get("z_center_frac", 0.5),
                                  (0.0, 0.0, 0.0))
        self.buffer: List[FrameMap] = []
        self.times: Dict[str, float] = {}
        self.merged = None
        # NEXT-3 rolling map (reading B9): one accumulated window, K = infinity
        self.rolling = bool(grid.get("rolling", False))
        V = self.dims[0] * self.dims[1] * self.dims[2]
        self.roll = (np.zeros(V, np.uint64), np.zeros(V, np.uint64),
                     np.full(V, 0xFFFFFFFF, np.uint32), np.zeros(V, np.uint64),
                     np.zeros(V, np.uint64)) if self.rolling else None

    def _t(self, key, t0):
        self.times[key] = self.times.get(key, 0.0) + (time.perf_counter() - t0)

    def shift(self, vehicle_xyz) -> np.ndarray:
        t0 = time.perf_counter()
        o = snap_origin(*self.dims, self.res, self.g.get("z_center_frac", 0.5), vehicle_xyz)
        d = o - self.origin
        self.origin = o
        if self.rolling and np.any(d != 0):
            self.roll = roll_window(self.dims, self.roll, d)
        self._t("shift", t0)
        return d

    def integrate(self, scans) -> FrameMap:
        """scans: iterable of (points [n,4] f32, pose [3,4] f64) -> pushes one frame."""
        t0 = time.perf_counter()
        h, m, mn, m1, m2, st = integrate_dense(self.dims, list(scans), self.res, self.origin)
        self._t("integrate", t0)
        t0 = time.perf_counter()
        fm = frame_map(h, m, mn, m1, m2, self.origin, st)
        self._t("frame_map", t0)
        self.buffer.append(fm)
        if len(self.buffer) > self.K:
            self.buffer.pop(0)
        if self.rolling:  # B9: the frame's counts join the window map
            H, Mi, MN, M1, M2 = self.roll
            self.roll = (H + h.astype(np.uint64), Mi + m.astype(np.uint64),
                         np.minimum(MN, mn.astype(np.uint32)), M1 + m1, M2 + m2)
            self.roll_frames = getattr(self, "roll_frames", 0) + 1
        return fm

    def compute_maps(self) -> Layers:
        if not self.buffer:
            raise RuntimeError("empty buffer")
        t0 = time.perf_counter()
        if self.rolling:  # B9: the accumulated window at the current origin
            o = self.origin.copy()
            H, Mi, mn, M1, M2 = self.roll
        else:
            o = self.buffer[-1].origin  # the newest buffer map's origin
            H, Mi, mn, M1, M2 = combine(self.dims, self.buffer, o)
        self._t("combine", t0)
        self.merged = (H, Mi, mn, M1, M2, o.copy())
        t0 = time.perf_counter()
        height, dens, hard, soft, qs, dfn = columns(self.dims, self.res, o[2], self.T, H, Mi, mn)
        self._t("columns", t0)
        t0 = time.perf_counter()
        ex = (hard | soft) if self.g.get("slope_skip_obstacles", False) else None
        sl, ro = slope_roughness(qs, dfn, self.res, int(self.g["slope_window"]),
                                 int(self.g["min_plane_points"]), ex)
        self._t("slope_roughness", t0)
        t0 = time.perf_counter()
        negf = negative8 if self.g.get("neg_8cone", False) else negative
        neg = negf(qs, dfn, int(self.g["neg_obs_search_cells"]), self.T[3])
        self._t("negative", t0)
        spr = spread(self.dims, self.res, H, M1, M2)
        return Layers(height, dens, hard, soft, neg, sl, ro, qs, dfn, spr)

    def merged_map(self) -> FrameMap:
        """The combined voxel map encoded as LUT + data (O7 + O6)."""
        H, Mi, mn, M1, M2, o = self.merged
        assert int(H.max(initial=0)) < 2 ** 32 and int(Mi.max(initial=0)) < 2 ** 32
        return frame_map(H.astype(np.uint32), Mi.astype(np.uint32), mn, M1, M2, o)
