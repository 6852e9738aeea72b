"""Seeded synthetic lidar workloads (harness input generator).

This module is the ONLY code shared by the CUDA path's callers (tests, bench,
smoke) and the oracle's callers.  It holds none of G-VOM's arithmetic: it
simulates a sensor (an analytic off-road world ray-cast by an Ouster-style
lidar) and returns sensor-frame points plus odometry poses, i.e. exactly the
inputs the paper's method consumes ("pointcloud and odometry data", PAPER.md
P:88).  Nothing here bins, ray-traces voxels, merges or reduces.

Recipe:
- Lidar: OS1-style rings with elevations uniformly spaced over the vertical
  FOV (OS1-64 +-16.6 deg, OS1-128 +-22.5 deg), C azimuth columns.  Points are
  emitted column-major, beam-fastest (index = column*rings + ring).
- Gaussian range noise sigma = 0.01 m (or noise-free).
- A backdrop sphere of radius 80 m around the sensor makes every beam return,
  so N = rings*columns exactly.
- Per-beam counter-based RNG keyed by (seed, frame, sensor, ring, column, ...)
  (splitmix64), base seed 13176 + config index.
- World: heightfield (sum of sinusoids, ramps, ditches, pits, steps), solid
  boxes and trunk cylinders, vegetation ellipsoids that terminate a beam with
  probability p per 0.25 m of chord (soft obstacles).

Geometry is evaluated in float64 with torch (CPU by default, multi-threaded);
the returned points are float32 [N, 4] (w = 0), in the sensor frame.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

BACKDROP_RANGE = 80.0
_GOLD = np.uint64(0x9E3779B97F4A7C15)


# ----------------------------------------------------------------------------
# counter-based RNG (splitmix64 finaliser); numpy uint64 wraps by definition
# ----------------------------------------------------------------------------
def _mix(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return z


def hash_u64(*keys) -> np.ndarray:
    """Hash a tuple of integer keys (scalars or broadcastable arrays)."""
    arrs = np.broadcast_arrays(*[np.asarray(k, dtype=np.int64) for k in keys])
    h = np.full(arrs[0].shape, 0x6A09E667F3BCC909, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for a in arrs:
            h = _mix(h ^ (a.astype(np.uint64) * _GOLD + np.uint64(0x632BE59BD9B4E019)))
    return h


def uniform(*keys) -> np.ndarray:
    """U[0,1) double from hashed keys."""
    return (hash_u64(*keys) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def normal(*keys) -> np.ndarray:
    u1 = uniform(*keys, 1)
    u2 = uniform(*keys, 2)
    return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * math.pi * u2)


# ----------------------------------------------------------------------------
# world description
# ----------------------------------------------------------------------------
@dataclass
class World:
    # sinusoids: (amplitude, wavelength, direction rad, phase rad)
    waves: List[Tuple[float, float, float, float]] = field(default_factory=list)
    base_z: float = 0.0
    # plane term  z += gx*x + gy*y
    plane: Tuple[float, float] = (0.0, 0.0)
    # ramps: (x0, y0, dir, width, run, slope_deg, plateau): trapezoid bump
    ramps: List[Tuple[float, float, float, float, float, float, float]] = field(default_factory=list)
    # ditches: (x0, y0, dir, width, length, depth) -- sharp-walled trench
    ditches: List[Tuple[float, float, float, float, float, float]] = field(default_factory=list)
    # pits: axis-aligned (xmin, xmax, ymin, ymax, depth)
    pits: List[Tuple[float, float, float, float, float]] = field(default_factory=list)
    # steps: (nx, ny, c, height): z += height where nx*x+ny*y > c
    steps: List[Tuple[float, float, float, float]] = field(default_factory=list)
    # solid AABBs (xmin, xmax, ymin, ymax, zmin, zmax)
    boxes: List[Tuple[float, float, float, float, float, float]] = field(default_factory=list)
    # solid vertical cylinders (cx, cy, r, zmin, zmax)
    cylinders: List[Tuple[float, float, float, float, float]] = field(default_factory=list)
    # vegetation ellipsoids (cx, cy, cz, rx, ry, rz, p)
    vegetation: List[Tuple[float, float, float, float, float, float, float]] = field(default_factory=list)
    # vegetation AABBs (xmin, xmax, ymin, ymax, zmin, zmax, p)
    veg_boxes: List[Tuple[float, float, float, float, float, float, float]] = field(default_factory=list)

    def height(self, x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
        h = torch.full_like(x, self.base_z)
        if self.plane != (0.0, 0.0):
            h = h + self.plane[0] * x + self.plane[1] * y
        for a, lam, d, ph in self.waves:
            h = h + a * torch.sin((2 * math.pi / lam) * (x * math.cos(d) + y * math.sin(d)) + ph)
        for x0, y0, d, w, run, sdeg, plat in self.ramps:
            u = (x - x0) * math.cos(d) + (y - y0) * math.sin(d)
            v = -(x - x0) * math.sin(d) + (y - y0) * math.cos(d)
            hh = run * math.tan(math.radians(sdeg))
            prof = torch.clamp(torch.minimum(u, 2 * run + plat - u), min=0.0) * math.tan(math.radians(sdeg))
            prof = torch.clamp(prof, max=hh)
            h = h + torch.where(v.abs() < w / 2, prof, torch.zeros_like(prof))
        for x0, y0, d, w, ln, dep in self.ditches:
            u = (x - x0) * math.cos(d) + (y - y0) * math.sin(d)
            v = -(x - x0) * math.sin(d) + (y - y0) * math.cos(d)
            h = h - dep * ((v.abs() < w / 2) & (u.abs() < ln / 2)).to(x.dtype)
        for x0, x1, y0, y1, dep in self.pits:
            h = h - dep * ((x > x0) & (x < x1) & (y > y0) & (y < y1)).to(x.dtype)
        for nx_, ny_, c, hgt in self.steps:
            h = h + hgt * ((nx_ * x + ny_ * y) > c).to(x.dtype)
        return h

    def height_bound(self) -> Tuple[float, float]:
        """Conservative (min, max) of the heightfield."""
        amp = sum(abs(a) for a, *_ in self.waves)
        lo, hi = self.base_z - amp, self.base_z + amp
        if self.plane != (0.0, 0.0):
            lo -= 1e9
            hi += 1e9
        for *_, run, sdeg, plat in self.ramps:
            hi += run * math.tan(math.radians(sdeg))
        for *_, dep in self.ditches:
            lo -= dep
        for *_, dep in self.pits:
            lo -= dep
        for *_, hgt in self.steps:
            if hgt > 0:
                hi += hgt
            else:
                lo += hgt
        return lo, hi


@dataclass
class Lidar:
    rings: int
    columns: int
    vfov_deg: Tuple[float, float]
    noise_sigma: float = 0.01

    def directions(self) -> torch.Tensor:
        """Unit directions in the sensor frame, [columns*rings, 3], beam-fastest."""
        el = torch.linspace(math.radians(self.vfov_deg[0]), math.radians(self.vfov_deg[1]),
                            self.rings, dtype=torch.float64)
        az = torch.arange(self.columns, dtype=torch.float64) * (2 * math.pi / self.columns)
        az_g, el_g = torch.meshgrid(az, el, indexing="ij")  # [C, R]
        d = torch.stack([torch.cos(el_g) * torch.cos(az_g), torch.cos(el_g) * torch.sin(az_g),
                         torch.sin(el_g)], dim=-1)
        return d.reshape(-1, 3)


OS1_64 = (64, (-16.6, 16.6))
OS1_128 = (128, (-22.5, 22.5))


def rot_zyx(yaw: float, pitch: float = 0.0, roll: float = 0.0) -> np.ndarray:
    cy, sy = math.cos(yaw), math.sin(yaw)
    cp, sp = math.cos(pitch), math.sin(pitch)
    cr, sr = math.cos(roll), math.sin(roll)
    rz = np.array([[cy, -sy, 0], [sy, cy, 0], [0, 0, 1]], dtype=np.float64)
    ry = np.array([[cp, 0, sp], [0, 1, 0], [-sp, 0, cp]], dtype=np.float64)
    rx = np.array([[1, 0, 0], [0, cr, -sr], [0, sr, cr]], dtype=np.float64)
    return rz @ ry @ rx


def pose_matrix(R: np.ndarray, t: Sequence[float]) -> np.ndarray:
    """3x4 row-major sensor->world [R | t] (float64)."""
    P = np.zeros((3, 4), dtype=np.float64)
    P[:, :3] = R
    P[:, 3] = np.asarray(t, dtype=np.float64)
    return P


# ----------------------------------------------------------------------------
# ray casting
# ----------------------------------------------------------------------------
def _cast_terrain(world: World, P: torch.Tensor, D: torch.Tensor, tmax: float,
                  dt: float = 0.1, chunk: int = 48) -> torch.Tensor:
    """First t in (0, tmax] with z(t) < h(x(t), y(t)); inf if none."""
    n = D.shape[0]
    dev = D.device
    out = torch.full((n,), math.inf, dtype=torch.float64, device=dev)
    lo_b, hi_b = world.height_bound()
    dz = D[:, 2]
    # skip the part of each ray that is certainly above the terrain bound
    t0 = torch.zeros(n, dtype=torch.float64, device=dev)
    if P[2] > hi_b:
        down = dz < 0
        t0 = torch.where(down, (hi_b - P[2]) / dz, torch.full_like(dz, math.inf))
        t0 = torch.clamp(t0, min=0.0)
    # upward rays above the bound never hit
    alive = t0 < tmax
    idx = torch.nonzero(alive).squeeze(1)
    tcur = t0[idx]
    steps = torch.arange(1, chunk + 1, dtype=torch.float64, device=dev) * dt
    while idx.numel() > 0:
        Dk = D[idx]
        ts = tcur[:, None] + steps[None, :]  # [m, chunk]
        x = P[0] + ts * Dk[:, 0:1]
        y = P[1] + ts * Dk[:, 1:2]
        z = P[2] + ts * Dk[:, 2:3]
        f = z - world.height(x, y)
        neg = f < 0
        anyneg = neg.any(dim=1)
        if anyneg.any():
            first = torch.argmax(neg.to(torch.int8), dim=1)
            sel = torch.nonzero(anyneg).squeeze(1)
            k = first[sel]
            b = ts[sel, k]
            a = b - dt
            Ds, Ps = Dk[sel], P
            for _ in range(40):
                m = 0.5 * (a + b)
                fm = (Ps[2] + m * Ds[:, 2]) - world.height(Ps[0] + m * Ds[:, 0], Ps[1] + m * Ds[:, 1])
                below = fm < 0
                b = torch.where(below, m, b)
                a = torch.where(below, a, m)
            out[idx[sel]] = b
        tcur = tcur + chunk * dt
        zc = P[2] + tcur * Dk[:, 2]
        keep = (~anyneg) & (tcur < tmax) & ~((Dk[:, 2] >= 0) & (zc > hi_b))
        idx = idx[keep]
        tcur = tcur[keep]
    out[out > tmax] = math.inf
    return out


def _az_interval_rays(az_sorted, order, center_az, half):
    """Indices of rays whose world azimuth is within [center-half, center+half]."""
    if half >= math.pi:
        return order
    lo = center_az - half
    hi = center_az + half
    segs = []
    for a, b in ((lo, hi),):
        # wrap into [-pi, pi)
        if a < -math.pi:
            segs.append((a + 2 * math.pi, math.pi))
            segs.append((-math.pi, b))
        elif b >= math.pi:
            segs.append((a, math.pi))
            segs.append((-math.pi, b - 2 * math.pi))
        else:
            segs.append((a, b))
    parts = []
    for a, b in segs:
        ta = torch.tensor([a], dtype=torch.float64, device=az_sorted.device)
        tb = torch.tensor([b], dtype=torch.float64, device=az_sorted.device)
        i0 = int(torch.searchsorted(az_sorted, ta)[0])
        i1 = int(torch.searchsorted(az_sorted, tb, right=True)[0])
        if i1 > i0:
            parts.append(order[i0:i1])
    if not parts:
        return order[:0]
    return torch.cat(parts)


def default_device() -> str:
    """Geometry device of the generator: the GPU when present (harness code;
    results are deterministic per device).  GVOM_SYNTH_DEVICE overrides."""
    import os
    env = os.environ.get("GVOM_SYNTH_DEVICE")
    if env:
        return env
    return "cuda" if torch.cuda.is_available() else "cpu"


def cast_scan(world: World, lidar: Lidar, pose: np.ndarray, *, seed: int, frame: int,
              sensor: int, noise: bool = True, device: Optional[str] = None) -> np.ndarray:
    """Simulate one scan; returns sensor-frame float32 points [N, 4] (w = 0)."""
    dev = torch.device(device or default_device())
    R = torch.from_numpy(np.ascontiguousarray(pose[:, :3])).to(dev)
    P = torch.from_numpy(np.ascontiguousarray(pose[:, 3])).to(dev)
    d_s = lidar.directions().to(dev)  # sensor frame
    D = d_s @ R.T  # world
    n = D.shape[0]
    t_best = torch.full((n,), BACKDROP_RANGE, dtype=torch.float64, device=dev)
    # terrain
    t_best = torch.minimum(t_best, _cast_terrain(world, P, D, BACKDROP_RANGE))
    # azimuth index for culling
    waz = torch.atan2(D[:, 1], D[:, 0])
    az_sorted, order = torch.sort(waz)

    def cull(cx, cy, rad):
        dx, dy = cx - float(P[0]), cy - float(P[1])
        dist = math.hypot(dx, dy)
        if dist - rad > BACKDROP_RANGE:
            return order[:0]
        if dist <= rad * 1.05 + 1e-9:
            return order
        half = math.asin(min(1.0, rad / dist)) * 1.05 + 1e-6
        return _az_interval_rays(az_sorted, order, math.atan2(dy, dx), half)

    # solid boxes (slab method)
    for (x0, x1, y0, y1, z0, z1) in world.boxes:
        cx, cy = 0.5 * (x0 + x1), 0.5 * (y0 + y1)
        ids = cull(cx, cy, 0.5 * math.hypot(x1 - x0, y1 - y0))
        if ids.numel() == 0:
            continue
        Dk = D[ids]
        tmin = torch.zeros(ids.numel(), dtype=torch.float64, device=dev)
        tmax = t_best[ids].clone()
        for ax, (a0, a1) in enumerate(((x0, x1), (y0, y1), (z0, z1))):
            da = Dk[:, ax]
            pa = float(P[ax])
            with np.errstate(divide="ignore"):
                inv = 1.0 / torch.where(da == 0, torch.full_like(da, 1e-300), da)
            ta = (a0 - pa) * inv
            tb = (a1 - pa) * inv
            tmin = torch.maximum(tmin, torch.minimum(ta, tb))
            tmax = torch.minimum(tmax, torch.maximum(ta, tb))
        hit = (tmin <= tmax) & (tmin > 1e-6)
        t_best[ids[hit]] = torch.minimum(t_best[ids[hit]], tmin[hit])
    # solid vertical cylinders
    for (cx, cy, r, z0, z1) in world.cylinders:
        ids = cull(cx, cy, r)
        if ids.numel() == 0:
            continue
        Dk = D[ids]
        ox, oy = float(P[0]) - cx, float(P[1]) - cy
        a = Dk[:, 0] ** 2 + Dk[:, 1] ** 2
        b = 2 * (ox * Dk[:, 0] + oy * Dk[:, 1])
        c = ox * ox + oy * oy - r * r
        disc = b * b - 4 * a * c
        ok = (disc >= 0) & (a > 0)
        sq = torch.sqrt(torch.clamp(disc, min=0))
        t = (-b - sq) / (2 * torch.where(a > 0, a, torch.ones_like(a)))
        z = float(P[2]) + t * Dk[:, 2]
        hit = ok & (t > 1e-6) & (z >= z0) & (z <= z1)
        t_best[ids[hit]] = torch.minimum(t_best[ids[hit]], t[hit])
    # vegetation: stochastic termination per 0.25 m of chord
    veg = [(i, v) for i, v in enumerate(world.vegetation)]
    for vid, (cx, cy, cz, rx, ry, rz, p) in veg:
        ids = cull(cx, cy, max(rx, ry))
        if ids.numel() == 0:
            continue
        Dk = D[ids]
        o = torch.tensor([(float(P[0]) - cx) / rx, (float(P[1]) - cy) / ry, (float(P[2]) - cz) / rz],
                         dtype=torch.float64, device=dev)
        dk = Dk / torch.tensor([rx, ry, rz], dtype=torch.float64, device=dev)
        a = (dk * dk).sum(1)
        b = 2 * (dk * o).sum(1)
        c = float((o * o).sum()) - 1.0
        disc = b * b - 4 * a * c
        ok = disc > 0
        sq = torch.sqrt(torch.clamp(disc, min=0))
        t0 = torch.clamp((-b - sq) / (2 * a), min=0.0)
        t1 = torch.minimum((-b + sq) / (2 * a), t_best[ids])
        ok = ok & (t1 > t0)
        if not bool(ok.any()):
            continue
        ids, t0, t1 = ids[ok], t0[ok], t1[ok]
        _veg_terminate(ids, t0, t1, p, t_best, seed, frame, sensor, vid, lidar.rings)
    for vid2, (x0, x1, y0, y1, z0, z1, p) in enumerate(world.veg_boxes):
        cx, cy = 0.5 * (x0 + x1), 0.5 * (y0 + y1)
        ids = cull(cx, cy, 0.5 * math.hypot(x1 - x0, y1 - y0))
        if ids.numel() == 0:
            continue
        Dk = D[ids]
        tmin = torch.zeros(ids.numel(), dtype=torch.float64, device=dev)
        tmax = t_best[ids].clone()
        for ax, (a0, a1) in enumerate(((x0, x1), (y0, y1), (z0, z1))):
            da = Dk[:, ax]
            pa = float(P[ax])
            inv = 1.0 / torch.where(da == 0, torch.full_like(da, 1e-300), da)
            ta = (a0 - pa) * inv
            tb = (a1 - pa) * inv
            tmin = torch.maximum(tmin, torch.minimum(ta, tb))
            tmax = torch.minimum(tmax, torch.maximum(ta, tb))
        ok = tmax > tmin
        if not bool(ok.any()):
            continue
        _veg_terminate(ids[ok], tmin[ok], tmax[ok], p, t_best, seed, frame, sensor,
                       100000 + vid2, lidar.rings)
    rng = t_best.cpu().numpy().copy()
    if noise and lidar.noise_sigma > 0:
        beam = np.arange(n, dtype=np.int64)
        rng = rng + lidar.noise_sigma * normal(seed, frame, sensor, beam % lidar.rings,
                                               beam // lidar.rings, 7)
    pts = np.zeros((n, 4), dtype=np.float32)
    pts[:, :3] = (d_s.cpu().numpy() * rng[:, None]).astype(np.float32)
    return pts


def _veg_terminate(ids, t0, t1, p, t_best, seed, frame, sensor, vid, rings):
    step = 0.25
    nsteps = torch.ceil((t1 - t0) / step).to(torch.int64)
    maxs = int(nsteps.max())
    idn = ids.cpu().numpy().astype(np.int64)
    ring = idn % rings
    col = idn // rings
    js = np.arange(maxs, dtype=np.int64)
    u = uniform(seed, frame, sensor, ring[:, None], col[:, None], vid, js[None, :], 11)
    u2 = uniform(seed, frame, sensor, ring[:, None], col[:, None], vid, js[None, :], 13)
    valid = js[None, :] < nsteps.cpu().numpy()[:, None]
    term = (u < p) & valid
    anyt = term.any(axis=1)
    if not anyt.any():
        return
    first = np.argmax(term, axis=1)
    rows = np.nonzero(anyt)[0]
    tt = t0.cpu().numpy()[rows] + (first[rows] + u2[rows, first[rows]]) * step
    tt = np.minimum(tt, t1.cpu().numpy()[rows])
    tgt = torch.from_numpy(idn[rows]).to(t_best.device)
    t_best[tgt] = torch.minimum(t_best[tgt], torch.from_numpy(tt).to(t_best.device))


# ----------------------------------------------------------------------------
# workloads (BASELINE.json configs[0..4])
# ----------------------------------------------------------------------------
@dataclass
class Scan:
    points: np.ndarray  # float32 [N, 4] sensor frame
    pose: np.ndarray  # float64 [3, 4] sensor->world
    rings: int


@dataclass
class Frame:
    vehicle_xyz: Tuple[float, float, float]
    scans: List[Scan]

    @property
    def n_points(self) -> int:
        return sum(s.points.shape[0] for s in self.scans)


@dataclass
class Workload:
    name: str
    grid: dict  # gvom config fields (metres / counts)
    frames: List[Frame]
    world: Optional[World] = None

    @property
    def points_per_frame(self) -> int:
        return max(f.n_points for f in self.frames)


def layer_params(res: float) -> dict:
    """Default layer parameters (SPEC S:264 -- not paper values)."""
    return dict(min_obstacle_height=0.3, max_obstacle_height=2.0, density_threshold=0.5,
                slope_window=5, min_plane_points=4, neg_obs_threshold=0.5,
                neg_obs_search_cells=int(math.floor(6.0 / res + 1e-9)))


def grid_cfg(nx, ny, nz, res, buffer_frames=8, **kw) -> dict:
    g = dict(nx=nx, ny=ny, nz=nz, res=res, z_center_frac=0.5, buffer_frames=buffer_frames)
    g.update(layer_params(res))
    g.update(kw)
    return g


def _random_world(seed: int, extent: float, n_trees: int, n_bushes: int, keepout, *,
                  waves=True, bush_p=(0.1, 0.3), canopy_p=0.3) -> World:
    rs = np.random.default_rng(seed)
    w = World()
    if waves:
        for i in range(4):
            w.waves.append((float(rs.uniform(0.2, 1.0)), float(rs.uniform(8.0, 40.0)),
                            float(rs.uniform(0, 2 * math.pi)), float(rs.uniform(0, 2 * math.pi))))

    def place():
        while True:
            x, y = rs.uniform(-extent, extent, size=2)
            if not keepout(x, y):
                return float(x), float(y)

    def ground(x, y):
        return float(w.height(torch.tensor([x], dtype=torch.float64),
                              torch.tensor([y], dtype=torch.float64))[0])

    for _ in range(n_trees):
        x, y = place()
        r = float(rs.uniform(0.1, 0.3))
        g = ground(x, y)
        hgt = float(rs.uniform(4.0, 10.0))
        w.cylinders.append((x, y, r, g - 1.0, g + hgt))
        crx = float(rs.uniform(1.5, 3.0))
        crz = float(rs.uniform(1.0, 2.0))
        w.vegetation.append((x, y, g + hgt - 0.5 * crz, crx, crx, crz, canopy_p))
    for _ in range(n_bushes):
        x, y = place()
        rx = float(rs.uniform(0.25, 1.0))
        ry = float(rs.uniform(0.25, 1.0))
        rz = float(rs.uniform(0.25, 1.0))
        g = ground(x, y)
        w.vegetation.append((x, y, g + 0.8 * rz, rx, ry, rz, float(rs.uniform(*bush_p))))
    return w


def _ground_at(world: World, x: float, y: float) -> float:
    return float(world.height(torch.tensor([x], dtype=torch.float64),
                              torch.tensor([y], dtype=torch.float64))[0])


def config1(seed: int = 13176 + 0, noise: bool = True) -> Workload:
    """Tiny: flat ground + box + pit, one 10k-point scan, 64x64x16 @ 0.25 m, static."""
    w = World()
    w.boxes.append((2.5, 3.5, -0.5, 0.5, 0.0, 1.0))
    w.pits.append((-3.75, -2.25, 1.25, 2.75, 1.0))
    # 16 x 625 = 10,000 points; a wide downward FOV so the box, the pit and the
    # near field are all observed from the 1 m mount
    lid = Lidar(16, 625, (-40.0, 15.0))
    pose = pose_matrix(np.eye(3), (0.0, 0.0, 1.0))
    pts = cast_scan(w, lid, pose, seed=seed, frame=0, sensor=0, noise=noise)
    fr = Frame((0.0, 0.0, 0.0), [Scan(pts, pose, lid.rings)])
    return Workload("c1_tiny_box_pit", grid_cfg(64, 64, 16, 0.25), [fr], w)


def _c2_world(seed):
    return _random_world(seed, 60.0, 150, 300, lambda x, y: x * x + y * y < 9.0)


def config2(seed: int = 13176 + 1, noise: bool = True, n_frames: int = 1) -> Workload:
    """Single OS1-64 scan (131,072 pts), rolling terrain + trees + bushes, 256x256x64 @ 0.25 m."""
    w = _c2_world(seed)
    lid = Lidar(OS1_64[0], 2048, OS1_64[1])
    frames = []
    for f in range(n_frames):
        # static vehicle; later frames are fresh scans (new noise / vegetation draws)
        g = _ground_at(w, 0.0, 0.0)
        pose = pose_matrix(np.eye(3), (0.0, 0.0, g + 1.5))
        pts = cast_scan(w, lid, pose, seed=seed, frame=f, sensor=0, noise=noise)
        frames.append(Frame((0.0, 0.0, g), [Scan(pts, pose, lid.rings)]))
    return Workload("c2_os1_64_rolling_trees", grid_cfg(256, 256, 64, 0.25), frames, w)


def arc_pose(world: World, s: float, radius: float = 50.0, height: float = 1.5):
    """Vehicle pose after arc length s along a circle of curvature 1/radius."""
    psi = s / radius
    x, y = radius * math.sin(psi), radius * (1.0 - math.cos(psi))
    g = _ground_at(world, x, y)
    e = 0.5
    cu, su = math.cos(psi), math.sin(psi)
    gf = _ground_at(world, x + e * cu, y + e * su)
    gb = _ground_at(world, x - e * cu, y - e * su)
    gl = _ground_at(world, x - e * su, y + e * cu)
    gr = _ground_at(world, x + e * su, y - e * cu)
    pitch = -math.atan2(gf - gb, 2 * e)
    roll = math.atan2(gl - gr, 2 * e)
    R = rot_zyx(psi, pitch, roll)
    return (x, y, g), pose_matrix(R, (x, y, g + height))


def config3(speed: float = 4.5, n_frames: int = 100, seed: int = 13176 + 2,
            noise: bool = True, columns: int = 2048) -> Workload:
    """100-scan OS1-128 sequence at 10 Hz along an arc (curvature 1/50) at `speed` m/s."""
    radius = 50.0

    def keep(x, y):
        return abs(math.hypot(x, y - radius) - radius) < 4.0

    w = _random_world(seed, 150.0, 936, 1872, keep)
    lid = Lidar(OS1_128[0], columns, OS1_128[1])
    frames = []
    for f in range(n_frames):
        veh, pose = arc_pose(w, speed * 0.1 * f, radius)
        pts = cast_scan(w, lid, pose, seed=seed, frame=f, sensor=0, noise=noise)
        frames.append(Frame(veh, [Scan(pts, pose, lid.rings)]))
    return Workload(f"c3_os1_128_seq_{speed:g}mps", grid_cfg(256, 256, 64, 0.25), frames, w)


def config4(seed: int = 13176 + 3, noise: bool = True) -> Workload:
    """3 x OS1-64 (393,216 pts/frame), ramps, ditches, dense vegetation, 512x512x64 @ 0.2 m."""
    w = _random_world(seed, 55.0, 100, 700, lambda x, y: x * x + y * y < 9.0, bush_p=(0.1, 0.4))
    rs = np.random.default_rng(seed + 99)
    for _ in range(6):
        w.ramps.append((float(rs.uniform(-40, 40)), float(rs.uniform(-40, 40)),
                        float(rs.uniform(0, 2 * math.pi)), float(rs.uniform(4, 10)),
                        float(rs.uniform(3, 7)), 15.0, float(rs.uniform(2, 6))))
    for _ in range(6):
        x0, y0 = rs.uniform(-45, 45, size=2)
        if x0 * x0 + y0 * y0 < 36:
            x0 += 10.0
        w.ditches.append((float(x0), float(y0), float(rs.uniform(0, math.pi)), 1.5,
                          float(rs.uniform(8, 25)), 1.0))
    g = _ground_at(w, 0.0, 0.0)
    scans = []
    lid = Lidar(OS1_64[0], 2048, OS1_64[1])
    for i, yaw in enumerate((0.0, 2 * math.pi / 3, -2 * math.pi / 3)):
        off = (0.3 * math.cos(yaw), 0.3 * math.sin(yaw))
        pose = pose_matrix(rot_zyx(yaw), (off[0], off[1], g + 1.8))
        pts = cast_scan(w, lid, pose, seed=seed, frame=0, sensor=i, noise=noise)
        scans.append(Scan(pts, pose, lid.rings))
    return Workload("c4_3x_os1_64_ramps_ditches", grid_cfg(512, 512, 64, 0.2),
                    [Frame((0.0, 0.0, g), scans)], w)


def config5(seed: int = 13176 + 4, noise: bool = True, streams: int = 8,
            columns: int = 4096) -> Workload:
    """8 streams x (128 x 4096) = 4,194,304 pts/frame, 1024x1024x128 @ 0.1 m, one frame (K=1)."""
    w = _random_world(seed, 60.0, 150, 500, lambda x, y: x * x + y * y < 9.0)
    g = _ground_at(w, 0.0, 0.0)
    lid = Lidar(OS1_128[0], columns, OS1_128[1])
    scans = []
    for i in range(streams):
        a = 2 * math.pi * i / streams
        pose = pose_matrix(rot_zyx(a + 0.1), (1.0 * math.cos(a), 1.0 * math.sin(a),
                                              g + 1.5 + 0.1 * (i % 3)))
        pts = cast_scan(w, lid, pose, seed=seed, frame=0, sensor=i, noise=noise)
        scans.append(Scan(pts, pose, lid.rings))
    return Workload("c5_8x_os1_128_large_map", grid_cfg(1024, 1024, 128, 0.1, buffer_frames=1),
                    [Frame((0.0, 0.0, g), scans)], w)


def workload(index: int, **kw) -> Workload:
    """BASELINE.json configs[index] (0-based)."""
    return [config1, config2, config3, config4, config5][index](**kw)


# ----------------------------------------------------------------------------
# scenario worlds for the oracle's pins (tests)
# ----------------------------------------------------------------------------
def scenario_scan(world: World, *, rings=32, columns=720, sensor_z=1.5, vfov=(-30.0, 10.0),
                  seed=1, noise=False, sensor_xy=(0.0, 0.0), yaw=0.0) -> Scan:
    lid = Lidar(rings, columns, vfov, noise_sigma=0.01)
    g = _ground_at(world, *sensor_xy)
    pose = pose_matrix(rot_zyx(yaw), (sensor_xy[0], sensor_xy[1], g + sensor_z))
    pts = cast_scan(world, lid, pose, seed=seed, frame=0, sensor=0, noise=noise)
    return Scan(pts, pose, rings)


def random_points(n: int, lo: float, hi: float, seed: int) -> np.ndarray:
    """Uniform float32 points [n, 4] (w = 0) in a cube, counter-based."""
    i = np.arange(n, dtype=np.int64)
    pts = np.zeros((n, 4), dtype=np.float32)
    for a in range(3):
        pts[:, a] = (lo + (hi - lo) * uniform(seed, i, a, 17)).astype(np.float32)
    return pts
