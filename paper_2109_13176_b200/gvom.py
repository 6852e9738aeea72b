"""Thin Python binding of libgvom.so (include/gvom.h) -- argument marshalling only.

Every step of the map update runs in the library's CUDA kernels.  PyTorch is
used for device memory (the caller-owned workspace and output tensors) and
streams.  There is no CPU fallback: if the library or a CUDA device is
missing, construction raises.

    m = GvomMap(grid_dict, max_points_per_frame=N)   # workspace on cuda:0
    m.shift(vehicle_xyz)
    m.integrate_scan([(points_f32_Nx4, pose_3x4, rings), ...])
    m.compute_maps()
    layers = m.export_layers()
"""
from __future__ import annotations

import collections
import ctypes as C
import os
from typing import Dict, Iterable, Optional, Sequence, Tuple

import numpy as np
import torch

from . import build_ext

LAYERS = ("height", "density", "hard", "soft", "neg", "slope", "roughness", "spread")
LAYER_ID = {"height": 0, "density": 1, "hard": 2, "soft": 3, "neg": 4, "slope": 5, "roughness": 6,
            "spread": 7}
LAYER_U8 = {"hard", "soft", "neg"}
STAGES = ("raycast", "rank_count", "rank_scan", "finalize", "endpoint", "columns", "slope",
          "negative", "memset", "h2d", "export", "merge", "integrate", "maps")
STATUS = {0: "ok", -1: "invalid argument", -2: "workspace too small", -3: "CUDA error",
          -4: "sensor outside the map", -5: "empty map buffer", -6: "capacity too small"}


class GvomError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: {STATUS.get(code, code)} ({code})")
        self.code = code


class SensorOutside(GvomError):
    pass


class Config(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("res", C.c_double),
                ("z_center_frac", C.c_double), ("buffer_frames", C.c_int32), ("flags", C.c_int32),
                ("max_points_per_frame", C.c_int64), ("min_obstacle_height", C.c_double),
                ("max_obstacle_height", C.c_double), ("density_threshold", C.c_double),
                ("slope_window", C.c_int32), ("min_plane_points", C.c_int32),
                ("neg_obs_threshold", C.c_double), ("neg_obs_search_cells", C.c_int32),
                ("pad1", C.c_int32)]


class Scan(C.Structure):
    _fields_ = [("xyzw", C.c_void_p), ("n", C.c_int64), ("sensor_to_world", C.c_double * 12),
                ("rings", C.c_int32), ("pad", C.c_int32)]


class Voxel(C.Structure):
    _fields_ = [("hits", C.c_uint32), ("misses", C.c_uint32), ("min_dz", C.c_uint32),
                ("reserved", C.c_uint32), ("m1", C.c_uint64), ("m2", C.c_uint64)]


_lib = None


def lib_path() -> str:
    # GVOM_LIBRARY: an alternative in-tree build (A/B timing of kernel variants)
    return os.environ.get("GVOM_LIBRARY") or build_ext.LIB


def load_library() -> C.CDLL:
    """Load the in-tree libgvom.so (build it with __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not os.path.exists(path):
        raise RuntimeError(f"libgvom.so not built ({path}); run __graft_entry__.build()")
    L = C.CDLL(path)
    P, I32, I64 = C.c_void_p, C.c_int32, C.c_int64
    sig = {
        "gvom_workspace_bytes": ([P], C.c_size_t),
        "gvom_create": ([P, P, C.c_size_t, P, P], I32),
        "gvom_destroy": ([P], I32),
        "gvom_set_stream": ([P, P], I32),
        "gvom_synchronize": ([P], I32),
        "gvom_shift": ([P, P, P], I32),
        "gvom_integrate_scan": ([P, P, I32], I32),
        "gvom_integrate_slab": ([P, P, I32, I32, I32], I32),
        "gvom_set_peers": ([P, P, P, I32, I32], I32),
        "gvom_row_work": ([P, I32, I32, P], I32),
        "gvom_compute_maps": ([P], I32),
        "gvom_export_2d": ([P, I32, P, C.c_size_t], I32),
        "gvom_export_layers": ([P, P, P], I32),
        "gvom_step": ([P, P, P, I32, P, P, P, P, C.c_size_t, P], I32),
        "gvom_export_layers_cost": ([P, P, P, P, P, C.c_size_t], I32),
        "gvom_export_window": ([P, P, P, P, P, P], I32),
        "gvom_graph_stats": ([P, P], I32),
        "gvom_debug_inject_fault": ([P, I32], I32),
        "gvom_map_origin": ([P, P], I32),
        "gvom_export_voxels": ([P, P, P, I64, P], I32),
        "gvom_export_frame": ([P, I32, P, P, I64, P, P], I32),
        "gvom_set_timing": ([P, I32], I32),
        "gvom_stage_times": ([P, P, I32], I32),
        "gvom_launch_count": ([P], I64),
        "gvom_status_string": ([I32], C.c_char_p),
        "gvom_partial_scan": ([P, P, I32, P, P, I64, P, I32, P], I32),
        "gvom_slab_occupancy": ([P, I32, I32, P, I64, P], I32),
        "gvom_slab_finalize": ([P, I32, I32, P, P, I64, I64], I32),
        "gvom_slot_buffers": ([P, I32, P, P, P], I32),
        "gvom_slab_finalize_peers": ([P, I32, I32, P, I32, P, I64, I64], I32),
        "gvom_obstacle_buffers": ([P, P, P], I32),
        "gvom_slab_complete": ([P, I64], I32),
        "gvom_compute_maps_slab": ([P, I32, I32, I32], I32),
        "gvom_surface_buffer": ([P, P], I32),
        "gvom_map_stream": ([P, P], I32),
        "gvom_costmap": ([P, P, P, C.c_size_t], I32),
        "gvom_abi_version": ([], I32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


EXPORTED = ("gvom_workspace_bytes", "gvom_create", "gvom_destroy", "gvom_set_stream",
            "gvom_synchronize", "gvom_shift", "gvom_integrate_scan", "gvom_compute_maps",
            "gvom_export_2d", "gvom_export_layers", "gvom_map_origin", "gvom_export_voxels", "gvom_export_frame",
            "gvom_set_timing", "gvom_stage_times", "gvom_launch_count", "gvom_status_string",
            "gvom_abi_version", "gvom_partial_scan", "gvom_slab_occupancy", "gvom_slab_finalize",
            "gvom_compute_maps_slab", "gvom_surface_buffer", "gvom_map_stream", "gvom_costmap",
            "gvom_step", "gvom_graph_stats", "gvom_export_layers_cost", "gvom_export_window",
            "gvom_slot_buffers", "gvom_slab_complete", "gvom_slab_finalize_peers",
            "gvom_obstacle_buffers", "gvom_debug_inject_fault", "gvom_integrate_slab",
            "gvom_set_peers", "gvom_row_work")


def make_config(grid: dict, max_points_per_frame: int) -> Config:
    c = Config()
    c.nx, c.ny, c.nz = int(grid["nx"]), int(grid["ny"]), int(grid["nz"])
    c.res = float(grid["res"])
    c.z_center_frac = float(grid.get("z_center_frac", 0.5))
    c.buffer_frames = int(grid.get("buffer_frames", 8))
    c.flags = ((1 if grid.get("pipeline", False) else 0)  # GVOM_FLAG_PIPELINE
               | (2 if grid.get("slope_skip_obstacles", False) else 0)  # ..._SLOPE_SKIP_OBSTACLES
               | (4 if grid.get("neg_8cone", False) else 0)  # GVOM_FLAG_NEG_8CONE
               | (8 if grid.get("rolling", False) else 0))  # GVOM_FLAG_ROLLING
    c.max_points_per_frame = int(max_points_per_frame)
    c.min_obstacle_height = float(grid["min_obstacle_height"])
    c.max_obstacle_height = float(grid["max_obstacle_height"])
    c.density_threshold = float(grid["density_threshold"])
    c.slope_window = int(grid["slope_window"])
    c.min_plane_points = int(grid["min_plane_points"])
    c.neg_obs_threshold = float(grid["neg_obs_threshold"])
    c.neg_obs_search_cells = int(grid["neg_obs_search_cells"])
    return c


def workspace_bytes(grid: dict, max_points_per_frame: int) -> int:
    cfg = make_config(grid, max_points_per_frame)
    return int(load_library().gvom_workspace_bytes(C.byref(cfg)))


def _check(rc: int, what: str):
    if rc != 0:
        if rc == -4:
            raise SensorOutside(rc, what)
        raise GvomError(rc, what)


ScanLike = Tuple  # (points [n,4] f32 tensor/ndarray, pose [3,4], rings)


class GvomMap:
    """One robot-centred voxel map + its buffer of per-scan maps (a gvom_handle)."""

    def __init__(self, grid: dict, max_points_per_frame: int, device="cuda",
                 stream: Optional[torch.cuda.Stream] = None,
                 workspace: Optional[torch.Tensor] = None):
        """workspace: a caller-allocated uint8 device tensor of at least
        workspace_bytes() (e.g. in torch symmetric memory, for gvom_set_peers);
        allocated here when None."""
        self.lib = load_library()
        if not torch.cuda.is_available():
            raise RuntimeError("GvomMap needs a CUDA device (no CPU fallback)")
        self.device = torch.device(device)
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.grid = dict(grid)
        self.cfg = make_config(grid, max_points_per_frame)
        self.nx, self.ny, self.nz = self.cfg.nx, self.cfg.ny, self.cfg.nz
        nbytes = int(self.lib.gvom_workspace_bytes(C.byref(self.cfg)))
        if nbytes == 0:
            raise GvomError(-1, "gvom_workspace_bytes (invalid config)")
        with torch.cuda.device(self.device):
            self.stream = stream or torch.cuda.current_stream(self.device)
            if workspace is None:
                workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            if workspace.numel() * workspace.element_size() < nbytes:
                raise GvomError(-2, "workspace smaller than gvom_workspace_bytes")
            self.workspace = workspace
        self.h = C.c_void_p()
        _check(self.lib.gvom_create(C.byref(self.cfg), C.c_void_p(self.workspace.data_ptr()),
                                    nbytes, C.c_void_p(self.stream.cuda_stream),
                                    C.byref(self.h)), "gvom_create")
        self._keep = collections.deque()
        self._dst_cache = {}  # marshalled destination arrays of recently used output sets

    # -- lifecycle -----------------------------------------------------------
    def close(self):
        if self.h:
            self.lib.gvom_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream: torch.cuda.Stream):
        self.stream = stream
        _check(self.lib.gvom_set_stream(self.h, C.c_void_p(stream.cuda_stream)), "set_stream")

    def synchronize(self):
        _check(self.lib.gvom_synchronize(self.h), "gvom_synchronize")
        self._keep.clear()

    def _retain(self, keep):
        """Keep a call's input tensors alive until the handle's stream passes
        the call: an event is recorded after it, and entries whose event has
        completed are dropped on every call (bounded, with no host sync)."""
        # events complete in stream order: drop finished entries from the front
        while self._keep and self._keep[0][0].query():
            self._keep.popleft()
        if keep:
            ev = torch.cuda.Event()
            ev.record(self.stream)
            self._keep.append((ev, keep))

    # -- the five calls ------------------------------------------------------
    def shift(self, vehicle_xyz: Sequence[float]) -> np.ndarray:
        p = (C.c_double * 3)(*[float(v) for v in vehicle_xyz])
        d = (C.c_int64 * 3)()
        _check(self.lib.gvom_shift(self.h, p, d), "gvom_shift")
        return np.array(d[:], dtype=np.int64)

    def _scan_array(self, scans: Iterable[ScanLike]):
        items = list(scans)
        arr = (Scan * max(1, len(items)))()
        keep = []
        for i, it in enumerate(items):
            pts, pose = it[0], it[1]
            rings = int(it[2]) if len(it) > 2 else 0
            if isinstance(pts, np.ndarray):
                pts = torch.from_numpy(np.ascontiguousarray(pts, dtype=np.float32))
            if pts.dtype != torch.float32 or pts.dim() != 2 or pts.shape[1] != 4:
                raise ValueError("points must be float32 [n, 4]")
            pts = pts.contiguous()
            keep.append(pts)
            arr[i].xyzw = pts.data_ptr() if pts.numel() else None
            arr[i].n = pts.shape[0]
            P = np.ascontiguousarray(np.asarray(pose, dtype=np.float64).reshape(12))
            C.memmove(C.addressof(arr[i].sensor_to_world), P.ctypes.data, 96)
            arr[i].rings = rings
        return arr, len(items), keep

    # -- multi-GPU slab partition (include/gvom.h) --------------
    def partial_scan(self, scans, miss: torch.Tensor, records: torch.Tensor, slab_y) -> list:
        """Trace this rank's rays into `miss` (int32 [V], zeroed by the call) and
        write its in-grid returns into `records` (int64 [cap], one 8-byte
        gvom_endpoint each) grouped by destination slab; returns the counts."""
        arr, n, keep = self._scan_array(scans)
        P = len(slab_y) - 1
        ys = (C.c_int32 * (P + 1))(*[int(v) for v in slab_y])
        cnt = (C.c_int64 * P)()
        _check(self.lib.gvom_partial_scan(self.h, arr, n, C.c_void_p(miss.data_ptr()),
                                          C.c_void_p(records.data_ptr()), records.numel(), ys, P,
                                          cnt), "gvom_partial_scan")
        self._retain(keep)
        return [int(c) for c in cnt]

    def slab_occupancy(self, y0: int, y1: int, records: torch.Tensor, n: int) -> int:
        k = C.c_int64()
        _check(self.lib.gvom_slab_occupancy(self.h, y0, y1, C.c_void_p(records.data_ptr()), n,
                                            C.byref(k)), "gvom_slab_occupancy")
        return k.value

    def slab_finalize(self, y0: int, y1: int, miss_slab: torch.Tensor, records: torch.Tensor,
                      n: int, base: int = 0):
        """LUT + data rows of the slab with global ranks (rows [base, base + k))."""
        _check(self.lib.gvom_slab_finalize(self.h, y0, y1, C.c_void_p(miss_slab.data_ptr()),
                                           C.c_void_p(records.data_ptr()), n, int(base)),
               "gvom_slab_finalize")

    def slab_finalize_peers(self, y0: int, y1: int, grid_ptrs, records: torch.Tensor, n: int,
                            base: int = 0):
        """Fused reduce-scatter + finalize: grid_ptrs are the P ranks' partial
        miss grids (device pointers this GPU can load from, e.g. symmetric
        memory buffer_ptrs)."""
        arr = (C.c_void_p * len(grid_ptrs))(*[int(p) for p in grid_ptrs])
        _check(self.lib.gvom_slab_finalize_peers(self.h, y0, y1, arr, len(grid_ptrs),
                                                 C.c_void_p(records.data_ptr()), n, int(base)),
               "gvom_slab_finalize_peers")

    def slot_buffers(self, age: int = 0):
        """(LUT int32 [V], data rows int64 [cap, 4]) of buffer map `age`, as
        torch views of the workspace (no copy; for the slab all-gather)."""
        lp, dp, cap = C.c_void_p(), C.c_void_p(), C.c_int64()
        _check(self.lib.gvom_slot_buffers(self.h, int(age), C.byref(lp), C.byref(dp),
                                          C.byref(cap)), "gvom_slot_buffers")
        V = self.nx * self.ny * self.nz

        class _View:  # __cuda_array_interface__ wrapper of library-owned memory
            def __init__(self, ptr, shape, typestr):
                self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr,
                                                 "data": (ptr, False), "version": 3,
                                                 "strides": None}
        lut = torch.as_tensor(_View(lp.value, (V,), "<i4"), device=self.device)
        data = torch.as_tensor(_View(dp.value, (max(int(cap.value), 1), 4), "<i8"),
                               device=self.device)
        return lut, data

    def slab_complete(self, k_total: int):
        _check(self.lib.gvom_slab_complete(self.h, int(k_total)), "gvom_slab_complete")

    def compute_maps_slab(self, y0: int, y1: int, phase: int):
        _check(self.lib.gvom_compute_maps_slab(self.h, y0, y1, phase), "gvom_compute_maps_slab")

    @property
    def map_stream(self) -> torch.cuda.Stream:
        """Stream that map processing and exports are ordered on."""
        ptr = C.c_void_p()
        _check(self.lib.gvom_map_stream(self.h, C.byref(ptr)), "gvom_map_stream")
        if ptr.value == self.stream.cuda_stream:
            return self.stream
        return torch.cuda.ExternalStream(ptr.value, device=self.device)

    def surface(self) -> torch.Tensor:
        """int32 [ny, nx] view of the library's surface buffer (q_s; INT32_MIN = none)."""
        ptr = C.c_void_p()
        _check(self.lib.gvom_surface_buffer(self.h, C.byref(ptr)), "gvom_surface_buffer")
        off = ptr.value - self.workspace.data_ptr()
        n = self.nx * self.ny * 4
        return self.workspace[off:off + n].view(torch.int32).view(self.ny, self.nx)

    def obstacles(self):
        """(hard, soft): uint8 [ny, nx] views of the library's obstacle layers."""
        hp, sp_ = C.c_void_p(), C.c_void_p()
        _check(self.lib.gvom_obstacle_buffers(self.h, C.byref(hp), C.byref(sp_)),
               "gvom_obstacle_buffers")
        n = self.nx * self.ny
        views = []
        for ptr in (hp, sp_):
            off = ptr.value - self.workspace.data_ptr()
            views.append(self.workspace[off:off + n].view(self.ny, self.nx))
        return tuple(views)

    def integrate_scan(self, scans: Iterable[ScanLike]):
        """scans: (points, pose[3,4], rings).  points: float32 [n,4] torch tensor
        (cuda or pinned/pageable cpu) or numpy array; host points are copied by
        the library inside the call (stream-ordered)."""
        arr, n, keep = self._scan_array(scans)
        rc = self.lib.gvom_integrate_scan(self.h, arr, n)
        _check(rc, "gvom_integrate_scan")
        self._retain(keep)  # input buffers must live until the stream passes

    def integrate_slab(self, scans: Iterable[ScanLike], y0: int, y1: int):
        """Ray-segment slab partition: every sensor of the frame, traced and
        binned only inside map rows [y0, y1) (local data ranks)."""
        arr, n, keep = self._scan_array(scans)
        _check(self.lib.gvom_integrate_slab(self.h, arr, n, int(y0), int(y1)),
               "gvom_integrate_slab")
        self._retain(keep)

    def set_peers(self, workspace_ptrs, slab_y, rank: int):
        """gvom_set_peers: every rank's workspace (device pointers this GPU can
        load from), the slab rows and this rank; [] clears."""
        P = len(workspace_ptrs)
        ws = (C.c_void_p * max(P, 1))(*[int(p) for p in workspace_ptrs])
        ys = (C.c_int32 * (P + 1))(*[int(v) for v in slab_y]) if P else None
        _check(self.lib.gvom_set_peers(self.h, ws if P else None, ys, P, int(rank)),
               "gvom_set_peers")

    def row_work(self, y0: int = 0, y1: Optional[int] = None,
                 out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """gvom_row_work: int64 [ny] on the device, rows [y0, y1) = the
        pass-throughs + returns of each row of the newest buffer map (the
        others untouched; zeros when `out` is None)."""
        y1 = self.ny if y1 is None else y1
        if out is None:
            out = torch.zeros(self.ny, dtype=torch.int64, device=self.device)
            self.stream.wait_stream(torch.cuda.current_stream(self.device))
        assert out.dtype == torch.int64 and out.is_cuda and out.numel() == self.ny
        _check(self.lib.gvom_row_work(self.h, int(y0), int(y1), C.c_void_p(out.data_ptr())),
               "gvom_row_work")
        return out

    def compute_maps(self):
        _check(self.lib.gvom_compute_maps(self.h), "gvom_compute_maps")

    def export_2d(self, layer: str, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        dt = torch.uint8 if layer in LAYER_U8 else torch.float32
        if out is None:
            out = torch.empty((self.ny, self.nx), dtype=dt, device=self.device)
        assert out.dtype == dt and out.is_contiguous()
        _check(self.lib.gvom_export_2d(self.h, LAYER_ID[layer], C.c_void_p(out.data_ptr()),
                                       out.numel() * out.element_size()), f"export_2d({layer})")
        return out

    def _layer_dst(self, out):
        if out is not None:  # a caller's output set seen before: reuse its marshalling
            key = tuple((out[n].data_ptr(), out[n].numel() * out[n].element_size(),
                         out[n].is_contiguous()) for n in LAYERS)
            hit = self._dst_cache.get(key)
            if hit is not None:
                return out, hit[0], hit[1]
        res = {}
        for name in LAYERS:
            t = None if out is None else out[name]
            if t is None:
                dt = torch.uint8 if name in LAYER_U8 else torch.float32
                t = torch.empty((self.ny, self.nx), dtype=dt, device=self.device)
            assert t.is_contiguous()
            res[name] = t
        ptrs = (C.c_void_p * len(LAYERS))(*[res[n].data_ptr() for n in LAYERS])
        sizes = (C.c_size_t * len(LAYERS))(*[res[n].numel() * res[n].element_size()
                                             for n in LAYERS])
        if out is not None:
            if len(self._dst_cache) >= 16:
                self._dst_cache.clear()
            self._dst_cache[key] = (ptrs, sizes)
        return res, ptrs, sizes

    def _cost_dst(self, weights, cost):
        w = (C.c_float * 7)(*[float(v) for v in weights])
        if cost is None:
            cost = torch.empty((self.ny, self.nx), dtype=torch.float32, device=self.device)
        assert cost.is_contiguous() and cost.dtype == torch.float32
        return w, cost

    def export_layers(self, out: Optional[Dict[str, torch.Tensor]] = None,
                      cost_weights=None, cost: Optional[torch.Tensor] = None
                      ) -> Dict[str, torch.Tensor]:
        """All layers with one gvom_export_layers call (one kernel when every
        destination is device memory); with cost_weights also the costmap,
        fused into the same pass (gvom_export_layers_cost), as key "cost"."""
        res, ptrs, sizes = self._layer_dst(out)
        if cost_weights is None:
            _check(self.lib.gvom_export_layers(self.h, ptrs, sizes), "gvom_export_layers")
            return res
        w, cost = self._cost_dst(cost_weights, cost)
        _check(self.lib.gvom_export_layers_cost(self.h, ptrs, sizes, w, C.c_void_p(cost.data_ptr()),
                                                cost.numel() * 4), "gvom_export_layers_cost")
        res["cost"] = cost
        return res

    def step(self, vehicle_xyz: Sequence[float], scans: Iterable[ScanLike],
             out: Optional[Dict[str, torch.Tensor]] = None, export: bool = True,
             cost_weights=None, cost: Optional[torch.Tensor] = None):
        """gvom_step: shift + integrate_scan + compute_maps (+ export of all
        layers into `out`, allocated if None; + the costmap with cost_weights,
        as key "cost") as one CUDA graph launch.  On a pipelined handle,
        pinned host outputs are complete after synchronize().
        Returns (shift delta, layers or None)."""
        p = (C.c_double * 3)(*[float(v) for v in vehicle_xyz])
        dlt = (C.c_int64 * 3)()
        arr, n, keep = self._scan_array(scans)
        res, ptrs, sizes = self._layer_dst(out) if export else (None, None, None)
        w, cp, cb = None, None, 0
        if cost_weights is not None:
            w, cost = self._cost_dst(cost_weights, cost)
            cp, cb = C.c_void_p(cost.data_ptr()), cost.numel() * 4
        _check(self.lib.gvom_step(self.h, p, arr, n, ptrs, sizes, w, cp, cb, dlt), "gvom_step")
        self._retain(keep)
        if cost_weights is not None:
            res = {} if res is None else res
            res["cost"] = cost
        return np.array(dlt[:], dtype=np.int64), res

    def export_window(self) -> Dict[str, np.ndarray]:
        """GVOM_FLAG_ROLLING: the window map, dense in L order (synchronous)."""
        V = self.nx * self.ny * self.nz
        t = {k: torch.empty(V, dtype=torch.int64, device=self.device)
             for k in ("hits", "misses", "m1", "m2")}
        t["min_dz"] = torch.empty(V, dtype=torch.int32, device=self.device)
        _check(self.lib.gvom_export_window(self.h, *[C.c_void_p(t[k].data_ptr()) for k in
                                                      ("hits", "misses", "min_dz", "m1", "m2")]),
               "gvom_export_window")
        self.synchronize()
        out = {k: v.cpu().numpy().view(np.uint64) for k, v in t.items() if k != "min_dz"}
        out["min_dz"] = t["min_dz"].cpu().numpy().view(np.uint32)
        return out

    def graph_stats(self) -> dict:
        o = (C.c_int64 * 3)()
        _check(self.lib.gvom_graph_stats(self.h, o), "gvom_graph_stats")
        return {"graph_launches": o[0], "instantiations": o[1], "eager_steps": o[2]}

    def inject_fault(self, what: int = 1):
        """Test hook: 1 = the next gvom_step capture fails (GVOM_FAULT_CAPTURE)."""
        _check(self.lib.gvom_debug_inject_fault(self.h, int(what)), "gvom_debug_inject_fault")

    def costmap(self, weights, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Weighted per-pixel sum of the layers; weights = (hard, soft,
        density, negative, slope, roughness, unknown)."""
        w = (C.c_float * 7)(*[float(v) for v in weights])
        if out is None:
            out = torch.empty((self.ny, self.nx), dtype=torch.float32, device=self.device)
        _check(self.lib.gvom_costmap(self.h, w, C.c_void_p(out.data_ptr()),
                                     out.numel() * out.element_size()), "gvom_costmap")
        return out

    def map_origin(self) -> np.ndarray:
        o = (C.c_int64 * 3)()
        _check(self.lib.gvom_map_origin(self.h, o), "gvom_map_origin")
        return np.array(o[:], dtype=np.int64)

    # -- voxel-map export (synchronous) --------------------------------------
    def _alloc_voxels(self, cap: int):
        V = self.nx * self.ny * self.nz
        lut = torch.empty(V, dtype=torch.int32, device=self.device)
        data = torch.empty((max(cap, 1), 8), dtype=torch.int32, device=self.device)  # 32 B rows
        return lut, data

    @staticmethod
    def _split(data: torch.Tensor, k: int) -> Dict[str, np.ndarray]:
        a = data[:k].cpu().numpy().view(np.uint32)
        return dict(hits=a[:, 0].copy(), misses=a[:, 1].copy(), min_dz=a[:, 2].copy(),
                    m1=a[:, 4:6].copy().view(np.uint64)[:, 0],
                    m2=a[:, 6:8].copy().view(np.uint64)[:, 0])

    def export_voxels(self) -> Tuple[np.ndarray, Dict[str, np.ndarray]]:
        """Combined voxel map of the last compute_maps: (LUT [V] int32, data SoA)."""
        cap = int(self.cfg.max_points_per_frame) * int(self.cfg.buffer_frames)
        cap = min(cap, self.nx * self.ny * self.nz)
        lut, data = self._alloc_voxels(cap)
        k = C.c_int64()
        _check(self.lib.gvom_export_voxels(self.h, C.c_void_p(lut.data_ptr()),
                                           C.c_void_p(data.data_ptr()), cap, C.byref(k)),
               "gvom_export_voxels")
        return lut.cpu().numpy(), self._split(data, k.value)

    def export_frame(self, age: int = 0):
        """Buffer map by age (0 = newest): (LUT, data SoA, origin)."""
        cap = min(int(self.cfg.max_points_per_frame), self.nx * self.ny * self.nz)
        lut, data = self._alloc_voxels(cap)
        k = C.c_int64()
        o = (C.c_int64 * 3)()
        _check(self.lib.gvom_export_frame(self.h, age, C.c_void_p(lut.data_ptr()),
                                          C.c_void_p(data.data_ptr()), cap, C.byref(k), o),
               "gvom_export_frame")
        return lut.cpu().numpy(), self._split(data, k.value), np.array(o[:], dtype=np.int64)

    # -- instrumentation -----------------------------------------------------
    def set_timing(self, enable: bool = True, stages: Optional[Iterable[str]] = None):
        """Bracket kernel launches with CUDA events: all stages, or only `stages`."""
        mask = 0
        if enable:
            mask = -1 if stages is None else sum(1 << STAGES.index(s) for s in stages)
        _check(self.lib.gvom_set_timing(self.h, mask), "gvom_set_timing")

    def stage_times(self) -> Dict[str, Tuple[float, int]]:
        buf = (C.c_double * (2 * len(STAGES)))()
        _check(self.lib.gvom_stage_times(self.h, buf, len(buf)), "gvom_stage_times")
        return {s: (buf[2 * i], int(buf[2 * i + 1])) for i, s in enumerate(STAGES)}

    def launch_count(self) -> int:
        return int(self.lib.gvom_launch_count(self.h))
