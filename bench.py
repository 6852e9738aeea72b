#!/usr/bin/env python
"""Benchmark of the G-VOM per-scan map update on B200 (driver contract).

One STEP = one full map update through the C ABI, i.e. every SURVEY.md 8(a)
row on one scan: gvom_shift + gvom_integrate_scan (transform, bin, ray cast,
LUT/data, buffer push) + gvom_compute_maps (combine K=8 buffer maps, column
reduce, slope/roughness, negative obstacles) + gvom_export_2d of all 7 layers.

Workload (default): BASELINE.json configs[1] -- an OS1-64-like 131,072-point
scan over rolling terrain with trees and bushes, 256x256x64 voxels at 0.25 m.
Frames cycle over `--frames` independently drawn scans of the same scene.

value  = lidar points integrated per second over whole steps (all ranks),
         inputs resident in HBM, L2 flushed (256 MiB write) between steps,
         device time from CUDA events on the library's stream.
e2e    = same metric through the public API with pinned HOST buffers: H2D of
         every scan and D2H of all layers of every step inside the timed region
         (value: the pipelined handle streaming scans back to back; the
         synchronous step-at-a-time numbers beside it).
roofline = the dominant kernel (ray cast): algorithmic bytes per launch
         (16 N + 8 M + 8 H) / its mean event-timed launch
         duration, against MEASURED_PEAKS.json hbm_gbs.
cpu_baseline = the oracle (oracle/, single-threaded C) on the same workload.

partitioned = (N = 1) the partitioned path of N > 1 on one rank: BASELINE
         configs[4] (8 streams, 4.2M points, 1024x1024x128) through the slab
         calls -- the N = 1 point of the strong-scaling curve.

--impl reference runs the oracle as the reference arm (CPU; rank 0 only).
N > 1 (torchrun): the partitioned path on BASELINE configs[4]:
the sensors of ONE frame sharded over the ranks; by default (--slab-mode
segments) their points are all-gathered and each rank traces the ray segments
inside its own y-slab (gvom_integrate_slab); --slab-mode reduce_scatter /
fused runs the dense miss-grid reduce-scatter (NCCL) / its symmetric-memory
fused finalize.  Strong scaling, time = max over ranks.  --replicas instead
runs independent per-GPU frame streams (weak scaling, no collective).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# stdout carries exactly one JSON line: keep NCCL's banner ("NCCL version ...") off it
os.environ.setdefault("NCCL_DEBUG", "WARN")
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
_JSON_OUT = None


def _stdout_to_stderr():
    """Everything any library writes to stdout (NCCL prints its version banner
    there at communicator creation whatever NCCL_DEBUG_FILE says) goes to
    stderr; the JSON line is written to the real stdout by emit()."""
    global _JSON_OUT
    if _JSON_OUT is None:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(line: dict):
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()

METRIC = "lidar points/s integrated and map updates/s (256×256×64), % HBM roofline"
L2_FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="gvom", choices=["gvom", "reference"])
    ap.add_argument("--config", type=int, default=None,
                    help="BASELINE.json configs index (default: 1 = c2; with N > 1 the "
                         "partitioned path on 4 = c5)")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent per-GPU frame streams instead of the "
                         "partitioned path")
    ap.add_argument("--no-l2-probe", action="store_true",
                    help="skip the L2 reduction-ceiling probe (roofline.l2_red)")
    ap.add_argument("--no-partitioned", action="store_true",
                    help="N = 1: skip the partitioned-path reference line (c5, one rank)")
    ap.add_argument("--frames", type=int, default=4, help="distinct scans cycled")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--neg8cone", action="store_true",
                    help="GVOM_FLAG_NEG_8CONE variant (8-cone negative-obstacle search)")
    ap.add_argument("--no-balance", action="store_true",
                    help="ray segments: keep equal-row slabs (default: bounds rebalanced "
                         "once from the warm-up frame's per-row work, gvom_row_work)")
    ap.add_argument("--slab-mode", default="segments",
                    choices=["segments", "reduce_scatter", "fused"],
                    help="partitioned path: ray segments per slab (default), the dense "
                         "miss-grid reduce-scatter, or its fused symmetric-memory variant "
                         "(gvom_slab_finalize_peers)")
    ap.add_argument("--rolling", action="store_true",
                    help="GVOM_FLAG_ROLLING variant (one accumulated window map, K = inf)")
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of oracle work")
    ap.add_argument("--slab", action="store_true",
                    help="the partitioned path (slab partition of one frame) at any N")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_workload(cfg_index: int, frames: int, rank: int):
    from paper_2109_13176_b200 import synth
    seed = 13176 + cfg_index + 1000 * rank
    if cfg_index == 0:
        return synth.config1(seed=seed)
    if cfg_index == 1:
        return synth.config2(seed=seed, n_frames=frames)
    if cfg_index == 2:
        return synth.config3(speed=12.0, n_frames=max(frames, 8), seed=seed)
    if cfg_index == 3:
        return synth.config4(seed=seed)
    return synth.config5(seed=seed)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def measured_traffic(workload: str):
    """DRAM bytes and warp instructions per k_raycast launch for this workload
    from the committed ncu --set full capture (profiles/raycast_traffic.json)."""
    p = os.path.join(ROOT, "profiles", "raycast_traffic.json")
    try:
        d = json.load(open(p))
        v = d["bytes_per_launch"].get(workload)
        inst = d.get("warp_inst_per_launch", {}).get(workload)
        return ((float(v) if v is not None else None), d["source"].get(workload),
                (float(inst) if inst is not None else None))
    except Exception:
        return None, None, None


def l2_red_ceiling():
    """the L2 reduction ceiling of the ray cast's miss counting --
    red.global.add.u32 into 16 / 64 / 512 MB arrays (tools library
    libgvom_probe.so, csrc/probe/l2_red_probe.cu).  Per size: random words
    (one L2 request per lane), one 128-byte line per warp instruction (32
    atomic ops per request), and runs of 4 lanes (one red per run, the merged
    shape of the ray cast's steps)."""
    import ctypes as C
    from paper_2109_13176_b200 import build_ext
    try:
        lib = C.CDLL(build_ext.PROBE_LIB)
    except OSError as e:
        return {"error": str(e)}
    lib.probe_red.argtypes = [C.c_int64, C.c_int, C.c_int64, C.POINTER(C.c_float),
                              C.POINTER(C.c_int64)]
    lib.probe_red.restype = C.c_int
    out = {}
    n_warp_iters = 1 << 20
    for mb in (16, 64, 512):
        row = {}
        for pat, name, lanes in ((0, "random_word", 32), (1, "line_per_warp", 32),
                                 (2, "runs_of_4", 8)):
            ms = C.c_float(0.0)
            ninst = C.c_int64(0)
            rc = lib.probe_red(mb << 20, pat, n_warp_iters, C.byref(ms), C.byref(ninst))
            if rc < 0 or ms.value <= 0:
                row[name] = None
                continue
            inst = ninst.value
            reqs = inst * (32 if pat == 0 else (1 if pat == 1 else 8))
            row[name] = {"g_red_lanes_s": inst * lanes / (ms.value / 1e3) / 1e9,
                         "g_l2_requests_s": reqs / (ms.value / 1e3) / 1e9,
                         "ms": ms.value}
        out[f"{mb}MB"] = row
    return out


def measured_red_requests(workload: str):
    """L2 reduction requests per k_raycast launch (committed ncu capture)."""
    p = os.path.join(ROOT, "profiles", "raycast_traffic.json")
    try:
        v = json.load(open(p)).get("red_requests_per_launch", {}).get(workload)
        return None if v is None else float(v)
    except Exception:
        return None


# issue peak: 148 SMs x 4 schedulers x one warp instruction per cycle at the
# measured boost clock (B200_PROFILING.md: 1965 MHz under load)
ISSUE_PEAK_GINST_S = 148 * 4 * 1.965


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev = dev
        self.proc = None
        self.f = None

    def __enter__(self):
        try:
            self.f = tempfile.TemporaryFile(mode="w+")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.proc is None or self.f is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.f.seek(0)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


class OneCore:
    """Pin the calling thread to one host core (the oracle is
    timed single-threaded, pinned with sched_setaffinity), restored on exit."""

    def __enter__(self):
        self.prev = None
        self.core = None
        try:
            self.prev = os.sched_getaffinity(0)
            self.core = max(self.prev)  # away from core 0 (interrupts, the driver)
            os.sched_setaffinity(0, {self.core})
        except (AttributeError, OSError):
            pass
        return self

    def __exit__(self, *a):
        if self.prev is not None:
            try:
                os.sched_setaffinity(0, self.prev)
            except OSError:
                pass


def oracle_run(w, budget_s: float, max_frames: int = 1000):
    """The oracle as it stands on this host (single thread pinned to one
    core), bounded by budget."""
    with OneCore() as oc:
        r = _oracle_run(w, budget_s, max_frames)
    r["pinned_core"] = oc.core
    return r


def _oracle_run(w, budget_s: float, max_frames: int = 1000):
    from oracle import oracle as O
    om = O.OracleMap(w.grid)
    t0 = time.perf_counter()
    frames = pts = 0
    while frames < max_frames:
        f = w.frames[frames % len(w.frames)]
        om.shift(f.vehicle_xyz)
        om.integrate([(s.points, s.pose) for s in f.scans])
        om.compute_maps()
        frames += 1
        pts += f.n_points
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    integ = om.times.get("integrate", 0.0) + om.times.get("frame_map", 0.0)
    return dict(value=pts / dt, unit="points/s", cores=1, kind="oracle",
                sample=f"{frames} full map updates ({pts} points) of {w.name}, "
                       f"single-threaded C oracle, {dt:.1f} s",
                updates_per_s=frames / dt, integrate_points_per_s=pts / integ if integ else None,
                host_cpu=_cpu_model(), host_cores=os.cpu_count())


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    if args.config is None:  # the config our arm runs at this N
        args.config = 4 if (world > 1 and not args.replicas) else 1
    w = load_workload(args.config, args.frames, 0)
    budget = float(os.environ.get("GVOM_REF_BUDGET_S", "60"))
    # warmup: one untimed update; then timed updates bounded by the budget
    from oracle import oracle as O
    om = O.OracleMap(w.grid)
    f = w.frames[0]
    om.shift(f.vehicle_xyz)
    om.integrate([(s.points, s.pose) for s in f.scans])
    om.compute_maps()
    r = oracle_run(w, budget, max_frames=max(1, args.steps))
    line = {
        "impl": "reference", "metric": METRIC, "value": r["value"], "unit": "points/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 / r["updates_per_s"], "higher_is_better": True,
        "scaling": "strong" if (world > 1 and not args.replicas) else "weak",
        "vs_baseline": None, "dtype": "f32+int", "data": "synthetic",
        "config": {"workload": w.name, "points_per_scan": w.points_per_frame,
                   "grid": f"{w.grid['nx']}x{w.grid['ny']}x{w.grid['nz']}@{w.grid['res']}m",
                   "buffer_frames": w.grid["buffer_frames"]},
        "map_updates_per_s": r["updates_per_s"],
        "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": r["value"], "unit": "points/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


def ensure_dist(dev):
    """torch.distributed for the slab path; a single process (plain `python
    bench.py`) gets a one-rank group on 127.0.0.1."""
    import torch.distributed as dist
    if dist.is_initialized():
        return
    if "RANK" not in os.environ:
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0",
                          WORLD_SIZE="1", LOCAL_RANK="0")
    dist.init_process_group("nccl", device_id=dev)


def slab_measure(cfg_index: int, steps: int, warmup: int, mode: str, frames: int = 1,
                 balance: bool = True):
    """the points of ONE frame are sharded across the ranks (sensor
    i -> rank i % N).  mode "segments": the points are all-gathered and each
    rank traces only the ray segments inside its y-slab; "reduce_scatter":
    dense partial miss grids reduce-scattered by y-slab over NCCL, returns
    routed to slab owners; "fused": those grids summed by the slab finalize
    over symmetric peer memory.  Surface rows all-gathered in every mode.
    Strong scaling: value = points of the whole frame per second, time = max
    over ranks.  Returns the JSON line (rank 0) or None."""
    import torch
    import torch.distributed as dist

    from paper_2109_13176_b200 import GvomMap, parallel
    rank, world, local = dist_env()
    dev = torch.device("cuda", local)
    ensure_dist(dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    w = load_workload(cfg_index, frames, 0)  # the same frame on every rank
    f = w.frames[0]
    grid = dict(w.grid)
    grid["buffer_frames"] = 1
    mine = [(torch.from_numpy(s.points).to(dev), s.pose, s.rings)
            for i, s in enumerate(f.scans) if i % world == rank]
    npts_all = f.n_points
    stream = torch.cuda.Stream(device=dev)
    # capacity for the whole frame: data rows sit at their global ranks
    m = GvomMap(grid, max_points_per_frame=max(1, npts_all), device=dev, stream=stream)
    if mode == "segments":
        sm = parallel.SegmentMapper(m)
    else:
        sm = parallel.SlabMapper(m, ep_capacity=npts_all, fused=(mode == "fused"))
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    # every rank knows every sensor's pose and point count (the vehicle's state):
    # the segment partition then moves only the points
    meta = [(i % world, s.points.shape[0], s.pose, s.rings) for i, s in enumerate(f.scans)]
    meta.sort(key=lambda t: t[0])

    def step():
        m.shift(f.vehicle_xyz)
        if mode == "segments":
            sm.integrate(mine, meta=meta)
        else:
            sm.integrate(mine)
        sm.compute_maps()

    balanced = mode == "segments" and balance and world > 1
    with torch.cuda.stream(stream):
        for i in range(warmup):
            step()
            if balanced and i == 0:  # slab bounds from the first frame's row work
                sm.rebalance()
        torch.cuda.synchronize()
        dist.barrier()
        total = 0.0
        n0 = m.launch_count()
        with ClockSampler(local) as clk:
            for _ in range(steps):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                step()
                b.record(stream)
                b.synchronize()
                total += a.elapsed_time(b)
        launches = m.launch_count() - n0
        dist.barrier()
    t = torch.tensor([total], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total = float(t[0])
    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": npts_all * steps / (total / 1e3), "unit": "points/s",
            "n_gpus": world, "steps": steps, "warmup": warmup,
            "ms_per_step": total / steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32+int", "data": "synthetic",
            "config": {"workload": w.name, "points_per_frame": npts_all, "sensors": len(f.scans),
                       "grid": f"{m.nx}x{m.ny}x{m.nz}@{w.grid['res']}m", "buffer_frames": 1,
                       "parallelism": f"slab{world}: sensors sharded, " + {
                           "segments": "points all-gathered, each rank traces the ray "
                                       "segments inside its rows (gvom_integrate_slab)",
                           "fused": "miss grids summed over peer memory in the slab finalize",
                           "reduce_scatter": "reduce-scatter of the miss grids by y-slab"}[mode],
                       "slabs": list(sm.ys),
                       "slab_bounds": ("rebalanced from the warm-up frame's per-row work "
                                       "(gvom_row_work)") if balanced else "equal rows",
                       "l2": "flushed (256 MiB write) between steps",
                       "step": "shift+partial_scan+exchange+slab_finalize+slab maps"},
            "map_updates_per_s": steps / (total / 1e3),
            "gpu_launches": launches, "clocks": clk.summary(),
        }
    del sm, m
    dist.barrier()
    return line


def main_slab(args):
    """The partitioned path as the bench line (N > 1 by default: BASELINE
    configs[4], the multi-GPU workload; --config chooses another)."""
    import torch.distributed as dist
    cfg = 4 if args.config is None else args.config
    line = slab_measure(cfg, args.steps, args.warmup, args.slab_mode,
                        balance=not args.no_balance)
    if line is not None:
        emit(line)
    dist.barrier()
    dist.destroy_process_group()
    return 0


def pipelined_ms(w, frames, dev_frames, npts, dev, stream, out, args, barrier):
    """integrate(t+1) overlaps compute_maps(t) + export(t); no L2 flush (a
    flush would serialise the overlap), timed over the whole sequence."""
    from paper_2109_13176_b200 import GvomMap
    import torch
    gp = dict(w.grid)
    gp["pipeline"] = True
    mp_ = GvomMap(gp, max_points_per_frame=npts, device=dev, stream=stream)
    ms_ = mp_.map_stream

    def pstep(i):  # gvom_step: two graphs per step, fenced by event nodes
        f = frames[i % len(frames)]
        mp_.step(f.vehicle_xyz, dev_frames[i % len(frames)], out)

    for i in range(args.warmup):
        pstep(i)
    mp_.synchronize()
    barrier()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for i in range(args.steps):
        pstep(i)
    b.record(ms_)
    mp_.synchronize()
    ms = a.elapsed_time(b)
    del mp_
    barrier()
    return ms


def pcie_probe(dev, h2d_bytes: int, d2h_bytes: int, reps: int = 20):
    """Host<->device copy bandwidth of this box for the step's own transfer
    sizes (pinned host memory, CUDA events): the e2e number's ceiling."""
    import torch
    out = {}
    for name, nbytes, to_dev in (("h2d", h2d_bytes, True), ("d2h", d2h_bytes, False)):
        h = torch.empty(max(nbytes, 16), dtype=torch.uint8).pin_memory()
        d = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=dev)
        s = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(s):
            for _ in range(3):
                (d.copy_(h, non_blocking=True) if to_dev else h.copy_(d, non_blocking=True))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(reps):
                (d.copy_(h, non_blocking=True) if to_dev else h.copy_(d, non_blocking=True))
            b.record(s)
        b.synchronize()
        out[f"{name}_gbs"] = nbytes * reps / (a.elapsed_time(b) / 1e3) / 1e9
    out["bytes"] = {"h2d": h2d_bytes, "d2h": d2h_bytes}
    return out


def e2e_line(npts, steps, world, sync_value, sync_wall_s, pipe_s, d2h_bytes):
    """The e2e object: a user's stream of scans through gvom_step with pinned
    host buffers -- H2D of every scan and D2H of every step's 8 layers inside
    the timed region.  value = the pipelined handle (GVOM_FLAG_PIPELINE: scan
    t+1's copy and integrate overlap map processing t), wall clock over
    the whole sequence; the synchronous numbers (one step at a time) beside it.
    The rolling map cannot pipeline: value = the synchronous one there."""
    sync_wall = npts * steps * world / sync_wall_s
    piped = None if math.isnan(pipe_s) else npts * steps * world / pipe_s
    return {
        "value": piped if piped is not None else sync_value, "unit": "points/s",
        "mode": "pipelined" if piped is not None else "synchronous",
        "h2d_bytes_per_step": 16 * npts, "d2h_bytes_per_step": d2h_bytes, "steps": steps,
        "timing": ("GVOM_FLAG_PIPELINE handle through gvom_step, pinned host points in, all "
                   "layers out to pinned host (outputs double-buffered), steps submitted back to "
                   "back, wall clock over the sequence to the final synchronize")
        if piped is not None else "CUDA events around each synchronous gvom_step",
        "synchronous_value": sync_value,
        "synchronous_timing": "CUDA events around each gvom_step (pinned host points in, 8 "
                              "layers out to pinned host), synchronised every step",
        "synchronous_wall_value": sync_wall,
        "synchronous_wall_timing": "perf_counter around the host call + synchronize (host "
                                   "submit and ctypes marshalling included; L2 flush outside)",
    }


def pipelined_e2e_s(w, frames, host_frames, host_outs, npts, dev, stream, steps, args, barrier):
    """End to end with the pipelined handle: pinned host points in, all layers
    out to pinned host (two output sets, alternating), steps submitted back to
    back; wall-clock seconds for `steps` steps up to the final synchronize."""
    from paper_2109_13176_b200 import GvomMap
    gp = dict(w.grid)
    gp["pipeline"] = True
    mp_ = GvomMap(gp, max_points_per_frame=npts, device=dev, stream=stream)

    def pstep(i):
        f = frames[i % len(frames)]
        mp_.step(f.vehicle_xyz, host_frames[i % len(frames)], host_outs[i % 2])

    for i in range(max(3, args.warmup)):
        pstep(i)
    mp_.synchronize()
    barrier()
    t0 = time.perf_counter()
    for i in range(steps):
        pstep(i)
    mp_.synchronize()
    dt = time.perf_counter() - t0
    del mp_
    barrier()
    return dt


def main():
    _stdout_to_stderr()
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    # N > 1: the partitioned path unless --replicas
    if args.slab or (world > 1 and not args.replicas):
        return main_slab(args)
    if args.config is None:
        args.config = 1  # BASELINE metric config (c2)
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    from paper_2109_13176_b200 import GvomMap, LAYERS
    w = load_workload(args.config, args.frames, rank)
    if args.neg8cone:
        w.grid["neg_8cone"] = True
        w.name += "+neg8cone"
    if args.rolling:
        w.grid["rolling"] = True
        w.grid["buffer_frames"] = 1
        w.name += "+rolling"
    frames = w.frames
    npts = w.points_per_frame
    stream = torch.cuda.Stream(device=dev)
    m = GvomMap(w.grid, max_points_per_frame=npts, device=dev, stream=stream)
    dev_frames = [[(torch.from_numpy(s.points).to(dev), s.pose, s.rings) for s in f.scans]
                  for f in frames]
    out = {k: torch.empty((m.ny, m.nx), dtype=(torch.uint8 if k in ("hard", "soft", "neg")
                                               else torch.float32), device=dev)
           for k in LAYERS}
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    torch.cuda.synchronize()

    def step(i, scans, outs):
        # the public one-call-per-scan API: shift + integrate + compute_maps +
        # export as one CUDA graph launch (gvom_step)
        f = frames[i % len(frames)]
        m.step(f.vehicle_xyz, scans, outs)

    def step_eager(i, scans, outs):
        # the same work as separate calls (instrumented pass: events per launch)
        f = frames[i % len(frames)]
        m.shift(f.vehicle_xyz)
        m.integrate_scan(scans)
        m.compute_maps()
        m.export_layers(outs)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    with torch.cuda.stream(stream):
        # The timed region runs the step graph with no event nodes inside it
        # (event-record nodes between a graph's kernels cost several us per
        # step).  The dominant kernel's launch time (roofline) and the whole
        # integrate / compute_maps calls are timed in a second pass of graphed
        # steps with events around them; the per-launch breakdown comes from a
        # third, instrumented pass of separate calls.
        for i in range(args.warmup):
            step(i, dev_frames[i % len(frames)], out)
        stream.synchronize()
        # ---- timed region: device-resident inputs --------------------------
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        launches0 = m.launch_count()
        barrier()
        with ClockSampler(local) as clk:
            for i in range(args.steps):
                flush.zero_()  # L2 flush, outside the step events
                ev[i][0].record(stream)
                step(i, dev_frames[i % len(frames)], out)
                ev[i][1].record(stream)
            stream.synchronize()
        barrier()
        launches = m.launch_count() - launches0
        gstats = m.graph_stats()
        # kernel pass: graphed steps with events around the ray cast and
        # around the integrate / compute_maps calls
        m.set_timing(True, stages=["raycast", "integrate", "maps"])
        for i in range(3):
            step(i, dev_frames[i % len(frames)], out)
        stream.synchronize()
        m.stage_times()  # clear
        for i in range(args.steps):
            flush.zero_()
            step(i, dev_frames[i % len(frames)], out)
        stage = m.stage_times()
        m.set_timing(False)
        # instrumented pass (not timed): every stage bracketed by events
        m.set_timing(True)
        n_inst = min(args.steps, 50)
        for i in range(n_inst):
            flush.zero_()
            step_eager(i, dev_frames[i % len(frames)], out)
        stage_all = m.stage_times()
        m.set_timing(False)
        step_ms = [a.elapsed_time(b) for a, b in ev]
        total_ms = sum(step_ms)
        # ---- counts for the algorithmic bytes (from the GPU's own output) --
        lut, data, _ = m.export_frame(0)
        H = int(data["hits"].sum())
        Mi = int(data["misses"].sum()) + int((-1 - lut[lut < 0].astype(np.int64)).sum())
        k = int(data["hits"].shape[0])
        # ---- e2e: pinned host in, pinned host out ---------------------------
        host_frames = [[(torch.from_numpy(s.points).pin_memory(), s.pose, s.rings) for s in f.scans]
                       for f in frames]
        host_out = {kk: torch.empty(v.shape, dtype=v.dtype).pin_memory() for kk, v in out.items()}
        e2e_steps = max(3, min(args.steps, 100))
        for i in range(3):
            step(i, host_frames[i % len(frames)], host_out)
        stream.synchronize()
        barrier()
        e2e_ms = 0.0
        e2e_wall = 0.0
        for i in range(e2e_steps):
            flush.zero_()
            stream.synchronize()  # the flush stays outside the wall-clock interval
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            a.record(stream)
            step(i, host_frames[i % len(frames)], host_out)
            b.record(stream)
            b.synchronize()
            e2e_wall += time.perf_counter() - t0
            e2e_ms += a.elapsed_time(b)
        barrier()

        # ---- pipelined sustained sequence (GVOM_FLAG_PIPELINE) --------
        # (not with the rolling map: GVOM_FLAG_ROLLING excludes pipelining)
        pipe_ms = pipe_e2e_s = float("nan")
        if not w.grid.get("rolling", False):
            pipe_ms = pipelined_ms(w, frames, dev_frames, npts, dev, stream, out, args, barrier)
            host_outs = [host_out, {kk: torch.empty(v.shape, dtype=v.dtype).pin_memory()
                                    for kk, v in out.items()}]
            pipe_e2e_s = pipelined_e2e_s(w, frames, host_frames, host_outs, npts, dev, stream,
                                         e2e_steps, args, barrier)

    t = torch.tensor([total_ms, e2e_ms, pipe_ms, e2e_wall, pipe_e2e_s], dtype=torch.float64,
                     device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, e2e_ms, pipe_ms = float(t[0]), float(t[1]), float(t[2])
    e2e_wall, pipe_e2e_s = float(t[3]), float(t[4])
    pts_total = npts * args.steps * world
    value = pts_total / (total_ms / 1e3)
    e2e_value = npts * e2e_steps * world / (e2e_ms / 1e3)

    peak, peak_src = peaks()
    traffic, traffic_src, inst = measured_traffic(w.name)
    ray_ms, ray_n = stage["raycast"]
    ray_launch_ms = ray_ms / max(ray_n, 1)
    scans_per_frame = len(frames[0].scans)
    launches_per_frame = max(1, round(ray_n / args.steps))  # sensors are batched per launch
    ray_bytes = (16 * npts + 8 * Mi + 8 * H) / launches_per_frame  # per launch
    ray_gbs = ray_bytes / (ray_launch_ms / 1e3) / 1e9
    V = m.nx * m.ny * m.nz
    # integrate / compute_maps: one event pair around each whole call inside
    # the timed, graphed steps (GVOM_STAGE_INTEGRATE / _MAPS)
    integ_ms = stage["integrate"][0] / max(stage["integrate"][1], 1)
    B_int = 16 * npts + 48 * H + 8 * Mi + 4 * V
    K = int(w.grid["buffer_frames"])
    maps_ms = stage["maps"][0] / max(stage["maps"][1], 1)

    l2_red = l2_red_ceiling() if rank == 0 and not args.no_l2_probe else None
    red_req = measured_red_requests(w.name)
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = oracle_run(w, args.cpu_budget)
        line = {
            "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32+int", "data": "synthetic",
            "config": {"workload": w.name, "points_per_scan": npts, "sensors": scans_per_frame,
                       "grid": f"{m.nx}x{m.ny}x{m.nz}@{w.grid['res']}m", "buffer_frames": K,
                       "frames_cycled": len(frames), "l2": "flushed (256 MiB write) between steps",
                       "step": "shift+integrate_scan+compute_maps+export of all 8 layers",
                       "launch": "gvom_step: one CUDA graph launch per step"},
            "graph": gstats,
            "map_updates_per_s": world * args.steps / (total_ms / 1e3),
            "roofline": {"bound": "hbm", "kernel": "k_raycast", "achieved": ray_gbs,
                         "peak": peak, "unit": "GB/s", "frac": ray_gbs / peak, "traffic": traffic,
                         "traffic_source": traffic_src, "peak_source": peak_src,
                         "launch_ms": ray_launch_ms,
                         "bytes_per_launch": ray_bytes,
                         "issue": None if inst is None else {
                             "warp_inst_per_launch": inst,
                             "achieved_ginst_s": inst / (ray_launch_ms / 1e3) / 1e9,
                             "peak_ginst_s": ISSUE_PEAK_GINST_S,
                             "frac": inst / (ray_launch_ms / 1e3) / 1e9 / ISSUE_PEAK_GINST_S,
                             "note": "the kernel's actual limiter: warp instructions (ncu, "
                                     "committed capture) / live launch time vs the SM issue "
                                     "peak; its miss RMWs are L2-resident at this size"},
                         "bytes_model": "16 N + 8 M + 8 H (points, miss RMW, endpoint bit RMW)",
                         "l2_red": l2_red,
                         "raycast_red": {
                             "g_increments_s": Mi / launches_per_frame / (ray_launch_ms / 1e3) / 1e9,
                             "g_l2_requests_s": (None if red_req is None else
                                                 red_req / (ray_launch_ms / 1e3) / 1e9),
                             "note": "miss increments (M per launch) and L2 reduction requests "
                                     "per launch (ncu lts__t_requests_srcunit_tex_op_red, "
                                     "committed capture) over the live launch time; compare "
                                     "l2_red (the probe's ceiling at the miss grid's size)"}},
            "integrate": {"ms_per_frame": integ_ms, "points_per_s": npts / (integ_ms / 1e3),
                          "B_int_bytes": B_int, "hbm_frac": B_int / (integ_ms / 1e3) / 1e9 / peak,
                          "H": H, "M": Mi, "k": k,
                          "timing": "events around gvom_integrate_scan in a second pass of graphed "
                                    "steps (GVOM_STAGE_INTEGRATE), L2 flushed between steps"},
            "compute_maps_ms": maps_ms,
            "compute_maps_timing": "events around gvom_compute_maps in a second pass of graphed "
                                   "steps (GVOM_STAGE_MAPS)",
            "stages_ms_per_step": {s: v[0] / n_inst for s, v in stage_all.items() if v[1]},
            "stages_note": "separate instrumented pass (events around every launch, "
                           "separate calls without a graph)",
            "e2e": dict(e2e_line(npts, e2e_steps, world, e2e_value, e2e_wall, pipe_e2e_s,
                                 m.nx * m.ny * (4 * 5 + 3)),
                        pcie=pcie_probe(dev, 16 * npts, m.nx * m.ny * (4 * 5 + 3))),
            "pipelined": None if math.isnan(pipe_ms) else {
                "value": pts_total / (pipe_ms / 1e3), "unit": "points/s",
                "map_updates_per_s": world * args.steps / (pipe_ms / 1e3),
                "note": "GVOM_FLAG_PIPELINE through gvom_step (integrate graph on the handle's "
                        "stream, map graph on the map stream): integrate(t+1) overlaps "
                        "compute_maps(t); sustained sequence, no L2 flush between steps"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
    if world == 1 and not args.no_partitioned:
        # the partitioned path (what N > 1 runs) at one rank: the N = 1 point of
        # its strong-scaling curve
        part = slab_measure(4, min(args.steps, 20), 3, args.slab_mode)
        if rank == 0:
            part["note"] = ("BASELINE configs[4] through the slab-partition path on one rank "
                            "(the N = 1 point of `bench.py --gpus N`, N > 1)")
            line["partitioned"] = part
    if rank == 0:
        emit(line)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
