"""Host-side cost of one gvom_step (the call's wall time, no synchronisation)
for a pipelined handle with pinned host points and outputs (c2), and where it
goes: python marshalling vs the library call.   python tools/host_submit.py"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_13176_b200 import GvomMap, synth  # noqa: E402
from paper_2109_13176_b200.gvom import LAYER_U8, LAYERS  # noqa: E402


def main(steps=300):
    w = synth.config2(n_frames=4)
    g = dict(w.grid)
    g["pipeline"] = True
    npts = max(f.n_points for f in w.frames)
    m = GvomMap(g, max_points_per_frame=npts)
    frames = [[(torch.from_numpy(s.points).pin_memory(), s.pose, s.rings) for s in f.scans]
              for f in w.frames]
    outs = [{k: torch.empty((m.ny, m.nx), dtype=torch.uint8 if k in LAYER_U8
                            else torch.float32).pin_memory() for k in LAYERS} for _ in range(2)]
    for i in range(10):
        m.step(w.frames[i % 4].vehicle_xyz, frames[i % 4], outs[i % 2])
    m.synchronize()
    call = []
    t0 = time.perf_counter()
    for i in range(steps):
        a = time.perf_counter()
        m.step(w.frames[i % 4].vehicle_xyz, frames[i % 4], outs[i % 2])
        call.append(time.perf_counter() - a)
    m.synchronize()
    total = time.perf_counter() - t0
    # the library call alone: same arguments, marshalled once
    p = (C.c_double * 3)(*[float(v) for v in w.frames[0].vehicle_xyz])
    dlt = (C.c_int64 * 3)()
    arr, n, keep = m._scan_array(frames[0])
    res, ptrs, sizes = m._layer_dst(outs[0])
    lib_t = []
    for i in range(steps):
        a = time.perf_counter()
        rc = m.lib.gvom_step(m.h, p, arr, n, ptrs, sizes, None, None, 0, dlt)
        lib_t.append(time.perf_counter() - a)
        assert rc == 0
    m.synchronize()
    pa = m.lib  # cudaPointerGetAttributes cost, through torch's cudart
    print(json.dumps({"steps": steps, "wall_us_per_step": 1e6 * total / steps,
                      "step_call_us_median": 1e6 * float(np.median(call)),
                      "lib_call_us_median": 1e6 * float(np.median(lib_t)),
                      "graph_stats": m.graph_stats()}))


if __name__ == "__main__":
    main()
