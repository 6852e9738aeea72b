"""gvom_step (include/gvom.h): shift + integrate + compute_maps + export as one
CUDA graph launch per frame must give exactly the results of the separate
calls (parity against the oracle, frame by frame), patch the cached graph
while the launch topology is unchanged, re-instantiate when it changes, and
run the same kernels without a graph when capture does not apply."""
import dataclasses

import numpy as np
import pytest
import torch

from paper_2109_13176_b200 import GvomMap, SensorOutside, synth
from paper_2109_13176_b200.gvom import LAYER_U8, LAYERS
from tests.gpu_helpers import compare_layers, layers_np, run_sequence, to_dev
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def test_step_c2_matches_oracle():
    m, _ = run_sequence(synth.workload(1), use_step=True)
    st = m.graph_stats()
    assert st["graph_launches"] == 1 and st["eager_steps"] == 0


@pytest.mark.parametrize("speed", [4.5, 12.0])
def test_step_motion_sequence_graph_updates(speed):
    # shift + merge + eviction through the graph path; one instantiation,
    # every later frame patches the cached graph with new arguments
    w = synth.config3(speed=speed, n_frames=12, columns=1024)
    m, _ = run_sequence(w, check_every=4, use_step=True)
    st = m.graph_stats()
    assert st["graph_launches"] == 12 and st["eager_steps"] == 0
    assert st["instantiations"] == 1, st


def test_step_c4_three_lidars():
    m, _ = run_sequence(synth.workload(3), use_step=True)
    assert m.graph_stats()["graph_launches"] == 1


def test_step_pinned_host_points_use_graph():
    m, _ = run_sequence(synth.workload(1), host=True, check_merged=False, use_step=True)
    assert m.graph_stats()["graph_launches"] == 1


def test_step_pageable_host_points_run_eagerly():
    w = synth.workload(0)
    f = w.frames[0]
    m = GvomMap(w.grid, max_points_per_frame=f.n_points)
    om = O.OracleMap(w.grid)
    om.shift(f.vehicle_xyz)
    om.integrate([(s.points, s.pose) for s in f.scans])
    _, lay = m.step(f.vehicle_xyz, [(s.points, s.pose, s.rings) for s in f.scans])
    m.synchronize()
    compare_layers({k: v.cpu().numpy() for k, v in lay.items()}, om.compute_maps())
    st = m.graph_stats()
    assert st["eager_steps"] == 1 and st["graph_launches"] == 0


def test_step_topology_change_reinstantiates():
    # an empty scan keeps the topology (sensors with equal ring counts share one
    # ray-cast and one endpoint launch): the cached graph is patched in place.
    # A scan with another ring count (unordered cloud) adds a batch: the graph
    # is re-instantiated, and coming back re-instantiates again.  Results match
    # the oracle throughout.
    w = synth.workload(3)
    f = w.frames[0]
    m = GvomMap(w.grid, max_points_per_frame=f.n_points)
    om = O.OracleMap(w.grid)
    empty = dataclasses.replace(f.scans[1], points=f.scans[1].points[:0])
    unordered = dataclasses.replace(f.scans[2], rings=0)
    seq = [(list(f.scans), 1), ([f.scans[0], empty, f.scans[2]], 1),
           ([f.scans[0], f.scans[1], unordered], 2), (list(f.scans), 3)]
    for i, (scans, inst) in enumerate(seq):
        om.shift(f.vehicle_xyz)
        om.integrate([(s.points, s.pose) for s in scans])
        m.step(f.vehicle_xyz, [to_dev(s) for s in scans], export=False)
        compare_layers(layers_np(m), om.compute_maps())
        st = m.graph_stats()
        assert st["graph_launches"] == i + 1 and st["instantiations"] == inst, (i, st)


def test_step_sensor_outside_rejected_before_capture():
    w = synth.workload(1)
    f = w.frames[0]
    m = GvomMap(w.grid, max_points_per_frame=f.n_points)
    m.step(f.vehicle_xyz, [to_dev(s) for s in f.scans])
    before = layers_np(m)
    far = synth.pose_matrix(np.eye(3), (500.0, 0.0, 0.0))
    with pytest.raises(SensorOutside):
        m.step(f.vehicle_xyz, [(torch.from_numpy(f.scans[0].points).cuda(), far, 64)])
    m.compute_maps()
    after = layers_np(m)
    for k in before:
        assert np.array_equal(np.nan_to_num(before[k], nan=-7), np.nan_to_num(after[k], nan=-7))
    # the handle still works, through the graph
    m.step(f.vehicle_xyz, [to_dev(s) for s in f.scans])
    assert m.graph_stats()["graph_launches"] == 2


@pytest.mark.parametrize("pinned", [True, False])
def test_step_host_outputs(pinned):
    # host destinations: pinned ones stay in the graph, each layer copied out as
    # soon as it is final; pageable ones run without a graph; same layers as the
    # device destinations
    w = synth.workload(1)
    f = w.frames[0]
    scans = [to_dev(s) for s in f.scans]
    ref = GvomMap(w.grid, max_points_per_frame=f.n_points)
    _, dev = ref.step(f.vehicle_xyz, scans)
    ref.synchronize()
    m = GvomMap(w.grid, max_points_per_frame=f.n_points)
    host = {k: torch.empty(v.shape, dtype=v.dtype) for k, v in dev.items()}
    if pinned:
        host = {k: v.pin_memory() for k, v in host.items()}
    m.step(f.vehicle_xyz, scans, host)
    m.synchronize()
    for k, v in dev.items():
        assert np.array_equal(np.nan_to_num(host[k].numpy(), nan=-7),
                              np.nan_to_num(v.cpu().numpy(), nan=-7)), k
    st = m.graph_stats()
    assert (st["graph_launches"], st["eager_steps"]) == ((1, 0) if pinned else (0, 1)), st


def test_step_on_pipelined_handle_with_variants():
    # GVOM_FLAG_PIPELINE + NEG_8CONE + SLOPE_SKIP_OBSTACLES through gvom_step:
    # two graphs per step (integrate on the handle's stream, map processing on
    # the map stream) fenced by external event nodes; frame by frame parity
    w = synth.config3(speed=4.5, n_frames=10, columns=512)
    grid = dict(w.grid)
    grid.update(pipeline=True, neg_8cone=True, slope_skip_obstacles=True)
    m, _ = run_sequence(synth.Workload(w.name + "_pipe_variants", grid, w.frames, w.world),
                        use_step=True, check_merged=False)
    st = m.graph_stats()
    assert st["graph_launches"] == len(w.frames) and st["eager_steps"] == 0, st


def test_pipelined_step_graphs_overlap_frames():
    # back-to-back pipelined steps without synchronisation (the slot fences are
    # graph event nodes), then every frame's layers checked against the oracle
    w = synth.config3(speed=12.0, n_frames=12, columns=512)
    grid = dict(w.grid)
    grid["pipeline"] = True
    npts = max(f.n_points for f in w.frames)
    m = GvomMap(grid, max_points_per_frame=npts)
    om = O.OracleMap(grid)
    outs, refs = [], []
    for f in w.frames:
        _, lay = m.step(f.vehicle_xyz, [to_dev(s) for s in f.scans])
        outs.append(lay)
        om.shift(f.vehicle_xyz)
        om.integrate([(s.points, s.pose) for s in f.scans])
        refs.append(om.compute_maps())
    m.synchronize()
    for lay, L in zip(outs, refs):
        compare_layers({k: v.cpu().numpy() for k, v in lay.items()}, L)
    st = m.graph_stats()
    assert st["graph_launches"] == len(w.frames), st


def test_pipelined_step_pinned_host_points_and_outputs():
    # pinned host points on a pipelined handle: each scan is copied on the
    # copy stream into one of two staging buffers while the previous scan's
    # integrate still runs; pinned host outputs (alternating sets).  Back to
    # back without synchronisation, then every frame against the oracle; an
    # eager integrate_scan from host memory in the middle shares staging 0.
    w = synth.config3(speed=12.0, n_frames=10, columns=512)
    grid = dict(w.grid)
    grid["pipeline"] = True
    npts = max(f.n_points for f in w.frames)
    m = GvomMap(grid, max_points_per_frame=npts)
    om = O.OracleMap(grid)
    outs, refs = [], []
    for i, f in enumerate(w.frames):
        scans = [to_dev(s, host=True) for s in f.scans]
        om.shift(f.vehicle_xyz)
        om.integrate([(s.points, s.pose) for s in f.scans])
        if i == 5:  # the separate calls, host points through staging buffer 0
            m.shift(f.vehicle_xyz)
            m.integrate_scan(scans)
            m.compute_maps()
            m.synchronize()
            compare_layers(layers_np(m), om.compute_maps())
            continue
        host = {k: torch.empty((m.ny, m.nx), dtype=torch.uint8 if k in LAYER_U8
                               else torch.float32).pin_memory() for k in LAYERS}
        _, lay = m.step(f.vehicle_xyz, scans, host)
        outs.append(lay)
        refs.append(om.compute_maps())
    m.synchronize()
    for lay, L in zip(outs, refs):
        compare_layers({k: v.cpu().numpy() for k, v in lay.items()}, L)
    st = m.graph_stats()
    assert st["graph_launches"] == len(w.frames) - 1 and st["eager_steps"] == 0, st


@pytest.mark.parametrize("pipeline", [False, True])
def test_step_capture_failure_rolls_back(pipeline):
    # a failed capture must not leave the ring naming a slot whose
    # frame never ran.  Frame 1's step fails (injected capture fault): the
    # state is as if it had never been called, so after frames 0 and 2 the
    # map equals the oracle's with frames 0 and 2 only (its shift stands).
    w = synth.config3(speed=12.0, n_frames=3, columns=1024)
    if pipeline:
        w.grid["pipeline"] = True
    m = GvomMap(w.grid, max_points_per_frame=w.points_per_frame)
    om = O.OracleMap(w.grid)
    for i, f in enumerate(w.frames):
        scans = [to_dev(s) for s in f.scans]
        if i == 1:
            m.inject_fault(1)
            with pytest.raises(Exception):
                m.step(f.vehicle_xyz, scans, export=False)
            om.shift(f.vehicle_xyz)
            continue
        m.step(f.vehicle_xyz, scans, export=False)
        om.shift(f.vehicle_xyz)
        om.integrate([(s.points, s.pose) for s in f.scans])
    compare_layers(layers_np(m), om.compute_maps())
    lut, data, origin = m.export_frame(1)
    assert np.array_equal(origin, om.buffer[-2].origin)
    assert np.array_equal(lut, om.buffer[-2].lut)


def test_destroy_with_pipelined_work_in_flight():
    # gvom_destroy drains the handle's streams (integrate, map, copy streams)
    # before releasing, so freeing the workspace right after is safe: steps are
    # submitted back to back with pinned host buffers, the handle is closed
    # without a synchronise, its workspace dropped, and a fresh handle then
    # reproduces the oracle on the same memory pool
    w = synth.config3(speed=12.0, n_frames=4, columns=512)
    grid = dict(w.grid)
    grid["pipeline"] = True
    npts = max(f.n_points for f in w.frames)
    for _ in range(3):
        m = GvomMap(grid, max_points_per_frame=npts)
        for f in w.frames:
            host = {k: torch.empty((m.ny, m.nx), dtype=torch.uint8 if k in LAYER_U8
                                   else torch.float32).pin_memory() for k in LAYERS}
            m.step(f.vehicle_xyz, [to_dev(s, host=True) for s in f.scans], host)
        m.close()
        del m
        torch.cuda.empty_cache()
    run_sequence(w, use_step=True, check_every=2)

