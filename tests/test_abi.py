"""CPU-side checks of the C-ABI library: it loads, exports every symbol that
include/gvom.h declares, validates configs and sizes its workspace (no compute
calls without a GPU), and the package has no CPU fallback."""
import ctypes as C
import os
import re

import pytest

import __graft_entry__
from paper_2109_13176_b200 import gvom, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    __graft_entry__.build()
    return gvom.load_library()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "gvom.h")).read()
    return sorted(set(re.findall(r"GVOM_API\s+[\w\s\*]+?\b(gvom_\w+)\s*\(", src)))


def test_header_declares_expected(lib):
    syms = declared_symbols()
    assert set(gvom.EXPORTED) == set(syms), (set(gvom.EXPORTED) ^ set(syms))


def test_every_declared_symbol_exported(lib):
    for s in declared_symbols():
        assert hasattr(lib, s), s


def test_abi_version_and_status_strings(lib):
    assert lib.gvom_abi_version() == 1
    assert lib.gvom_status_string(-4) == b"sensor outside the map"
    assert lib.gvom_status_string(0) == b"ok"


def test_struct_layouts_match_header():
    # 8-byte aligned C structs: sizes fixed by include/gvom.h
    assert C.sizeof(gvom.Voxel) == 32
    assert C.sizeof(gvom.Scan) == 8 + 8 + 96 + 8
    assert C.sizeof(gvom.Config) == 12 + 4 + 8 + 8 + 4 + 4 + 8 + 8 * 3 + 8 + 8 + 4 + 4


def test_workspace_sizing(lib):
    g = synth.grid_cfg(256, 256, 64, 0.25)
    n = gvom.workspace_bytes(g, 131072)
    V = 256 * 256 * 64
    # K = 8 LUTs dominate; data rows + bitmasks + staging + layers on top
    assert 8 * 4 * V < n < 8 * 4 * V * 1.5
    bad = dict(g)
    bad["slope_window"] = 4
    assert gvom.workspace_bytes(bad, 10) == 0
    bad = dict(g)
    bad["res"] = -1.0
    assert gvom.workspace_bytes(bad, 10) == 0


def test_cone_search_limits(lib):
    # packed sweep keys: (K + 3) << (16 + ceil(log2 nz)) < 2^32 (include/gvom.h)
    g = synth.grid_cfg(64, 64, 2048, 0.25)
    for K, ok in ((28, True), (29, False), (60, False)):
        g["neg_obs_search_cells"] = K
        assert (gvom.workspace_bytes(g, 10) > 0) == ok, K
    g = synth.grid_cfg(64, 64, 1000, 0.25)  # nz rounds up to 1024
    for K, ok in ((60, True), (61, False)):
        g["neg_obs_search_cells"] = K
        assert (gvom.workspace_bytes(g, 10) > 0) == ok, K
    # the sweep's shared-memory ring must hold two key lines of max(nx, ny)
    g = synth.grid_cfg(4096, 8, 8, 0.25)
    g["neg_obs_search_cells"] = 8
    assert gvom.workspace_bytes(g, 10) > 0
    g = synth.grid_cfg(8192, 8, 8, 0.25)
    g["neg_obs_search_cells"] = 8
    assert gvom.workspace_bytes(g, 10) == 0
    # GVOM_FLAG_NEG_8CONE: the search tile (32 + 2K)^2 and its summed-area table fit in smem
    g = synth.grid_cfg(64, 64, 16, 0.25)
    g["neg_8cone"] = True
    for K, ok in ((82, True), (83, False)):
        g["neg_obs_search_cells"] = K
        assert (gvom.workspace_bytes(g, 10) > 0) == ok, K


def test_create_rejects_bad_arguments(lib):
    cfg = gvom.make_config(synth.grid_cfg(8, 8, 8, 0.25), 16)
    h = C.c_void_p()
    # null workspace and misaligned workspace are rejected before touching CUDA
    assert lib.gvom_create(C.byref(cfg), None, 1 << 20, None, C.byref(h)) == -1
    assert lib.gvom_create(C.byref(cfg), C.c_void_p(0x1001), 1 << 30, None, C.byref(h)) == -1
    assert lib.gvom_create(C.byref(cfg), C.c_void_p(0x100000), 16, None, C.byref(h)) == -2


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        gvom.GvomMap(synth.grid_cfg(8, 8, 8, 0.25), 16)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2109_13176_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "from oracle" not in src and "import oracle" not in src, f
                assert "gvom_oracle" not in src, f
