"""The two-warps-per-ray-tile ray cast (k_raycast_split: half 1 resumes every
walk at ceil(Tw / 2) from the exact state there; the default for frames of
more than two waves) must give the oracle's maps bit for bit on every frame
size.  GVOM_RAY_SPLIT=1 forces it and is read once per process, so the parity
tests run in a child process with it set."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def test_split_ray_cast_parity():
    env = dict(os.environ, GVOM_RAY_SPLIT="1")
    tests = ["test_gpu_parity.py::test_c1_tiny", "test_gpu_parity.py::test_c2_single_scan",
             "test_gpu_parity.py::test_c3_motion_sequence",
             "test_gpu_parity.py::test_c4_three_lidars_full_size",
             "test_gpu_parity.py::test_ragged_small_clouds",
             "test_gpu_random.py"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        *[os.path.join(HERE, t) for t in tests]],
                       cwd=os.path.dirname(HERE), env=env, capture_output=True, text=True,
                       timeout=1500)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
