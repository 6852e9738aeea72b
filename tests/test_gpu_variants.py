"""The non-default kernel variants behind A/B switches must give the oracle's
maps bit for bit too, so an A/B timing never compares a wrong kernel:

* GVOM_COL_FAST=1   -- k_columns_fast (three round trips per column);
* GVOM_SLOPE_COMPACT=1 -- k_slope_c over the compacted column list;
* GVOM_COL_EARLY=1  -- k_columns<true> (edge loads issued first);
* GVOM_NEG_DEFER=0  -- the negative decision right after the cone sweep
  (k_neg_decide) instead of inside the export.

The switches are read once per process, so each set runs the parity tests in
a child process (as test_gpu_split.py does for the split ray cast)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))

TESTS = ["test_gpu_parity.py::test_c1_tiny", "test_gpu_parity.py::test_c2_single_scan",
         "test_gpu_parity.py::test_c3_motion_sequence",
         "test_gpu_parity.py::test_ragged_small_clouds", "test_gpu_random.py",
         "test_gpu_step.py"]


@pytest.mark.parametrize("switches", [
    {"GVOM_COL_FAST": "1", "GVOM_SLOPE_COMPACT": "1"},
    {"GVOM_COL_EARLY": "1", "GVOM_NEG_DEFER": "0"},
], ids=["colfast_slopecompact", "col_early_neg_eager"])
def test_variant_parity(switches):
    env = dict(os.environ, **switches)
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        *[os.path.join(HERE, t) for t in TESTS]],
                       cwd=os.path.dirname(HERE), env=env, capture_output=True, text=True,
                       timeout=1500)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
