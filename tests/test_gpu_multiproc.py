"""The partitioned path across real GPUs: torchrun, one process per GPU, NCCL
and symmetric memory (tests/multi_gpu_worker.py).  Runs when at least two
GPUs are visible and skips otherwise (the round's GPU box has one; the
emulated-rank tests in test_gpu_slab.py cover the kernels there)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("config", [0, 3])
def test_partitioned_path_two_gpus(config):
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip(f"needs >= 2 GPUs (found {n})")
    P = 4 if n >= 4 else 2
    env = dict(os.environ, GVOM_MP_CONFIG=str(config))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={P}", "--master-addr", "127.0.0.1",
                        "--master-port", str(29700 + config), os.path.join(HERE, "multi_gpu_worker.py")],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    for mode in ("segments", "segments_balanced", "reduce_scatter", "fused", "segments_motion"):
        assert f"MULTI-GPU {mode} P={P} ok" in r.stdout
