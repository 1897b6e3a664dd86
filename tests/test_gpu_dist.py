"""Slab-sharded frame on >= 2 GPUs (torchrun, NCCL) is bit-identical to the
single-GPU pipeline (runs only where two GPUs are visible)."""

import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs 2 GPUs")
@pytest.mark.parametrize("config,extra", [("c1", []), ("c2", []),
                                          ("c1", ["--graphs", "--gop", "3", "--frames", "7"]),
                                          ("c1", ["--nccl"]),
                                          ("c1", ["--nccl", "--graphs", "--gop", "3", "--frames", "5"])])
def test_sharded_frame_matches_single_gpu(config, extra):
    n = min(torch.cuda.device_count(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + n + 10 * len(extra) + 100 * ("--nccl" in extra)),
           str(ROOT / "tools" / "dist_check.py"), "--config", config, *extra]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert "DIST OK" in res.stdout
