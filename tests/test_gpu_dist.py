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


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")
def test_peer_wait_times_out_instead_of_hanging():
    """A flag no peer ever raises: the bounded wait gives up after its
    timeout, records the flag index in the host-mapped error word, and the
    host check raises (PS_ERR_CUDA -> RuntimeError) instead of hanging the
    stream (ps_peer.cu peer_wait_kernel, ps_peer_status)."""
    import time

    from paper_2103_05875_b200 import _native as N
    from paper_2103_05875_b200 import distributed as dd

    dev = torch.device("cuda", 0)
    flags = torch.zeros(3, dtype=torch.int64, device=dev)
    flags[0] = 5
    flags[2] = 5  # flag 1 never reaches 5
    err = torch.zeros(1, dtype=torch.int32, pin_memory=True)
    st = torch.cuda.current_stream(dev).cuda_stream
    t0 = time.perf_counter()
    N.call("ps_peer_wait", flags.data_ptr(), 3, 5, None, 0, err.data_ptr(), 50_000_000, st)
    torch.cuda.synchronize(dev)
    assert time.perf_counter() - t0 < 10.0
    assert int(err[0]) == 2  # flag index 1, stored + 1
    with pytest.raises(RuntimeError, match="never signalled"):
        N.call("ps_peer_status", err.data_ptr())
    # satisfied flags: returns at once, error word untouched
    flags[1] = 7
    err.zero_()
    N.call("ps_peer_wait", flags.data_ptr(), 3, 5, None, 0, err.data_ptr(), 50_000_000, st)
    torch.cuda.synchronize(dev)
    assert int(err[0]) == 0
    N.call("ps_peer_status", err.data_ptr())
    # the process-wide word used by the sharded frame starts healthy
    dd.check_peers()
