"""Device plumbing: tensor staging, streams and caller-owned workspaces.

PyTorch is used only for device memory and streams; all arithmetic on the
hot path is in the CUDA library.
"""

from __future__ import annotations

import numpy as np
import torch

_NP_TO_TORCH = {
    np.dtype(np.uint8): torch.uint8,
    np.dtype(np.uint16): torch.uint16,
    np.dtype(np.uint32): torch.uint32,
    np.dtype(np.int32): torch.int32,
    np.dtype(np.int64): torch.int64,
    np.dtype(np.float32): torch.float32,
    np.dtype(np.bool_): torch.bool,
}


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise RuntimeError("probestream needs a CUDA device (B200, sm_100a); none is visible")


def is_tensor(x) -> bool:
    return isinstance(x, torch.Tensor)


def device_of(*xs) -> torch.device:
    for x in xs:
        if isinstance(x, torch.Tensor) and x.is_cuda:
            return x.device
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def to_device(x, dtype=None, device=None) -> torch.Tensor:
    """numpy / list / tensor -> contiguous CUDA tensor (zero-copy if already one)."""
    if isinstance(x, torch.Tensor):
        t = x
        if dtype is not None and t.dtype != dtype:
            t = t.to(dtype)
        if not t.is_cuda:
            t = t.to(device or device_of())
        return t.contiguous()
    arr = np.asarray(x)
    if dtype is not None:
        npd = {v: k for k, v in _NP_TO_TORCH.items()}[dtype]
        arr = arr.astype(npd, copy=False)
    arr = np.ascontiguousarray(arr)
    t = torch.from_numpy(arr) if arr.dtype in _NP_TO_TORCH else torch.from_numpy(arr.astype(np.int64))
    return t.to(device or device_of(), non_blocking=False)


def to_numpy(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class Workspace:
    """Grow-only scratch buffer per device (the C ABI never allocates)."""

    _bufs: dict = {}

    @classmethod
    def get(cls, nbytes: int, device: torch.device, slot: str = "default") -> torch.Tensor:
        key = (device.index, slot)
        buf = cls._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
            cls._bufs[key] = buf
        return buf
