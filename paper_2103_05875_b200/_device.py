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
    """Scratch memory for one C-ABI call (the C ABI never allocates).

    ``slot`` is either a caller-owned uint8 CUDA tensor -- the frame pipeline
    (server.KindStream, distributed.DistKindStream, UpdateAtlasLayout) owns
    one per stage, sized once for its probe count, so no two sessions or
    streams ever share scratch and a captured CUDA graph's pointers stay
    valid -- or a name, for the one-off drop-in calls of the reference API:
    those run on the current stream and get a buffer from a per-(device,
    name) cache.  A larger request replaces the cached buffer; the old one
    goes back to PyTorch's stream-ordered caching allocator, which is safe
    because only current-stream drop-in calls use named slots."""

    _bufs: dict = {}

    @classmethod
    def get(cls, nbytes: int, device: torch.device, slot="default") -> torch.Tensor:
        if isinstance(slot, torch.Tensor):
            if slot.numel() < nbytes or slot.dtype != torch.uint8:
                raise ValueError(f"workspace of {slot.numel()} bytes < the {nbytes} needed")
            return slot
        key = (device.index, slot)
        buf = cls._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
            cls._bufs[key] = buf
        return buf


def workspace(nbytes: int, device) -> torch.Tensor:
    """A caller-owned workspace tensor of ``nbytes`` (see Workspace)."""
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


# --- active flags on the device, for any ProbeVolume-like object ------------------------

_ACTIVE_CACHE: dict = {}
_ACTIVE_CACHE_MAX = 64


def active_flags(volume, device) -> torch.Tensor:
    """uint8 copy of ``volume.active`` on ``device``.

    Works for the reference's own ``ProbeVolume`` (volume.py:68-144), which
    only has the numpy ``active`` flags (read-only after __post_init__),
    and for any duck-typed volume.  Cached per (flags array, device); the
    cache holds a reference to the array, so its id cannot be reused by a
    different array while the entry lives."""
    flags = volume.active
    if isinstance(flags, torch.Tensor):
        t = flags.to(device=device, dtype=torch.uint8)
        return t.contiguous()
    key = (id(flags), str(device))
    hit = _ACTIVE_CACHE.get(key)
    if hit is not None and hit[0] is flags:
        return hit[1]
    arr = np.asarray(flags, dtype=bool).reshape(-1)
    t = torch.from_numpy(arr.astype(np.uint8)).to(device)
    if len(_ACTIVE_CACHE) >= _ACTIVE_CACHE_MAX:
        _ACTIVE_CACHE.pop(next(iter(_ACTIVE_CACHE)))
    if not (isinstance(flags, np.ndarray) and not flags.flags.writeable):
        return t  # mutable flags: never cached
    _ACTIVE_CACHE[key] = (flags, t)
    return t
