"""Probe index buffer (§8(f) row 4).

The reference's server module, which would carry this, is absent;
the spec fixes the format: ``uvarint(count)`` then, per (slot, probe) entry in
slot order, ``uvarint(slot delta)`` and ``uvarint(zigzag(probe delta))`` with
the previous entry starting at (0, 0).  ``encode_index_device`` builds it on
the GPU from the slot assignment's device entries; ``decode_index`` is the
client-side inverse (host).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as D
from . import _native as N


def encode_index_device(entries: torch.Tensor, entry_count: torch.Tensor, out=None, out_len=None,
                        workspace=None):
    """Stream-ordered index buffer of the first ``entry_count`` entries; a
    session passes its own ``workspace`` (uint8 tensor), one-off calls use a
    named per-device slot on the current stream."""
    cap = int(entries.shape[0])
    dev = entries.device
    if out is None:
        out = torch.empty(1 + 20 * max(cap, 1), dtype=torch.uint8, device=dev)
    if out_len is None:
        out_len = torch.zeros(1, dtype=torch.int64, device=dev)
    ws = D.Workspace.get(N.lib().ps_index_workspace_bytes(cap), dev,
                         "index" if workspace is None else workspace)
    N.call("ps_encode_index", entries.data_ptr(), entry_count.data_ptr(), cap, out.data_ptr(),
           out_len.data_ptr(), ws.data_ptr(), ws.numel(), D.stream_ptr(dev))
    return out, out_len


def encode_index_buffer(entries) -> bytes:
    """(slot, probe) pairs sorted by slot -> bytes; unsorted input is rejected."""
    arr = np.asarray(list(entries), dtype=np.int64).reshape(-1, 2)
    if len(arr) > 1 and np.any(np.diff(arr[:, 0]) <= 0):
        raise ValueError("index entries must be strictly increasing in slot")
    dev = D.device_of()
    t = torch.from_numpy(arr.copy()).to(dev) if len(arr) else torch.zeros((1, 2), dtype=torch.int64, device=dev)
    cnt = torch.tensor([len(arr)], dtype=torch.int64, device=dev)
    out, ln = encode_index_device(t, cnt)
    return bytes(out[: int(ln.item())].cpu().numpy().tobytes())


def decode_index(data: bytes) -> list:
    def varint(pos):
        v = shift = 0
        while True:
            b = data[pos]
            pos += 1
            v |= (b & 0x7F) << shift
            if not b & 0x80:
                return v, pos
            shift += 7

    count, pos = varint(0)
    out, slot, probe = [], 0, 0
    for _ in range(count):
        ds, pos = varint(pos)
        dz, pos = varint(pos)
        slot += ds
        probe += (dz >> 1) ^ -(dz & 1)
        out.append((slot, probe))
    if pos != len(data):
        raise ValueError("trailing bytes in index buffer")
    return out
