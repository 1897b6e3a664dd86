"""Temporal delta against the previous streamed frame (stage 4 tail).

Restates the codec's temporal prediction (codec.py:207-215 residual,
:250-272 SKIP rule, :348 key-frame rule) as an encoder-ready output instead
of an entropy-coded bitstream:

* ``residual = (cur - prev) mod 2^bits`` in the plane dtype (the codec views
  it as int16 / int8 before zig-zag, codec.py:212);
* ``skip[p, by, bx] = 1`` iff the clipped 16x16 block of plane ``p`` is
  bit-identical to the reference block (codec.py:264-272);
* ``prev is None`` is a key frame: no temporal reference, nothing is SKIP.

``pack_delta`` fuses plane packing with the delta in one pass over the
update atlas (the pipeline's K6).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .packing import PlaneKind, PlaneSet, widened_width
from .volume import AtlasKind, kind_of

BLOCK_SIDE = 16  # codec.py:35


def skip_shape(h: int, w: int) -> tuple:
    return (3, -(-h // BLOCK_SIDE), -(-w // BLOCK_SIDE))


def temporal_delta(cur: PlaneSet, prev: PlaneSet | None):
    """Returns (residual, skip) as numpy when ``cur`` is numpy, else tensors."""
    if prev is not None and (prev.kind != cur.kind or tuple(prev.data.shape) != tuple(cur.data.shape)):
        raise ValueError("reference frame does not match the current frame")
    was_np = not D.is_tensor(cur.data)
    dev = D.device_of(cur.data, prev.data if prev is not None else None)
    tdt = cur.kind.torch_dtype
    c = D.to_device(cur.data, tdt, dev) if was_np else cur.data.contiguous()
    p = None
    if prev is not None:
        p = D.to_device(prev.data, tdt, dev) if not D.is_tensor(prev.data) else prev.data.contiguous()
    _, h, w = c.shape
    residual = torch.zeros_like(c)
    skip = torch.zeros(skip_shape(h, w), dtype=torch.uint8, device=dev)
    eb = 2 if cur.kind is PlaneKind.COLOR_10IN16 else 1
    N.call("ps_temporal_delta", eb, c.data_ptr(), D.ptr(p), h, w, residual.data_ptr(),
           skip.data_ptr(), D.stream_ptr(dev))
    if was_np:
        return D.to_numpy(residual), D.to_numpy(skip)
    return residual, skip


def pack_delta(texels: torch.Tensor, kind, planes_prev: torch.Tensor | None, *,
               planes_out: torch.Tensor | None = None, residual: torch.Tensor | None = None,
               skip: torch.Tensor | None = None, key_dev: torch.Tensor | None = None):
    """Pack a (contiguous) update atlas and diff it against the previous planes
    in one kernel.  Returns (planes, residual, skip) CUDA tensors."""
    k = kind_of(kind)
    dev = texels.device
    if k is AtlasKind.COLOR:
        h, w = texels.shape
        pshape, pdt = (3, h, w), torch.uint16
    else:
        h, w, _ = texels.shape
        pshape, pdt = (3, h, widened_width(w)), torch.uint8
    if planes_out is None:
        planes_out = torch.empty(pshape, dtype=pdt, device=dev)
    if residual is None:
        residual = torch.empty(pshape, dtype=pdt, device=dev)
    if skip is None:
        skip = torch.empty(skip_shape(pshape[1], pshape[2]), dtype=torch.uint8, device=dev)
    N.call("ps_pack_delta", k.native, texels.data_ptr(), h, w, w, planes_out.data_ptr(),
           D.ptr(planes_prev), residual.data_ptr(), skip.data_ptr(), D.ptr(key_dev),
           D.stream_ptr(dev))
    return planes_out, residual, skip
