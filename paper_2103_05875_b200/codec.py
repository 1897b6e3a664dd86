"""Lossless LPF1 frame encoding on the GPU (§8(f) row 1).

Drop-in for ``probestream.codec.encode_frame`` (codec.py:335-366): the same
stream state, key-frame rule (first frame, ``frame_count % gop_length == 0``
or forced, codec.py:348), block modes and byte stream -- produced by
``csrc/ps_codec.cu`` and bit-identical to the reference's bytes
(tests/test_gpu_codec.py against reference-made golden frames).

``encode_frame_device`` keeps planes, reference and the encoded frame on the
device (the paper hands only compressed bitstreams to the host).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .packing import PlaneKind, PlaneSet

BLOCK_SIDE = 16
MIN_ZERO_RUN = 2
MODE_SKIP, MODE_DELTA, MODE_RAW = 0, 1, 2
FRAME_MAGIC = b"LPF1"
DEFAULT_GOP_LENGTH = 30
_HEADER = struct.Struct("<4sBIIHHBBI")
_CHECKSUM = struct.Struct("<I")


class CodecError(Exception):
    pass


class CorruptFrameError(CodecError):
    pass


class MissingReferenceError(CodecError):
    pass


class SequenceError(CodecError):
    pass


class DimensionMismatchError(CodecError):
    pass


class EntropyDecodeError(CodecError):
    pass


@dataclass
class CodecStreamState:
    """codec.py:130-144; ``reference`` holds the previous planes (on the device
    when the planes were CUDA tensors)."""

    stream_id: int
    role: str = "encoder"
    gop_length: int = DEFAULT_GOP_LENGTH
    frame_count: int = 0
    reference: PlaneSet | None = field(default=None, repr=False)

    def __post_init__(self) -> None:
        if self.role not in ("encoder", "decoder"):
            raise ValueError(f"role must be encoder or decoder, got {self.role!r}")
        if self.gop_length < 1:
            raise ValueError("GOP length must be >= 1")


@dataclass
class EncodedFrame:
    stream_id: int
    frame_seq: int
    key: bool
    width: int
    height: int
    plane_count: int
    element_bits: int
    payload: bytes

    @property
    def plane_kind(self) -> PlaneKind:
        return PlaneKind.COLOR_10IN16 if self.element_bits == 16 else PlaneKind.VISIBILITY_BYTES

    @property
    def raw_bytes(self) -> int:
        return self.plane_count * self.width * self.height * (self.element_bits // 8)

    @property
    def encoded_size(self) -> int:
        return _HEADER.size + len(self.payload) + _CHECKSUM.size

    def to_bytes(self) -> bytes:
        if getattr(self, "_wire", None) is not None:
            return self._wire
        import zlib

        body = _HEADER.pack(FRAME_MAGIC, 1 if self.key else 0, self.stream_id, self.frame_seq,
                            self.width, self.height, self.plane_count, self.element_bits,
                            len(self.payload)) + self.payload
        return body + _CHECKSUM.pack(zlib.crc32(body))

    @classmethod
    def from_device_bytes(cls, wire: bytes) -> "EncodedFrame":
        magic, flags, sid, seq, w, h, planes, bits, plen = _HEADER.unpack_from(wire, 0)
        if magic != FRAME_MAGIC:
            raise CodecError("bad frame magic from the device encoder")
        f = cls(sid, seq, bool(flags & 1), w, h, planes, bits,
                wire[_HEADER.size:_HEADER.size + plen])
        f._wire = wire  # header + payload + device CRC32
        return f


class _Buffers:
    cache: dict = {}

    @classmethod
    def get(cls, h, w, eb, device, owner=None):
        key = (h, w, eb, str(device), owner)
        b = cls.cache.get(key)
        if b is None:
            cap = N.lib().ps_encode_frame_capacity(h, w, eb)
            out = torch.empty(cap, dtype=torch.uint8, device=device)
            ln = torch.zeros(1, dtype=torch.int64, device=device)
            ws = torch.empty(N.lib().ps_encode_workspace_bytes(h, w, eb), dtype=torch.uint8,
                             device=device)
            b = cls.cache[key] = (out, ln, ws)
        return b


def encode_frame_device(planes: torch.Tensor, reference: torch.Tensor | None, stream_id: int,
                        frame_seq: int, out=None, frame_len=None, workspace=None):
    """Encode one frame on the device; returns (frame buffer uint8, length
    int64[1]) -- the first ``length`` bytes are the LPF1 wire frame.  A
    session passes its own ``out`` / ``frame_len`` / ``workspace``
    (server.KindStream does); otherwise buffers come from a cache keyed by
    (shape, stream id) for one-off calls on the current stream."""
    if planes.dim() != 3 or planes.shape[0] != 3:
        raise ValueError("plane data must be (3, h, w)")
    eb = planes.element_size()
    _, h, w = planes.shape
    dev = planes.device
    if out is None or frame_len is None or workspace is None:
        o, ln, ws = _Buffers.get(h, w, eb, dev, int(stream_id))
    out = o if out is None else out
    frame_len = ln if frame_len is None else frame_len
    ws = ws if workspace is None else D.Workspace.get(
        N.lib().ps_encode_workspace_bytes(h, w, eb), dev, workspace)
    ref = reference.contiguous() if reference is not None else None
    N.call("ps_encode_frame", eb, planes.contiguous().data_ptr(), D.ptr(ref), h, w,
           int(stream_id) & 0xFFFFFFFF, int(frame_seq) & 0xFFFFFFFF, out.data_ptr(), out.numel(),
           frame_len.data_ptr(), ws.data_ptr(), ws.numel(), D.stream_ptr(dev))
    return out, frame_len


def encode_frame(planes: PlaneSet, state: CodecStreamState, force_key: bool = False) -> EncodedFrame:
    """Encode one frame and advance the stream state (closed loop, lossless)."""
    if state.role != "encoder":
        raise CodecError("encode_frame requires an encoder stream state")
    if state.reference is not None and (
            tuple(state.reference.data.shape) != tuple(planes.data.shape)
            or state.reference.kind != planes.kind):
        raise DimensionMismatchError(
            f"frame {tuple(planes.data.shape)} does not match stream "
            f"{tuple(state.reference.data.shape)}")
    key = force_key or state.reference is None or state.frame_count % state.gop_length == 0
    data = planes.data
    tdt = planes.kind.torch_dtype
    cur = data if D.is_tensor(data) else torch.from_numpy(np.ascontiguousarray(data)).to(D.device_of())
    ref = None
    if not key:
        rd = state.reference.data
        ref = rd if D.is_tensor(rd) else torch.from_numpy(np.ascontiguousarray(rd)).to(cur.device)
    out, ln = encode_frame_device(cur.view(tdt) if cur.dtype != tdt else cur, ref,
                                  state.stream_id, state.frame_count)
    n = int(ln.item())
    wire = bytes(out[:n].cpu().numpy().tobytes())
    seq = state.frame_count
    state.frame_count = seq + 1
    state.reference = PlaneSet(planes.kind, cur.clone())
    frame = EncodedFrame.from_device_bytes(wire)
    assert frame.frame_seq == seq
    return frame


def compression_ratio(planes: PlaneSet, frame: EncodedFrame) -> float:
    nbytes = planes.data.numel() * planes.data.element_size() if D.is_tensor(planes.data) \
        else planes.data.nbytes
    return nbytes / frame.encoded_size


# --- client side: decode (codec.py:369-395) ------------------------------------------


def decode_frame_device(frame: torch.Tensor, payload_len: int, reference: torch.Tensor | None,
                        h: int, w: int, elem_bytes: int, out: torch.Tensor | None = None):
    """Decode a frame whose bytes are on the device; returns (planes, status)
    where status is an int32[1] device word (0 = ok, 1 corrupt, 2 entropy)."""
    dev = frame.device
    tdt = torch.uint16 if elem_bytes == 2 else torch.uint8
    if out is None:
        out = torch.empty((3, h, w), dtype=tdt, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = torch.empty(N.lib().ps_decode_workspace_bytes(h, w), dtype=torch.uint8, device=dev)
    ref = reference.contiguous() if reference is not None else None
    N.call("ps_decode_frame", elem_bytes, frame.data_ptr(), int(payload_len), D.ptr(ref), h, w,
           out.data_ptr(), status.data_ptr(), ws.data_ptr(), ws.numel(), D.stream_ptr(dev))
    return out, status


def decode_frame(frame: EncodedFrame, state: CodecStreamState) -> PlaneSet:
    """Decode one frame, verify sequencing, advance the stream state."""
    if state.role != "decoder":
        raise CodecError("decode_frame requires a decoder stream state")
    if not frame.key:
        if state.reference is None:
            raise MissingReferenceError(f"P-frame seq {frame.frame_seq} with no prior state")
        if frame.frame_seq != state.frame_count:
            raise SequenceError(f"frame seq {frame.frame_seq}, decoder expected {state.frame_count}")
        if tuple(state.reference.data.shape[1:]) != (frame.height, frame.width):
            raise DimensionMismatchError("frame dims do not match stream state")
    eb = frame.element_bits // 8
    dev = D.device_of()
    wire = np.frombuffer(frame.to_bytes(), np.uint8)
    buf = torch.from_numpy(wire.copy()).to(dev)
    ref = None
    if not frame.key:
        rd = state.reference.data
        ref = rd if D.is_tensor(rd) else torch.from_numpy(np.ascontiguousarray(rd)).to(dev)
    planes, status = decode_frame_device(buf, len(frame.payload), ref, frame.height, frame.width, eb)
    st = int(status.item())
    if st & 1:
        raise CorruptFrameError("malformed frame payload")
    if st & 2:
        raise EntropyDecodeError("malformed entropy-coded block")
    kind = frame.plane_kind
    result = PlaneSet(kind, planes)
    state.reference = PlaneSet(kind, planes.clone())
    state.frame_count = frame.frame_seq + 1
    return result
