"""Restatement of the reference's lossless frame encoder (codec.py, varint.py).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__``); pinned against byte
streams produced by the reference's own ``encode_frame``
(tests/golden/codec.npz).

* entropy coder: zero-run-length tokens with LEB128 headers
  (codec.py:76-103): a maximal zero run of >= 2 bytes becomes
  ``uvarint(len << 1 | 1)``; everything else goes out as literal segments
  ``uvarint(len << 1)`` + bytes;
* residual stream: ``(cur - pred)`` in the plane dtype viewed signed,
  zig-zag, LEB128 (codec.py:211-215, varint.py:16-84);
* block modes SKIP / DELTA / RAW with DELTA only if strictly shorter
  (codec.py:239-292), 16x16 blocks with clipped edges (codec.py:250-257),
  left-neighbour intra prediction in key frames (codec.py:275-277);
* LPF1 container: ``<4sBIIHHBBI`` header, payload, CRC32 (codec.py:147-183).
"""

from __future__ import annotations

import struct
import zlib

import numpy as np

BLOCK = 16
SKIP, DELTA, RAW = 0, 1, 2
HEADER = struct.Struct("<4sBIIHHBBI")


def uvarint(v: int) -> bytes:
    out = bytearray()
    while True:
        b = v & 0x7F
        v >>= 7
        if v:
            out.append(b | 0x80)
        else:
            out.append(b)
            return bytes(out)


def entropy_encode(data: bytes) -> bytes:
    n = len(data)
    out = bytearray()
    lit_start = 0
    i = 0
    while i < n:
        if data[i] == 0:
            j = i
            while j < n and data[j] == 0:
                j += 1
            if j - i >= 2:
                if i > lit_start:
                    out += uvarint((i - lit_start) << 1)
                    out += data[lit_start:i]
                out += uvarint(((j - i) << 1) | 1)
                lit_start = j
            i = j
        else:
            i += 1
    if lit_start < n:
        out += uvarint((n - lit_start) << 1)
        out += data[lit_start:]
    return bytes(out)


def residual_stream(cur: np.ndarray, pred: np.ndarray) -> bytes:
    signed = np.int16 if cur.dtype == np.uint16 else np.int8
    r = (cur - pred).astype(cur.dtype).view(signed).astype(np.int64).reshape(-1)
    z = ((r << 1) ^ (r >> 63)).astype(np.uint64)
    return b"".join(uvarint(int(v)) for v in z)


def encode_block(cur: np.ndarray, pred) -> bytes:
    raw = entropy_encode(np.ascontiguousarray(cur).view(np.uint8).tobytes())
    if pred is not None:
        delta = entropy_encode(residual_stream(cur, pred))
        if len(delta) < len(raw):
            return bytes([DELTA]) + uvarint(len(delta)) + delta
    return bytes([RAW]) + uvarint(len(raw)) + raw


def encode_payload(planes: np.ndarray, ref) -> bytes:
    out = bytearray()
    _, h, w = planes.shape
    for p in range(planes.shape[0]):
        cur = planes[p]
        for y0 in range(0, h, BLOCK):
            for x0 in range(0, w, BLOCK):
                blk = cur[y0:y0 + BLOCK, x0:x0 + BLOCK]
                bh, bw = blk.shape
                if ref is not None:
                    rb = ref[p][y0:y0 + bh, x0:x0 + bw]
                    if np.array_equal(blk, rb):
                        out.append(SKIP)
                        continue
                    out += encode_block(blk, rb)
                elif x0 >= BLOCK:
                    out += encode_block(blk, cur[y0:y0 + bh, x0 - BLOCK:x0 - BLOCK + bw])
                else:
                    out += encode_block(blk, None)
    return bytes(out)


def frame_bytes(planes: np.ndarray, ref, stream_id: int, seq: int, key: bool) -> bytes:
    payload = encode_payload(planes, None if key else ref)
    _, h, w = planes.shape
    bits = 16 if planes.dtype == np.uint16 else 8
    body = HEADER.pack(b"LPF1", 1 if key else 0, stream_id, seq, w, h, planes.shape[0], bits,
                       len(payload)) + payload
    return body + struct.pack("<I", zlib.crc32(body))
