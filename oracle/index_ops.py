"""Restatement of the probe index buffer (§8(f)4).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__``).  The reference ships no
``encode_index_buffer`` (the server module is absent); the spec
fixes the format on top of the reference's varint primitives, which are
restated here and pinned against the reference's own outputs
(tests/golden/index.npz, made by tests/golden/make_golden.py from
``probestream.varint``):

* ``zigzag``          varint.py:16-19  ((v << 1) ^ (v >> 63))
* ``encode_uvarint``  varint.py:27-38  (LEB128: 7 bits per byte, LSB group
                                         first, bit 7 = continuation)
* index buffer        SPEC.md:355-362: uvarint(count), then per entry
                      uvarint(slot - previous slot), uvarint(zigzag(probe -
                      previous probe)), both previous values starting at 0;
                      entries strictly increasing in slot.
"""

from __future__ import annotations


def zigzag(v: int) -> int:
    """varint.py:16-19 for one int64 value."""
    v = int(v)
    return ((v << 1) ^ (v >> 63)) & 0xFFFFFFFFFFFFFFFF


def encode_uvarint(value: int) -> bytes:
    """varint.py:27-38."""
    if value < 0:
        raise ValueError("varint values must be non-negative")
    out = bytearray()
    while True:
        bits = value & 0x7F
        value >>= 7
        if value:
            out.append(0x80 | bits)
        else:
            out.append(bits)
            return bytes(out)


def encode_index_buffer(entries) -> bytes:
    entries = [(int(s), int(p)) for s, p in entries]
    for (s0, _), (s1, _) in zip(entries, entries[1:]):
        if s1 <= s0:
            raise ValueError("index entries must be strictly increasing in slot")
    out = bytearray(encode_uvarint(len(entries)))
    ps = pp = 0
    for slot, probe in entries:
        out += encode_uvarint(slot - ps)
        out += encode_uvarint(zigzag(probe - pp))
        ps, pp = slot, probe
    return bytes(out)


def size_bound(count: int) -> int:
    """SPEC.md:358's ``2 bytes x count + 5``; it holds whenever every slot
    delta is < 128 and every probe delta is in [-64, 63] (one byte each), e.g.
    consecutive slots of a coherent probe run.  Larger deltas need more
    LEB128 bytes whatever the encoder (a probe jump of 2^20 needs 3)."""
    return 2 * count + 5
