"""The thread-per-block LPF1 passes (csrc/ps_codec.cu) replace the warp-wide
zero-run encoder with two byte-serial state machines: ``Sizer`` (entropy
size from the zero-run structure alone, vlen(2L[+1]) = 1 + (L >= 64)) and
``Emitter`` (tokens with one-byte literal headers widened in place when a
literal reaches 64 bytes).  These are line-for-line Python mirrors of the two
device structs, checked against the oracle's restatement of the reference
entropy coder (codec.py:76-103) on random and adversarial block streams."""

import numpy as np
import pytest

from oracle import codec_ops as co


class Sizer:  # mirrors ps_codec.cu: struct Sizer
    def __init__(self):
        self.run = self.lit = self.size = 0

    def push(self, byte):
        if byte == 0:
            self.run += 1
            return
        if self.run >= 2:
            if self.lit:
                self.size += 1 + (self.lit >= 64) + self.lit
            self.size += 1 + (self.run >= 64)
            self.lit = 0
        else:
            self.lit += self.run
        self.lit += 1
        self.run = 0

    def finish(self):
        if self.run >= 2:
            if self.lit:
                self.size += 1 + (self.lit >= 64) + self.lit
            self.size += 1 + (self.run >= 64)
        elif self.lit + self.run:
            L = self.lit + self.run
            self.size += 1 + (L >= 64) + L
        return self.size


class Emitter:  # mirrors ps_codec.cu: struct Emitter
    def __init__(self):
        self.o = bytearray(1024)
        self.pos = self.run = self.lit = self.hdr = 0

    def lit_byte(self, v):
        if self.lit == 0:
            self.hdr = self.pos
            self.pos += 1
        self.o[self.pos] = v
        self.pos += 1
        self.lit += 1

    def close_lit(self):
        if not self.lit:
            return
        if self.lit >= 64:
            self.o[self.hdr + 2:self.pos + 1] = self.o[self.hdr + 1:self.pos]
            self.pos += 1
            self.o[self.hdr:self.hdr + 2] = co.uvarint(self.lit << 1)
        else:
            self.o[self.hdr] = self.lit << 1
        self.lit = 0

    def close_run(self):
        self.close_lit()
        v = co.uvarint((self.run << 1) | 1)
        self.o[self.pos:self.pos + len(v)] = v
        self.pos += len(v)

    def push(self, byte):
        if byte == 0:
            self.run += 1
            return
        if self.run >= 2:
            self.close_run()
        elif self.run == 1:
            self.lit_byte(0)
        self.lit_byte(byte)
        self.run = 0

    def finish(self):
        if self.run >= 2:
            self.close_run()
        elif self.run == 1:
            self.lit_byte(0)
        self.close_lit()
        return bytes(self.o[:self.pos])


def _streams():
    rng = np.random.default_rng(3)
    yield b""
    yield b"\x00"
    yield b"\x00\x00"
    yield b"\x07"
    yield b"\x00\x07\x00"
    yield bytes(768)
    yield bytes([1]) * 768
    yield bytes([0, 5] * 384)
    yield bytes([0, 0, 5] * 256)
    yield bytes([5] * 63 + [0, 0] + [5] * 64 + [0] + [5] * 200)
    for n in (16, 63, 64, 65, 127, 128, 256, 512, 768):
        for p0 in (0.0, 0.3, 0.6, 0.9, 1.0):
            yield bytes(np.where(rng.random(n) < p0, 0, rng.integers(1, 256, n)).astype(np.uint8))


@pytest.mark.parametrize("data", list(_streams()))
def test_sizer_and_emitter_match_reference_entropy(data):
    want = co.entropy_encode(data)
    s, e = Sizer(), Emitter()
    for b in data:
        s.push(b)
        e.push(b)
    assert s.finish() == len(want)
    assert e.finish() == want


def test_varint_streams_of_residual_blocks():
    """Residual varint streams (the DELTA mode input) of random 16x16 blocks."""
    rng = np.random.default_rng(5)
    for dt in (np.uint16, np.uint8):
        hi = 1024 if dt == np.uint16 else 256
        for _ in range(20):
            cur = rng.integers(0, hi, (16, 16)).astype(dt)
            pred = cur.copy()
            m = rng.random((16, 16)) < 0.2
            pred[m] = rng.integers(0, hi, int(m.sum())).astype(dt)
            data = co.residual_stream(cur, pred)
            s = Sizer()
            for b in data:
                s.push(b)
            assert s.finish() == len(co.entropy_encode(data))
