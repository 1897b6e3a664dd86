"""§8(f) row 1: the GPU LPF1 encoder produces the reference encode_frame's
bytes exactly (golden streams made by the reference), including the CRC."""

import zlib

import numpy as np
import pytest
import torch

from oracle import codec_ops as co

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def codec():
    from paper_2103_05875_b200 import build_native

    build_native.build()
    from paper_2103_05875_b200 import codec, packing

    return codec, packing


def test_golden_streams_bit_exact(codec, golden):
    cdc, packing = codec
    g = golden("codec")
    for s in range(int(g["nseq"])):
        state = cdc.CodecStreamState(int(g[f"s{s}_stream"]), gop_length=int(g[f"s{s}_gop"]))
        for f in range(int(g[f"s{s}_frames"])):
            planes = g[f"s{s}_f{f}_planes"]
            kind = (packing.PlaneKind.COLOR_10IN16 if planes.dtype == np.uint16
                    else packing.PlaneKind.VISIBILITY_BYTES)
            frame = cdc.encode_frame(packing.PlaneSet(kind, planes), state, force_key=(f == 5))
            wire = frame.to_bytes()
            assert wire == g[f"s{s}_f{f}_bytes"].tobytes(), (s, f)
            assert frame.key == bool(g[f"s{s}_f{f}_key"])


@pytest.mark.parametrize("dtype,shape", [(np.uint16, (3, 100, 130)), (np.uint8, (3, 77, 200)),
                                         (np.uint8, (3, 1, 1)), (np.uint16, (3, 16, 33))])
def test_random_sequences_vs_oracle(codec, dtype, shape):
    cdc, packing = codec
    rng = np.random.default_rng(shape[1] * 7 + shape[2])
    hi = 1024 if dtype == np.uint16 else 256
    kind = packing.PlaneKind.COLOR_10IN16 if dtype == np.uint16 else packing.PlaneKind.VISIBILITY_BYTES
    cur = rng.integers(0, hi, size=shape, dtype=dtype)
    cur[:, : shape[1] // 3] = 0
    state = cdc.CodecStreamState(9, gop_length=3)
    ref = None
    for f in range(5):
        if f:
            m = rng.random(shape) < 0.05
            cur = cur.copy()
            cur[m] = rng.integers(0, hi, size=int(m.sum()), dtype=dtype)
        key = ref is None or f % 3 == 0
        want = co.frame_bytes(cur, ref, 9, f, key)
        got = cdc.encode_frame(packing.PlaneSet(kind, torch.from_numpy(cur).cuda()), state).to_bytes()
        assert got == want, f
        ref = cur


def test_large_frame_crc_and_length(codec):
    """A C2-sized visibility update atlas (3 x 2048 x 2731): CRC over
    megabytes is combined from 4 KB chunks; checked against zlib."""
    cdc, packing = codec
    rng = np.random.default_rng(3)
    planes = rng.integers(0, 256, size=(3, 2048, 2731), dtype=np.uint8)
    planes[:, :1000] = 0
    t = torch.from_numpy(planes).cuda()
    out, ln = cdc.encode_frame_device(t, None, 5, 0)
    wire = out[: int(ln.item())].cpu().numpy().tobytes()
    body, crc = wire[:-4], int.from_bytes(wire[-4:], "little")
    assert crc == zlib.crc32(body)
    assert len(body) - 23 == int.from_bytes(wire[19:23], "little")
    # P-frame with one changed element: all SKIP but one block
    p2 = planes.copy()
    p2[1, 5, 7] ^= 1
    out2, ln2 = cdc.encode_frame_device(torch.from_numpy(p2).cuda(), t, 5, 1)
    w2 = out2[: int(ln2.item())].cpu().numpy().tobytes()
    nblocks = 3 * 128 * 171
    assert len(w2) < 23 + 4 + nblocks + 600
    assert w2 == co.frame_bytes(p2, planes, 5, 1, False)
