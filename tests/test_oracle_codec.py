"""Pin the encoder restatement against the reference's encode_frame bytes."""

import numpy as np

from oracle import codec_ops as co


def test_entropy_kats(golden):
    g = golden("codec")
    for i in range(int(g["nent"])):
        assert co.entropy_encode(g[f"ent{i}_in"].tobytes()) == g[f"ent{i}_out"].tobytes(), i


def test_frames_match_reference_bytes(golden):
    g = golden("codec")
    for s in range(int(g["nseq"])):
        gop = int(g[f"s{s}_gop"])
        ref = None
        for f in range(int(g[f"s{s}_frames"])):
            planes = g[f"s{s}_f{f}_planes"]
            key = bool(g[f"s{s}_f{f}_key"])
            assert key == (ref is None or f % gop == 0 or f == 5)
            got = co.frame_bytes(planes, ref, int(g[f"s{s}_stream"]), f, key)
            assert got == g[f"s{s}_f{f}_bytes"].tobytes(), (s, f)
            ref = planes
