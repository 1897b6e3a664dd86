"""The index-buffer oracle (§8(f)4) pinned against the reference's varint
primitives (tests/golden/index.npz, generated from probestream.varint)."""

import numpy as np
import pytest

from oracle import index_ops


def test_varint_primitives_match_reference(golden):
    g = golden("index")
    assert [index_ops.zigzag(v) for v in g["zz_in"]] == [int(v) for v in g["zz_out"]]
    blob = b"".join(index_ops.encode_uvarint(int(v)) for v in g["uv_in"])
    assert blob == g["uv_out"].tobytes()
    assert [len(index_ops.encode_uvarint(int(v))) for v in g["uv_in"]] == list(g["uv_lens"])


def test_index_buffer_matches_reference_composition(golden):
    g = golden("index")
    for i in range(int(g["n"])):
        e = [tuple(r) for r in g[f"e{i}"].tolist()]
        assert index_ops.encode_index_buffer(e) == g[f"b{i}"].tobytes(), i


def test_spec_examples_and_bound():
    assert index_ops.encode_index_buffer([]) == b"\x00"                      # empty -> 1 byte
    assert len(index_ops.encode_index_buffer([(0, 5), (1, 9)])) <= 9
    run = [(i, 1000 + i) for i in range(400)]
    assert len(index_ops.encode_index_buffer(run)) < 1024                     # "<1 kB"
    rng = np.random.default_rng(3)
    for n in (1, 100, 10_000):
        probes = 50_000 + np.cumsum(rng.integers(-64, 64, size=n))           # deltas in [-64, 63]
        slots = np.cumsum(rng.integers(1, 128, size=n)) - 1                  # deltas in [1, 127]
        e = list(zip(slots.tolist(), probes.tolist()))
        assert len(index_ops.encode_index_buffer(e)) <= index_ops.size_bound(n)
    with pytest.raises(ValueError):
        index_ops.encode_index_buffer([(2, 1), (1, 3)])
