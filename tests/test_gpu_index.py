"""§8(f) row 4: probe index buffer built on the GPU, byte
for byte against the oracle (oracle/index_ops.py), which is pinned against
the reference's varint / zig-zag primitives (tests/golden/index.npz)."""

import numpy as np
import pytest

from oracle import index_ops

pytestmark = pytest.mark.gpu


def test_index_buffer_bytes_match_oracle_and_golden(golden):
    from paper_2103_05875_b200.index_buffer import decode_index, encode_index_buffer

    g = golden("index")
    for i in range(int(g["n"])):
        e = [tuple(r) for r in g[f"e{i}"].tolist()]
        blob = encode_index_buffer(e)
        assert blob == g[f"b{i}"].tobytes(), i
        assert blob == index_ops.encode_index_buffer(e)
        assert decode_index(blob) == e
    rng = np.random.default_rng(2)
    for n in (1, 17, 4096, 131072):
        slots = np.sort(rng.choice(10 * n, size=n, replace=False))
        probes = rng.integers(0, 131072, size=n)
        ent = list(zip(slots.tolist(), probes.tolist()))
        assert encode_index_buffer(ent) == index_ops.encode_index_buffer(ent)
    with pytest.raises(ValueError):
        encode_index_buffer([(2, 1), (1, 3)])


def test_index_buffer_spec_bound():
    """size <= 2 B x count + 5 for coherent entries (slot deltas
    < 128, probe deltas in [-64, 63]); the spec's examples."""
    from paper_2103_05875_b200.index_buffer import encode_index_buffer

    assert encode_index_buffer([]) == b"\x00"
    assert len(encode_index_buffer([(0, 5), (1, 9)])) <= 9
    assert len(encode_index_buffer([(i, 1000 + i) for i in range(400)])) < 1024
    rng = np.random.default_rng(9)
    for n in (1, 1000, 131072):
        probes = 65_000 + np.cumsum(rng.integers(-64, 64, size=n))
        slots = np.cumsum(rng.integers(1, 128, size=n)) - 1
        blob = encode_index_buffer(list(zip(slots.tolist(), probes.tolist())))
        assert len(blob) <= index_ops.size_bound(n)
