"""§8(f) row 4: probe index buffer built on the GPU."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_index_buffer_round_trip_and_bounds():
    from paper_2103_05875_b200.index_buffer import decode_index, encode_index_buffer

    assert encode_index_buffer([]) == b"\x00"  # empty list -> 1 byte
    e = [(0, 5), (1, 9)]
    blob = encode_index_buffer(e)
    assert len(blob) <= 9 and decode_index(blob) == e
    consecutive = [(i, 1000 + i) for i in range(400)]
    blob = encode_index_buffer(consecutive)
    assert len(blob) < 1024 and decode_index(blob) == consecutive  # "<1 kB" (PAPER §3.4)
    rng = np.random.default_rng(2)
    for n in (1, 17, 4096):
        slots = np.sort(rng.choice(10 * n, size=n, replace=False))
        probes = rng.integers(0, 131072, size=n)
        ent = list(zip(slots.tolist(), probes.tolist()))
        blob = encode_index_buffer(ent)
        assert decode_index(blob) == ent
    with pytest.raises(ValueError):
        encode_index_buffer([(2, 1), (1, 3)])
