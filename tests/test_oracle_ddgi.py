"""Pin the stage (1)+(2) oracle pieces against the reference's golden vectors
(fibonacci sphere, texel directions, triangle raycast), and check that the
product's host-side tables (ray set, texel directions) agree with the oracle.
CPU only."""

import numpy as np
import pytest

from oracle import ddgi


def test_fibonacci_matches_reference(golden):
    g = golden("geometry")
    assert np.array_equal(ddgi.fibonacci_sphere(64), g["fib64"])
    assert np.array_equal(ddgi.fibonacci_sphere(256), g["fib256"])


def test_texel_directions_match_reference(golden):
    g = golden("geometry")
    np.testing.assert_allclose(ddgi.texel_directions(8).reshape(8, 8, 3), g["texdir8"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(ddgi.texel_directions(16).reshape(16, 16, 3), g["texdir16"], rtol=0, atol=1e-15)


def test_raycast_matches_reference_exactly(golden):
    g = golden("geometry")
    t, prim = ddgi.raycast(g["tris"], g["ray_o"], g["ray_d"])
    hit = prim >= 0
    assert np.array_equal(hit, g["hit"])
    assert np.array_equal(t[hit], g["t"][hit])  # bit-exact float64
    assert np.all(np.isinf(t[~hit]))
    v = g["tris"]
    n = np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0])
    n = n / np.maximum(np.linalg.norm(n, axis=1, keepdims=True), 1e-30)
    nn = n[prim[hit]]
    flip = np.sum(nn * g["ray_d"][hit], axis=1) > 0
    nn[flip] *= -1
    assert np.array_equal(nn, g["normal"][hit])


def test_occluded_consistent_with_raycast(golden):
    g = golden("geometry")
    t, prim = ddgi.raycast(g["tris"], g["ray_o"], g["ray_d"])
    tmax = np.where(np.isfinite(t), t * 1.0001, 10.0)
    assert np.array_equal(ddgi.occluded(g["tris"], g["ray_o"], g["ray_d"], tmax), prim >= 0)
    tmax = np.where(np.isfinite(t), t * 0.9999, 10.0)
    assert not ddgi.occluded(g["tris"], g["ray_o"], g["ray_d"], tmax)[prim >= 0].any()


@pytest.mark.parametrize("count", [64, 256])
def test_product_ray_table_matches_oracle(count):
    from paper_2103_05875_b200 import probes

    for frame in (0, 1, 17):
        a = probes.frame_ray_directions(count, 3, frame)[:, :3]
        b = ddgi.ray_table(count, 3, frame)
        np.testing.assert_allclose(a, b, rtol=0, atol=2e-7)
        np.testing.assert_allclose(np.linalg.norm(a.astype(np.float64), axis=1), 1.0, atol=1e-6)
    # same base set as the reference fibonacci sphere, only reordered
    base = probes.base_ray_set(count)
    ref = ddgi.fibonacci_sphere(count)
    assert np.array_equal(np.sort(base.view("f8,f8,f8"), axis=0), np.sort(ref.view("f8,f8,f8"), axis=0))


def test_product_texel_table_matches_oracle():
    from paper_2103_05875_b200 import probes

    tab = probes.texel_direction_table()
    assert np.array_equal(tab[:64, :3], ddgi.texel_directions(8).astype(np.float32))
    assert np.array_equal(tab[64:, :3], ddgi.texel_directions(16).astype(np.float32))


def test_quantize_is_round_half_even():
    irr = np.zeros((1, 64, 3), np.float32)
    irr[0, 0] = [0.5 / 1023, 1.5 / 1023, 2.0]  # ties and saturation
    q = ddgi.quantize_color(irr, 1.0)
    r, g, b = q[0, 0, 0] & 1023, (q[0, 0, 0] >> 10) & 1023, q[0, 0, 0] >> 20
    assert (r, g, b) == (np.rint(np.float32(0.5 / 1023) * np.float32(1023)), 2, 1023)
