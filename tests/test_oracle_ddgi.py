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


@pytest.mark.parametrize("rays,h", [(64, 0.0), (256, 0.97)])
def test_oracle_blend_is_fp32_accurate(rays, h):
    """The float32 oracle blend (float64 ray sums rounded once, float32
    normalisation and hysteresis) equals an all-float64 blend of the same
    float32 inputs to 1e-6 relative: the oracle is an honest fp32 DDGI
    blend, with plain (not tf32-rounded) float32 weights."""
    rng = np.random.default_rng(rays)
    dirs = ddgi.ray_table(rays, 5, 1).astype(np.float32)
    w = ddgi.blend_weights(dirs, 50.0)
    # weights are plain float32: the low 13 mantissa bits are not all zero
    assert np.any(w[0].view(np.uint32) & np.uint32(0x1FFF))
    assert np.any(w[1].view(np.uint32) & np.uint32(0x1FFF))
    P = 24
    rgb = rng.gamma(2.0, 0.3, size=(P, rays, 3)).astype(np.float32)
    rgb[:, ::7] = 0.0  # sky-less misses / unlit hits
    dep = rng.uniform(0.05, 12.0, size=(P, rays)).astype(np.float32)
    prev_i = rng.uniform(0, 2, size=(P, 64, 3)).astype(np.float32) if h else None
    prev_m = rng.uniform(0, 20, size=(P, 256, 2)).astype(np.float32) if h else None
    irr, mom = ddgi.blend(rgb, dep, w, prev_i, prev_m, h)
    irr64, mom64 = ddgi.blend_f64(rgb, dep, w, prev_i, prev_m, h)
    if not h:
        np.testing.assert_allclose(irr, irr64, rtol=1e-6, atol=1e-7)
        np.testing.assert_allclose(mom, mom64, rtol=1e-6, atol=1e-7)
    else:
        # fma(h, prev - frame, frame) in float32: the difference prev - frame
        # is rounded once, so the error scales with |prev| + |frame|
        f_irr, f_mom = ddgi.blend_f64(rgb, dep, w, None, None, 0.0)
        for got, want, prev, frame in ((irr, irr64, prev_i, f_irr), (mom, mom64, prev_m, f_mom)):
            tol = 1e-6 * np.abs(want) + 2 * np.spacing(np.abs(prev) + np.abs(frame).astype(np.float32))
            assert np.all(np.abs(got - want) <= tol)


def test_oracle_weights_follow_the_definition():
    """Colour weight = max(0, n.d) within 2 ulp of the float64 dot product;
    depth weight = that cosine ^ sharpness rounded once."""
    dirs = ddgi.ray_table(256, 2, 3).astype(np.float32)
    wc, wd, inv_c, inv_d = ddgi.blend_weights(dirs, 50.0)
    n8 = ddgi.texel_directions(8).astype(np.float32).astype(np.float64)
    exact = np.maximum(n8 @ dirs[:, :3].astype(np.float64).T, 0.0)
    assert np.all(np.abs(wc - exact) <= 2 * np.spacing(np.float32(1.0)))
    _, cd = ddgi.texel_cosines(dirs)
    assert np.array_equal(wd, np.power(cd.astype(np.float64), 50.0).astype(np.float32))
    np.testing.assert_allclose(inv_c, 1.0 / wc.astype(np.float64).sum(1), rtol=1.2e-7)
    np.testing.assert_allclose(inv_d, 1.0 / wd.astype(np.float64).sum(1), rtol=1.2e-7)
