"""GPU parity for stages (1)+(2): BVH traversal vs the float64 brute-force
raycast oracle (reference semantics), shading, the DDGI blend (tolerance
1e-4 relative / 1e-5 absolute, per BASELINE north_star) and the quantised
atlas (bit-exact given the float state)."""

import numpy as np
import pytest
import torch

from oracle import ddgi
from oracle import stream_ops as so

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-4, 1e-5


@pytest.fixture(scope="module")
def pkg():
    from paper_2103_05875_b200 import build_native

    build_native.build()
    import paper_2103_05875_b200 as p
    from paper_2103_05875_b200 import probes, scene

    return p, probes, scene


def _records(upd):
    rec = upd.ray_records.cpu().numpy().reshape(-1, upd.rays_per_probe, 8)
    rgb = rec[..., 0:3]
    depth = rec[..., 3]
    t = rec[..., 4]
    prim = rec[..., 5].view(np.int32)
    mask = rec[..., 6].view(np.int32)
    return rgb, depth, t, prim, mask


def _check_trace(upd, sc, frame, max_mismatch=2e-3):
    """Traversal + shading against the oracle; returns agreement stats."""
    rgb, depth, t, prim, mask = _records(upd)
    P, R = prim.shape
    ids = np.arange(upd.probe_begin, upd.probe_end)
    pos = upd.volume.probe_positions(ids).astype(np.float32).astype(np.float64)
    dirs = upd.ray_dirs.cpu().numpy()[:, :3].astype(np.float64)
    O = np.repeat(pos, R, axis=0)
    Dd = np.tile(dirs, (P, 1))
    t_ref, prim_ref = ddgi.raycast(sc.vertices, O, Dd)
    prim_g = prim.reshape(-1)
    t_g = t.reshape(-1).astype(np.float64)
    hit_ref = prim_ref >= 0
    hit_g = prim_g >= 0
    same_hit = hit_ref == hit_g
    both = hit_ref & hit_g
    rel = np.abs(t_g[both] - t_ref[both]) / np.maximum(t_ref[both], 1e-6)
    # same primitive, or a different one at (numerically) the same distance
    # (shared edges / coplanar overlaps)
    prim_ok = (prim_g[both] == prim_ref[both]) | (rel < 1e-5)
    mismatch = (~same_hit).sum() + (~prim_ok).sum()
    rate = mismatch / len(prim_g)
    assert rate <= max_mismatch, f"traversal mismatch rate {rate:.2e}"
    assert np.all(rel[prim_ok] < 1e-4), rel.max()
    # shading with the oracle's own shadow rays, on rays whose hit agrees
    lights = [(l.position, l.intensity) for l in upd.dscene.scene.lights]
    maps = None
    if upd.shadows == "map":
        # the device's maps, checked against the oracle's own on a sample
        S = upd.shadow_map_size
        g_maps = upd.shadow_maps[: len(lights)].cpu().numpy().astype(np.float64)
        dirs_map = ddgi.shadow_map_dirs(S).reshape(-1, 3).astype(np.float64)
        rng = np.random.default_rng(frame)
        for li, (lp, _) in enumerate(lights):
            pick = rng.choice(len(dirs_map), size=min(2000, len(dirs_map)), replace=False)
            t_map, _ = ddgi.raycast(sc.vertices, np.asarray(lp, np.float64)[None, :], dirs_map[pick])
            g = g_maps[li].reshape(-1)[pick]
            assert (np.isfinite(t_map) != np.isfinite(g)).mean() < 2e-3
            fin = np.isfinite(t_map) & np.isfinite(g)
            close = np.abs(g[fin] - t_map[fin]) <= 1e-4 * t_map[fin] + 1e-6
            assert close.mean() > 0.995, close.mean()
        maps = g_maps  # lookups are then compared on identical map values
    rgb_ref, dep_ref, mask_ref = ddgi.shade(sc.vertices, sc.albedo, sc.emission, lights, sc.sky, O,
                                            Dd, t_ref, prim_ref, upd.max_distance, upd.normal_bias,
                                            upd.shadows, upd.shadow_map_size, upd.shadow_bias, maps)
    agree = same_hit.copy()
    agree[np.nonzero(both)[0][~prim_ok]] = False
    agree &= prim_g == np.where(hit_ref, prim_ref, -1)
    mask_agree = agree & (mask.reshape(-1) == mask_ref)
    assert (agree & ~mask_agree).sum() <= max(2, 2e-3 * len(prim_g)), "shadow mismatch"
    np.testing.assert_allclose(rgb.reshape(-1, 3)[mask_agree], rgb_ref[mask_agree], rtol=RTOL, atol=ATOL)
    np.testing.assert_allclose(depth.reshape(-1)[agree], dep_ref[agree], rtol=RTOL, atol=ATOL)
    return rate


def _check_blend(upd, prev_irr, prev_mom, h):
    rgb, depth, *_ = _records(upd)
    w = ddgi.check_device_weights(upd.w_color.cpu().numpy(), upd.w_depth.cpu().numpy(),
                                  upd.ray_dirs.cpu().numpy(), upd.sharpness)
    irr, mom = ddgi.blend(rgb, depth, w, prev_irr, prev_mom, h)
    g_irr = upd.irradiance.cpu().numpy()
    g_mom = upd.moments.cpu().numpy()
    np.testing.assert_allclose(g_irr, irr, rtol=RTOL, atol=ATOL)
    np.testing.assert_allclose(g_mom, mom, rtol=RTOL, atol=ATOL)
    return g_irr, g_mom


def _check_atlas(upd):
    """Quantisation + guard band from the device float state: bit-exact."""
    ids = np.arange(upd.probe_begin, upd.probe_end)
    color = upd.color.texels.cpu().numpy()
    vis = upd.visibility.texels.cpu().numpy()
    want_c = np.zeros_like(color)
    want_v = np.zeros_like(vis)
    ddgi.write_blocks(want_c, "color", upd.color.probes_per_row, ids,
                      ddgi.quantize_color(upd.irradiance.cpu().numpy(), upd.irradiance_scale))
    ddgi.write_blocks(want_v, "visibility", upd.visibility.probes_per_row, ids,
                      ddgi.quantize_moments(upd.moments.cpu().numpy()))
    for p in ids[:: max(1, len(ids) // 64)]:
        br, bc = divmod(int(p), upd.color.probes_per_row)
        assert np.array_equal(color[br * 10:(br + 1) * 10, bc * 10:(bc + 1) * 10],
                              want_c[br * 10:(br + 1) * 10, bc * 10:(bc + 1) * 10])
        br, bc = divmod(int(p), upd.visibility.probes_per_row)
        assert np.array_equal(vis[br * 18:(br + 1) * 18, bc * 18:(bc + 1) * 18],
                              want_v[br * 18:(br + 1) * 18, bc * 18:(bc + 1) * 18])
    if upd.probe_begin == 0 and upd.probe_end == upd.volume.probe_count:
        assert np.array_equal(color, want_c)
        assert np.array_equal(vis, want_v)


@pytest.mark.parametrize("shadows", ["map", "rays"])
def test_cornell_box_config1(pkg, shadows):
    """Config 1: analytic Cornell box, 8x8x8 probes, 64 rays, three frames."""
    p, probes, scene = pkg
    sc = scene.cornell_box()
    vol = scene.volume_for(sc, (8, 8, 8))
    upd = probes.ProbeUpdater(vol, sc, rays_per_probe=64, hysteresis=0.9, record_rays=True,
                              irradiance_scale=2.0, shadows=shadows, shadow_map_size=128)
    irr = np.zeros((512, 64, 3), np.float32)
    mom = np.zeros((512, 256, 2), np.float32)
    for f in range(3):
        upd.update(f)
        torch.cuda.synchronize()
        _check_trace(upd, sc, f)
        irr, mom = _check_blend(upd, irr, mom, 0.0 if f == 0 else 0.9)
        _check_atlas(upd)
    # guard bands valid on every produced block
    from paper_2103_05875_b200.packing import guard_band_valid

    c = upd.color.texels.cpu().numpy()
    for pid in range(0, 512, 37):
        br, bc = divmod(pid, upd.color.probes_per_row)
        assert guard_band_valid(c[br * 10:(br + 1) * 10, bc * 10:(bc + 1) * 10])
    # something is lit and something is in shadow
    assert upd.irradiance.max().item() > 0.01


@pytest.mark.parametrize("shadows", ["map", "rays", "none"])
def test_interior_hall_sampled_probes(pkg, shadows):
    """Config 2 scene (~270k triangles), 256 rays; a sampled probe range is
    checked against the float64 brute-force oracle."""
    p, probes, scene = pkg
    sc = scene.interior_hall()
    vol = scene.volume_for(sc, (32, 16, 32))
    # a slab of probes in the middle of the hall (contiguous id range)
    begin = 16 + 32 * (8 + 16 * 16)
    upd = probes.ProbeUpdater(vol, sc, rays_per_probe=256, record_rays=True, shadows=shadows,
                              probe_range=(begin, begin + 6), irradiance_scale=4.0)
    upd.update(0)
    torch.cuda.synchronize()
    _check_trace(upd, sc, 0)
    _check_blend(upd, None, None, 0.0)
    _check_atlas(upd)


def test_slab_sharding_is_consistent(pkg):
    """Two half ranges give the same atlas/state as one full range."""
    p, probes, scene = pkg
    sc = scene.cornell_box()
    vol = scene.volume_for(sc, (8, 8, 8))
    full = probes.ProbeUpdater(vol, sc, rays_per_probe=64)
    full.update(0)
    a = probes.ProbeUpdater(vol, sc, rays_per_probe=64, probe_range=(0, 256))
    b = probes.ProbeUpdater(vol, sc, rays_per_probe=64, probe_range=(256, 512))
    a.update(0)
    b.update(0)
    torch.cuda.synchronize()
    assert torch.equal(full.irradiance[:256], a.irradiance)
    assert torch.equal(full.irradiance[256:], b.irradiance)
    merged = a.color.texels.view(torch.int32) | b.color.texels.view(torch.int32)
    assert torch.equal(merged, full.color.texels.view(torch.int32))


def _axis_ray_set(count=64, seed=11):
    """Directions that stress the octant-specialised node test: the six axes
    with signed-zero components, the eight diagonals, then random ones."""
    z = -0.0
    fixed = [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1),
             (1, z, z), (z, z, -1), (z, 1, z), (-1, z, 0)]
    fixed += [(sx, sy, sz) for sx in (1, -1) for sy in (1, -1) for sz in (1, -1)]
    d = np.array(fixed, np.float64)
    rng = np.random.default_rng(seed)
    r = rng.normal(size=(count - len(d), 3))
    d = np.concatenate([d, r])
    n = np.linalg.norm(d, axis=1, keepdims=True)
    d = np.where(d == 0, d, d / n)  # keeps the signed zeros
    out = np.zeros((count, 4), np.float32)
    out[:, :3] = d
    return out


@pytest.mark.parametrize("probe_range", [None, (3 * 64, 4 * 64)])
def test_axis_aligned_and_signed_zero_rays(pkg, monkeypatch, probe_range):
    """Axis-aligned rays (tiny reciprocal stand-ins, -0.0 components) through
    the octant-specialised BVH4 trace -- deep slab (2x2x8 tiles) and a
    one-plane slab (4x4x2 tiles) -- against the float64 oracle."""
    p, probes, scene = pkg
    monkeypatch.setattr(probes, "frame_ray_directions", lambda count, seed, frame: _axis_ray_set(count))
    sc = scene.cornell_box()
    vol = scene.volume_for(sc, (8, 8, 8))
    kw = {"probe_range": probe_range} if probe_range else {}
    upd = probes.ProbeUpdater(vol, sc, rays_per_probe=64, record_rays=True, shadows="rays", **kw)
    upd.update(0)
    torch.cuda.synchronize()
    _check_trace(upd, sc, 0)
    _check_blend(upd, None, None, 0.0)
