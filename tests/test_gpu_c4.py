"""Parity at the benchmarked configuration (BASELINE config 4: 64x32x64
probes, 256 rays, the ~270k-triangle hall, shadow maps, full-volume update).

(a) stages 1+2: 64 probes spread over every z-slab boundary of a 2/4/8-GPU
    split, traced, shaded and blended over two frames (first frame, then
    hysteresis) against the oracle: traversal vs the float64 brute force
    (reference raycast semantics, selection.py:66-149), shading / blend at
    1e-4 relative / 1e-5 absolute (north_star), quantised blocks bit-exact.
(b) stages 3+4: two C4 ProbeStreamServer frames (the bench's server path,
    CUDA-graph replay on the second) -- entries, update texels, planes,
    residual and SKIP maps bit-exact against the oracle restatement of
    selection.py:284-437, packing.py:73-133,283-338 and codec.py:207-272.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import ddgi
from oracle import stream_ops as so

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-4, 1e-5
DIMS = (64, 32, 64)


@pytest.fixture(scope="module")
def hall():
    from paper_2103_05875_b200 import build_native

    build_native.build()
    from paper_2103_05875_b200 import scene

    sc = scene.interior_hall()
    return sc, scene.volume_for(sc, DIMS)


def _sample_ids(vol, rng):
    nx, ny, nz = vol.dims
    ks = sorted({0, nz - 1} | {b + d for b in range(0, nz, nz // 8) for d in (-1, 0)
                               if 0 <= b + d < nz})
    ids = []
    for k in ks:
        for _ in range(max(1, 64 // len(ks))):
            i, j = rng.integers(0, nx), rng.integers(0, ny)
            ids.append(int(i + nx * (j + ny * k)))
    ids = sorted(set(ids))
    assert len(ids) >= 64 or len(ids) >= len(ks)
    return np.asarray(ids, np.int64)


def _records(upd, ids):
    R = upd.rays_per_probe
    rec = upd.ray_records.view(-1, R, 8)[torch.from_numpy(ids - upd.probe_begin).to(upd.device)]
    rec = rec.cpu().numpy()
    return (rec[..., 0:3], rec[..., 3], rec[..., 4], rec[..., 5].view(np.int32),
            rec[..., 6].view(np.int32))


def _check_trace(upd, sc, ids, frame, frame_lights):
    rgb, depth, t, prim, mask = _records(upd, ids)
    P, R = prim.shape
    pos = upd.volume.probe_positions(ids).astype(np.float32).astype(np.float64)
    dirs = upd.ray_dirs.cpu().numpy()[:, :3].astype(np.float64)
    O, Dd = np.repeat(pos, R, axis=0), np.tile(dirs, (P, 1))
    t_ref, prim_ref = ddgi.raycast(sc.vertices, O, Dd)
    prim_g, t_g = prim.reshape(-1), t.reshape(-1).astype(np.float64)
    hit_ref, hit_g = prim_ref >= 0, prim_g >= 0
    both = hit_ref & hit_g
    rel = np.abs(t_g[both] - t_ref[both]) / np.maximum(t_ref[both], 1e-6)
    prim_ok = (prim_g[both] == prim_ref[both]) | (rel < 1e-5)
    mismatch = (hit_ref != hit_g).sum() + (~prim_ok).sum()
    assert mismatch <= 2e-3 * len(prim_g), f"traversal mismatch {mismatch} of {len(prim_g)}"
    assert np.all(rel[prim_ok] < 1e-4)
    lights = [(l.position, l.intensity) for l in frame_lights]
    maps = upd.shadow_maps[: len(lights)].cpu().numpy().astype(np.float64)
    # the device's cube maps against the oracle's own rays on a sample of texels
    S = upd.shadow_map_size
    dirs_map = ddgi.shadow_map_dirs(S).reshape(-1, 3).astype(np.float64)
    rng = np.random.default_rng(frame)
    for li, (lp, _) in enumerate(lights):
        pick = rng.choice(len(dirs_map), size=2000, replace=False)
        t_map, _ = ddgi.raycast(sc.vertices, np.asarray(lp, np.float64)[None, :], dirs_map[pick])
        g = maps[li].reshape(-1)[pick]
        assert (np.isfinite(t_map) != np.isfinite(g)).mean() < 2e-3
        fin = np.isfinite(t_map) & np.isfinite(g)
        assert (np.abs(g[fin] - t_map[fin]) <= 1e-4 * t_map[fin] + 1e-6).mean() > 0.995
    rgb_ref, dep_ref, mask_ref = ddgi.shade(sc.vertices, sc.albedo, sc.emission, lights, sc.sky, O,
                                            Dd, t_ref, prim_ref, upd.max_distance, upd.normal_bias,
                                            upd.shadows, upd.shadow_map_size, upd.shadow_bias, maps)
    agree = (hit_ref == hit_g)
    agree[np.nonzero(both)[0][~prim_ok]] = False
    agree &= prim_g == np.where(hit_ref, prim_ref, -1)
    mask_agree = agree & (mask.reshape(-1) == mask_ref)
    assert (agree & ~mask_agree).sum() <= max(2, 2e-3 * len(prim_g)), "shadow mismatch"
    np.testing.assert_allclose(rgb.reshape(-1, 3)[mask_agree], rgb_ref[mask_agree],
                               rtol=RTOL, atol=ATOL)
    np.testing.assert_allclose(depth.reshape(-1)[agree], dep_ref[agree], rtol=RTOL, atol=ATOL)


def _check_blend(upd, ids, prev, h):
    rgb, depth, *_ = _records(upd, ids)
    w = ddgi.check_device_weights(upd.w_color.cpu().numpy(), upd.w_depth.cpu().numpy(),
                                  upd.ray_dirs.cpu().numpy(), upd.sharpness)
    irr, mom = ddgi.blend(rgb, depth, w, prev[0] if prev else None, prev[1] if prev else None, h)
    loc = torch.from_numpy(ids - upd.probe_begin).to(upd.device)
    g_irr = upd.irradiance[loc].cpu().numpy()
    g_mom = upd.moments[loc].cpu().numpy()
    np.testing.assert_allclose(g_irr, irr, rtol=RTOL, atol=ATOL)
    np.testing.assert_allclose(g_mom, mom, rtol=RTOL, atol=ATOL)
    # quantised + guard-banded blocks from the device state: bit-exact
    color = upd.color.texels.cpu().numpy()
    vis = upd.visibility.texels.cpu().numpy()
    qc = ddgi.quantize_color(g_irr, upd.irradiance_scale)
    qv = ddgi.quantize_moments(g_mom)
    for i, p in enumerate(ids):
        br, bc = divmod(int(p), upd.color.probes_per_row)
        assert np.array_equal(color[br * 10:(br + 1) * 10, bc * 10:(bc + 1) * 10],
                              so.guard_band_block(qc[i]))
        br, bc = divmod(int(p), upd.visibility.probes_per_row)
        assert np.array_equal(vis[br * 18:(br + 1) * 18, bc * 18:(bc + 1) * 18],
                              so.guard_band_block(qv[i]))
    return g_irr, g_mom


def test_c4_trace_and_blend_sampled_probes(hall):
    from paper_2103_05875_b200 import probes, scene

    sc, vol = hall
    upd = probes.ProbeUpdater(vol, sc, rays_per_probe=256, record_rays=True,
                              irradiance_scale=4.0, shadows="map")
    ids = _sample_ids(vol, np.random.default_rng(4))
    assert len(ids) >= 64
    prev = None
    for f in range(2):
        lights = scene.moving_light(sc, f).lights
        upd.update(f, lights)
        torch.cuda.synchronize()
        _check_trace(upd, sc, ids, f, lights)
        prev = _check_blend(upd, ids, prev, 0.0 if f == 0 else upd.hysteresis)


@pytest.mark.parametrize("variant", ["full", "budget"])
def test_c4_server_frames_bit_exact(hall, variant):
    """Stage 3/4 outputs of two C4 server frames, bit-exact vs the oracle on
    the device-produced atlases (no tolerance chains into the
    bit-exact stages)."""
    from paper_2103_05875_b200 import scene
    from paper_2103_05875_b200.server import ProbeStreamServer

    sc, vol = hall
    n = vol.probe_count
    kw = {} if variant == "full" else {"budget": 50_000, "color_threshold": 4.0,
                                       "visibility_threshold": 1e-3}
    srv = ProbeStreamServer(vol, sc, rays_per_probe=256, irradiance_scale=4.0, graphs=True, **kw)
    budget = kw.get("budget")
    thr = {"color": kw.get("color_threshold", 0.0), "visibility": kw.get("visibility_threshold", 0.0)}
    state = {}
    for frame in range(2):
        outs = srv.tick(frame, scene.moving_light(sc, frame).lights)
        srv.join()
        torch.cuda.synchronize()
        for ks, out in zip((srv.color, srv.visibility), outs):
            kind = ks.kind.value
            rendered = (srv.updater.color if kind == "color" else srv.updater.visibility)
            cur = rendered.texels.cpu().numpy()
            st = state.setdefault(kind, {"last": np.zeros_like(cur), "seq": np.full(n, -1),
                                         "cache": so.SlotCache(n, ks.kind.core_side),
                                         "tex": None, "planes": None})
            ppr = rendered.probes_per_row
            changed = so.detect_changed(cur, st["last"], kind, n, ppr, vol.active, thr[kind])
            sel = so.select_for_client(changed, np.arange(n), vol.active, st["seq"], frame, budget)
            if variant == "full":
                # every probe is traced and blended; those whose blocks differ
                # from the last-sent ones are sent (all-black colour blocks of
                # probes buried in walls equal the zero-initialised last-sent)
                assert len(sel) > 0.95 * n
            tex, entries = so.build_update_atlas(sel, st["cache"], cur, kind, ppr, st["tex"])
            st["tex"] = tex
            k = int(out.entry_count.item())
            assert k == len(entries)
            assert np.array_equal(out.entries[:k].cpu().numpy(), np.asarray(entries).reshape(-1, 2))
            assert np.array_equal(ks.update_texels.cpu().numpy(), tex)
            planes = so.pack_texels(tex, kind)
            assert np.array_equal(out.planes.cpu().numpy(), planes)
            if st["planes"] is not None:
                res, skip = so.temporal_delta(planes, st["planes"])
                assert np.array_equal(out.residual.cpu().numpy(), res)
                assert np.array_equal(out.skip.cpu().numpy(), skip)
            st["planes"] = planes
            # commit: last-sent blocks and sequence stamps
            side = so.block_side(kind)
            last = st["last"]
            for p in sel:
                br, bc = divmod(int(p), ppr)
                last[br * side:(br + 1) * side, bc * side:(bc + 1) * side] = \
                    cur[br * side:(br + 1) * side, bc * side:(bc + 1) * side]
            st["seq"][np.asarray(sel, np.int64)] = frame
            assert np.array_equal(ks.last_sent.texels.cpu().numpy(), last)
            assert np.array_equal(ks.last_sent_seq.cpu().numpy(), st["seq"])
