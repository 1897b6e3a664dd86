"""CPU baseline of one server frame, built from the oracle port.

TEST / BASELINE INFRASTRUCTURE ONLY: ``bench.py`` times this as the
``cpu_baseline`` / ``--impl reference`` leg.  Stage (1) is the reference's
own ray query algorithm (brute-force ``SceneGeometry.raycast`` semantics,
selection.py:66-149, restated in C with OpenMP over all host threads);
stages (3)-(4) are the numpy restatements of the reference's functions in
``stream_ops`` at the full probe count.  Stage (1)+(2) are timed on a bounded
sample of probes and scaled linearly to the volume (rays are independent).
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import ddgi
from . import stream_ops as so


def time_frame(scene, volume, rays_per_probe: int, sample_probes: int = 4, seed: int = 0,
               frame: int = 0, shadows: str = "map", max_distance=None, bias=None,
               stages_full: bool = True, rng_seed: int = 0, shadow_map_size: int = 256,
               map_sample: int = 2048) -> dict:
    """Returns a dict of seconds per stage and the extrapolated frame time."""
    n = volume.probe_count
    (x0, y0, z0), (x1, y1, z1) = scene.bounds
    diag = float(np.sqrt((x1 - x0) ** 2 + (y1 - y0) ** 2 + (z1 - z0) ** 2))
    max_distance = diag if max_distance is None else max_distance
    bias = 1e-3 * diag if bias is None else bias
    rng = np.random.default_rng(rng_seed)
    ids = np.sort(rng.choice(n, size=min(sample_probes, n), replace=False))
    dirs = ddgi.ray_table(rays_per_probe, seed, frame).astype(np.float64)
    lights = [(l.position, l.intensity) for l in scene.lights]

    # load (and if needed build) the C oracle and spin up its thread pool
    # outside the timed regions
    ddgi.raycast(scene.vertices[:1], np.zeros((1, 3)), np.ones((64, 3)))
    map_s = 0.0
    maps = None
    if shadows == "map" and lights:
        # cube distance maps are a fixed per-frame cost: time a sample of map
        # texels per light with the same brute-force query and scale it
        S = shadow_map_size
        dirs_map = ddgi.shadow_map_dirs(S).reshape(-1, 3).astype(np.float64)
        pick = rng.choice(len(dirs_map), size=min(map_sample, len(dirs_map)), replace=False)
        maps = np.full((len(lights), 6 * S * S), np.inf)
        m0 = time.perf_counter()
        for li, (lp, _) in enumerate(lights):
            tm, _ = ddgi.raycast(scene.vertices, np.asarray(lp, np.float64)[None, :], dirs_map[pick])
            maps[li, pick] = tm
        map_s = (time.perf_counter() - m0) * (6 * S * S) / len(pick)
        maps = maps.reshape(len(lights), 6, S, S)

    t0 = time.perf_counter()
    pos = volume.probe_positions(ids).astype(np.float32).astype(np.float64)
    O = np.repeat(pos, rays_per_probe, axis=0)
    D = np.tile(dirs, (len(ids), 1))
    t, prim = ddgi.raycast(scene.vertices, O, D)
    rgb, depth, _ = ddgi.shade(scene.vertices, scene.albedo, scene.emission, lights, scene.sky,
                               O, D, t, prim, max_distance, bias, shadows, shadow_map_size, 0.02,
                               maps)
    t1 = time.perf_counter()
    w = ddgi.blend_weights(dirs.astype(np.float32), 50.0)
    irr, mom = ddgi.blend(rgb.reshape(len(ids), rays_per_probe, 3).astype(np.float32),
                          depth.reshape(len(ids), rays_per_probe).astype(np.float32), w,
                          None, None, 0.0)
    ddgi.quantize_color(irr, 1.0)
    ddgi.quantize_moments(mom)
    t2 = time.perf_counter()
    per_probe = (t2 - t0) / len(ids)
    out = {"trace_shade_s_per_probe": (t1 - t0) / len(ids),
           "blend_s_per_probe": (t2 - t1) / len(ids),
           "shadow_map_s": map_s,
           "sample_probes": int(len(ids)),
           "sample_rays": int(len(ids) * rays_per_probe)}
    stages = 0.0
    if stages_full:
        ppr = so.default_probes_per_row(n)
        act = np.asarray(volume.active, bool)
        for kind in ("color", "visibility"):
            shp = so.atlas_shape(kind, n, ppr)
            dt = np.uint32 if kind == "color" else np.uint16
            cur = rng.integers(0, 2**16, size=shp, dtype=dt)
            last = cur ^ dt(1)  # every probe changed: the full-volume update
            s0 = time.perf_counter()
            changed = so.detect_changed(cur, last, kind, n, ppr, act)
            sel = so.select_for_client(changed, changed, act, np.zeros(n, np.int64), 1)
            cache = so.SlotCache(n, so.BLOCK_SIDE[kind] - 2)
            upd, _ = so.build_update_atlas(sel, cache, cur, kind, ppr)
            planes = so.pack_texels(upd, kind)
            so.temporal_delta(planes, planes ^ planes.dtype.type(1))
            stages += time.perf_counter() - s0
    out["stages_s"] = stages
    out["frame_s"] = per_probe * n + map_s + stages
    out["threads"] = os.cpu_count()
    return out
