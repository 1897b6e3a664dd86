"""CPU baseline of one server frame: the reference's CPU path, sampled.

TEST / BASELINE INFRASTRUCTURE ONLY: ``bench.py`` times this as the
``cpu_baseline`` / ``--impl reference`` leg; nothing in the product package
imports it.

One *step* does a bounded sample of each part of the frame and reports the
wall time it actually took plus a per-probe cost for every part:

* stage (1)+(2): ``sample_probes`` probes traced with the reference's own ray
  query algorithm (brute-force ``SceneGeometry.raycast`` semantics,
  selection.py:66-149, restated in C, float64, OpenMP over all host threads),
  shaded and blended by the numpy DDGI restatement (``ddgi``);
* shadow maps: ``map_sample`` cube-map texels per light, same query;
* stages (3)-(4) on the whole volume (or a z-slab of ``stage_probes`` probes; every probe changed,
  the full-volume update): the REAL reference functions ``detect_changed``
  (selection.py:284), ``select_for_client`` (:413), ``build_update_atlas``
  (packing.py:320) and ``pack_texels`` (:154) when the reference package is
  importable ($PROBESTREAM_REF or the offline install ``baseline/_ref``,
  which travels to the GPU box), else their numpy restatements in
  ``stream_ops``; the temporal delta (inside the reference's
  ``encode_frame``, codec.py:207-272, seconds per block loop) is always the
  numpy restatement.

Every part is linear in its sample (rays are independent, the stage
functions are per-probe block loops), so the whole-volume frame costs
``n * (trace_blend/probe + stages/probe) + map_texels * map/texel``; the
reported rate is ``n / that``.
"""

from __future__ import annotations

import importlib
import os
import sys
import time
from pathlib import Path

import numpy as np

from . import ddgi
from . import stream_ops as so

ROOT = Path(__file__).resolve().parents[1]


def load_reference():
    """The reference ``probestream`` package from $PROBESTREAM_REF or
    ``baseline/_ref``, or None (never reads /root/reference at run time)."""
    if "probestream" in sys.modules:
        mod = sys.modules["probestream"]
        for sub in ("volume", "selection", "packing"):
            importlib.import_module(f"probestream.{sub}")
        return mod
    cands = [os.environ.get("PROBESTREAM_REF"), str(ROOT / "baseline" / "_ref")]
    for c in cands:
        if c and (Path(c) / "probestream" / "__init__.py").exists():
            sys.path.insert(0, c)
            try:
                mod = importlib.import_module("probestream")
                for sub in ("volume", "selection", "packing"):
                    importlib.import_module(f"probestream.{sub}")
                return mod
            except Exception:  # pragma: no cover - broken install
                sys.path.remove(c)
    return None


def time_stages(dims, stage_probes: int, rng, prefer_reference: bool = True) -> dict:
    """Stages (3)-(4), colour + visibility, on the first ``stage_probes``
    probes (a z-slab when it is a multiple of nx*ny): every probe changed,
    no budget.  Returns seconds, the implementation used and the selected
    counts."""
    nx, ny, nz = dims
    plane = nx * ny
    n = max(plane, min(stage_probes, nx * ny * nz) // plane * plane)
    sub = (nx, ny, n // plane)
    ref = load_reference() if prefer_reference else None
    out = {"probes": n, "impl": "reference" if ref is not None else "port", "s": 0.0,
           "selected": {}, "parts_s": {}}
    if ref is not None:
        V = ref.volume
        vol = V.ProbeVolume(sub)
        kinds = ((V.AtlasKind.COLOR, "color"), (V.AtlasKind.VISIBILITY, "visibility"))
    else:
        act = np.ones(n, bool)
        kinds = ((None, "color"), (None, "visibility"))
    for K, kind in kinds:
        ppr = so.default_probes_per_row(n)
        shp = so.atlas_shape(kind, n, ppr)
        dt = np.uint32 if kind == "color" else np.uint16
        cur = rng.integers(0, 2**16, size=shp, dtype=dt)
        last = cur ^ dt(1)  # every probe changed: the full-volume update
        parts = {}
        s0 = time.perf_counter()
        if ref is not None:
            a_cur = V.ProbeAtlas(K, n, ppr, cur)
            a_last = V.ProbeAtlas(K, n, ppr, last)
            changed = ref.selection.detect_changed(a_cur, a_last, vol)
            s1 = time.perf_counter()
            sel = ref.selection.select_for_client(changed, changed, vol, np.zeros(n, np.int64), 1)
            s2 = time.perf_counter()
            layout = ref.packing.UpdateAtlasLayout(n, K.core_side)
            upd, _ = ref.packing.build_update_atlas(sel, layout, a_cur)
            s3 = time.perf_counter()
            planes = np.asarray(ref.packing.pack_texels(upd, K).data)
        else:
            changed = so.detect_changed(cur, last, kind, n, ppr, act)
            s1 = time.perf_counter()
            sel = so.select_for_client(changed, changed, act, np.zeros(n, np.int64), 1)
            s2 = time.perf_counter()
            cache = so.SlotCache(n, so.BLOCK_SIDE[kind] - 2)
            upd, _ = so.build_update_atlas(sel, cache, cur, kind, ppr)
            s3 = time.perf_counter()
            planes = so.pack_texels(upd, kind)
        s4 = time.perf_counter()
        so.temporal_delta(planes, planes ^ planes.dtype.type(1))
        s5 = time.perf_counter()
        parts.update(detect=s1 - s0, select=s2 - s1, build=s3 - s2, pack=s4 - s3, delta=s5 - s4)
        out["parts_s"][kind] = {k: round(v, 4) for k, v in parts.items()}
        out["s"] += s5 - s0
        out["selected"][kind] = int(len(sel))
    return out


def time_frame(scene, volume, rays_per_probe: int, sample_probes: int = 4, seed: int = 0,
               frame: int = 0, shadows: str = "map", max_distance=None, bias=None,
               stage_probes: int | None = None, rng_seed: int = 0, shadow_map_size: int = 256,
               map_sample: int = 1024, prefer_reference: bool = True) -> dict:
    """One sampled step.  Returns per-part seconds, per-probe costs, the wall
    time of the step and the whole-volume frame time those costs imply."""
    w0 = time.perf_counter()
    n = volume.probe_count
    (x0, y0, z0), (x1, y1, z1) = scene.bounds
    diag = float(np.sqrt((x1 - x0) ** 2 + (y1 - y0) ** 2 + (z1 - z0) ** 2))
    max_distance = diag if max_distance is None else max_distance
    bias = 1e-3 * diag if bias is None else bias
    rng = np.random.default_rng(rng_seed)
    ids = np.sort(rng.choice(n, size=min(sample_probes, n), replace=False))
    dirs = ddgi.ray_table(rays_per_probe, seed, frame).astype(np.float64)
    lights = [(l.position, l.intensity) for l in scene.lights]

    map_s = 0.0
    map_texels = 0
    maps = None
    if shadows == "map" and lights:
        S = shadow_map_size
        dirs_map = ddgi.shadow_map_dirs(S).reshape(-1, 3).astype(np.float64)
        pick = rng.choice(len(dirs_map), size=min(map_sample, len(dirs_map)), replace=False)
        maps = np.full((len(lights), 6 * S * S), np.inf)
        m0 = time.perf_counter()
        for li, (lp, _) in enumerate(lights):
            tm, _ = ddgi.raycast(scene.vertices, np.asarray(lp, np.float64)[None, :], dirs_map[pick])
            maps[li, pick] = tm
        map_s = time.perf_counter() - m0
        map_texels = len(lights) * len(pick)
        maps = maps.reshape(len(lights), 6, S, S)
    map_frame_s = map_s / map_texels * len(lights) * 6 * shadow_map_size ** 2 if map_texels else 0.0

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
    st = time_stages(volume.dims, stage_probes or n, rng, prefer_reference)
    wall = time.perf_counter() - w0
    per_probe_tb = (t2 - t0) / len(ids)
    per_probe_st = st["s"] / st["probes"]
    frame_s = n * (per_probe_tb + per_probe_st) + map_frame_s
    return {
        "wall_s": wall,
        "sample_probes": int(len(ids)),
        "sample_rays": int(len(ids) * rays_per_probe),
        "trace_shade_s": t1 - t0,
        "blend_s": t2 - t1,
        "trace_blend_s_per_probe": per_probe_tb,
        "map_sample_texels": map_texels,
        "map_sample_s": map_s,
        "shadow_map_frame_s": map_frame_s,
        "stage_probes": st["probes"],
        "stages_s": st["s"],
        "stages_impl": st["impl"],
        "stages_s_per_probe": per_probe_st,
        "stages_parts_s": st["parts_s"],
        "selected": st["selected"],
        "frame_s": frame_s,
        "probe_updates_per_s": n / frame_s,
        "threads": os.cpu_count(),
    }


def warm_up(scene) -> None:
    """Load (and if needed build) the C oracle and spin up its thread pool,
    and import the reference package, outside any timed region."""
    ddgi.raycast(scene.vertices[:1], np.zeros((1, 3)), np.ones((64, 3)))
    load_reference()
