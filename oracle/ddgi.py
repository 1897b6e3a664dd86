"""CPU oracle for stages (1)+(2): ray set, traversal, shading, DDGI blend.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__``).

PARITY UNPINNED for the DDGI arithmetic itself: the reference has no probe
tracer and no irradiance/depth blend, so this module restates
the algorithm documented in ``paper_2103_05875_b200/probes.py`` and
DESIGN.md.  The pieces that the reference does pin are restated from it and
checked against its golden vectors (tests/golden/geometry.npz):

* ``fibonacci_sphere``      selection.py:241-249
* ``texel_directions``      volume.py:286-314 (texel centres + oct_decode)
* ``raycast`` (C, float64)  selection.py:66-149 for triangles
* guard band rule           packing.py:180-196 (via stream_ops.guard_band_block)
* texel formats             volume.py:150-153, :221-226
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

from . import stream_ops as so

HERE = Path(__file__).resolve().parent
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        so_path = HERE / "build" / "libraycast.so"
        if not so_path.exists() or so_path.stat().st_mtime < (HERE / "raycast.c").stat().st_mtime:
            subprocess.run(["make", "-C", str(HERE)], check=True, capture_output=True)
        lib = ctypes.CDLL(str(so_path))
        vp, i64 = ctypes.c_void_p, ctypes.c_int64
        lib.oracle_raycast.argtypes = [vp, i64, vp, vp, i64, vp, vp]
        lib.oracle_occluded.argtypes = [vp, i64, vp, vp, vp, i64, vp]
        lib.oracle_set_threads.argtypes = [ctypes.c_int]
        # every host thread, whatever OMP_NUM_THREADS a launcher exported
        lib.oracle_set_threads(int(os.environ.get("PS_ORACLE_THREADS", os.cpu_count() or 1)))
        _LIB = lib
    return _LIB


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def raycast(tris: np.ndarray, origins: np.ndarray, dirs: np.ndarray):
    """Nearest hit (t, prim) per ray, float64 brute force; prim -1 = miss."""
    tris = np.ascontiguousarray(tris, np.float64)
    o = np.ascontiguousarray(np.broadcast_to(origins, dirs.shape), np.float64)
    d = np.ascontiguousarray(dirs, np.float64)
    n = len(d)
    t = np.empty(n, np.float64)
    prim = np.empty(n, np.int64)
    _lib().oracle_raycast(_p(tris), len(tris), _p(o), _p(d), n, _p(t), _p(prim))
    return t, prim


def occluded(tris, origins, dirs, tmax):
    tris = np.ascontiguousarray(tris, np.float64)
    o = np.ascontiguousarray(origins, np.float64)
    d = np.ascontiguousarray(dirs, np.float64)
    tm = np.ascontiguousarray(tmax, np.float64)
    out = np.empty(len(d), np.uint8)
    _lib().oracle_occluded(_p(tris), len(tris), _p(o), _p(d), _p(tm), len(d), _p(out))
    return out.astype(bool)


# --- ray set ---------------------------------------------------------------------------


def fibonacci_sphere(n: int) -> np.ndarray:
    k = np.arange(n, dtype=np.float64) + 0.5
    z = 1.0 - 2.0 * k / n
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    phi = np.pi * (1.0 + np.sqrt(5.0)) * k
    return np.column_stack([r * np.cos(phi), r * np.sin(phi), z])


def oct_uv(d: np.ndarray) -> np.ndarray:
    """volume.py:262-283 without validation."""
    d = d / np.linalg.norm(d, axis=1, keepdims=True)
    l1 = np.abs(d).sum(axis=1)
    p = d[:, :2] / l1[:, None]
    sgn = np.where(p >= 0.0, 1.0, -1.0)
    folded = (1.0 - np.abs(p[:, ::-1])) * sgn
    p = np.where(d[:, 2:3] < 0.0, folded, p)
    return p * 0.5 + 0.5


def texel_directions(side: int) -> np.ndarray:
    c = (np.arange(side) + 0.5) / side
    uu, vv = np.meshgrid(c, c, indexing="xy")
    f = np.stack([uu, vv], -1).reshape(-1, 2) * 2.0 - 1.0
    z = 1.0 - np.abs(f[:, 0]) - np.abs(f[:, 1])
    sgn = np.where(f >= 0.0, 1.0, -1.0)
    xy = np.where((z < 0.0)[:, None], (1.0 - np.abs(f[:, ::-1])) * sgn, f)
    d = np.column_stack([xy, z])
    return d / np.linalg.norm(d, axis=1, keepdims=True)


def coherence_order(dirs: np.ndarray) -> np.ndarray:
    """Permutation sorting directions by the Morton code of their 10-bit
    octahedral uv (stable)."""
    q = np.clip(np.floor(oct_uv(dirs) * 1024.0).astype(np.int64), 0, 1023)
    code = np.zeros(len(dirs), np.int64)
    for bit in range(10):
        code |= ((q[:, 0] >> bit) & 1) << (2 * bit)
        code |= ((q[:, 1] >> bit) & 1) << (2 * bit + 1)
    return np.argsort(code, kind="stable")


def rotation(seed: int, frame: int) -> np.ndarray:
    w, x, y, z = (lambda q: q / np.linalg.norm(q))(np.random.default_rng(seed + frame).normal(size=4))
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


def ray_table(count: int, seed: int, frame: int) -> np.ndarray:
    base = fibonacci_sphere(count)
    base = base[coherence_order(base)]
    return (rotation(seed, frame) @ base.T).T.astype(np.float32)


# --- shading (float64, given hits) --------------------------------------------------------


def shadow_map_dirs(S: int) -> np.ndarray:
    """(6, S, S, 3) texel directions of a cube distance map, float32 as the
    device computes them: face f looks along axis f//2 (negative if f odd),
    texel (j, i) adds u_i on axis (a+1)%3 and w_j on axis (a+2)%3."""
    c = ((np.arange(S, dtype=np.float32) + np.float32(0.5)) / np.float32(S)) * np.float32(2) - np.float32(1)
    out = np.zeros((6, S, S, 3), np.float32)
    for f in range(6):
        a = f // 2
        out[f, :, :, a] = np.float32(-1.0 if f % 2 else 1.0)
        out[f, :, :, (a + 1) % 3] = c[None, :]
        out[f, :, :, (a + 2) % 3] = c[:, None]
    norm = np.sqrt(np.sum(out.astype(np.float64) ** 2, axis=-1, keepdims=True))
    return (out / norm).astype(np.float32)


def shadow_maps(tris, lights, S: int) -> np.ndarray:
    """(L, 6, S, S) nearest-hit distance from each light (inf on a miss)."""
    d = shadow_map_dirs(S).reshape(-1, 3).astype(np.float64)
    maps = []
    for lp, _ in lights:
        t, _prim = raycast(tris, np.asarray(lp, np.float64)[None, :], d)
        maps.append(t.reshape(6, S, S))
    return np.stack(maps) if maps else np.zeros((0, 6, S, S))


def cube_lookup(maps_l, v, S):
    """Map value for light-to-point vectors v (n, 3) of one light."""
    av = np.abs(v)
    a = np.where((av[:, 0] >= av[:, 1]) & (av[:, 0] >= av[:, 2]), 0,
                 np.where(av[:, 1] >= av[:, 2], 1, 2))
    rows = np.arange(len(v))
    m = av[rows, a]
    sgn = v[rows, a]
    u = v[rows, (a + 1) % 3] / m
    w = v[rows, (a + 2) % 3] / m
    f = 2 * a + (sgn < 0)
    i = np.clip(np.floor((u * 0.5 + 0.5) * S).astype(np.int64), 0, S - 1)
    j = np.clip(np.floor((w * 0.5 + 0.5) * S).astype(np.int64), 0, S - 1)
    return maps_l[f, j, i]


def shade(tris, albedo, emission, lights, sky, origins, dirs, t, prim, max_distance, bias,
          shadows="rays", shadow_map_size=256, shadow_bias=0.02, maps=None):
    """Radiance and depth per ray, float64; returns (rgb (n,3), depth (n,), mask).

    shadows: "rays" (exact shadow ray), "map" (cube distance maps from the
    lights, see shadow_map_dirs), "none"."""
    if shadows is True:
        shadows = "rays"
    elif not shadows:
        shadows = "none"
    if shadows == "map" and maps is None:
        maps = shadow_maps(tris, lights, shadow_map_size)
    n = len(dirs)
    rgb = np.tile(np.asarray(sky, np.float64), (n, 1))
    depth = np.full(n, float(max_distance))
    mask = np.zeros(n, np.int64)
    hit = prim >= 0
    if not hit.any():
        return rgb, depth, mask
    v = np.asarray(tris, np.float64)
    nrm = np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0])
    nrm = nrm / np.maximum(np.linalg.norm(nrm, axis=1, keepdims=True), 1e-30)
    nrm = nrm.astype(np.float32).astype(np.float64)  # the device table holds float normals
    idx = np.nonzero(hit)[0]
    pid = prim[idx]
    o, d, th = origins[idx], dirs[idx], t[idx]
    nn = nrm[pid]
    nn = np.where((np.sum(nn * d, axis=1) > 0)[:, None], -nn, nn)
    x = o + d * th[:, None]
    s = x + bias * nn
    acc = np.zeros((len(idx), 3))
    for li, (lp, li_rgb) in enumerate(lights):
        lv = np.asarray(lp, np.float64) - s
        d2 = np.sum(lv * lv, axis=1)
        dist = np.sqrt(d2)
        u = lv / dist[:, None]
        cos = np.sum(nn * u, axis=1)
        ok = (d2 > 0) & (cos > 0)
        if shadows == "rays" and ok.any():
            blocked = occluded(tris, s[ok], u[ok], dist[ok])
            vis = ok.copy()
            vis[np.nonzero(ok)[0][blocked]] = False
        elif shadows == "map" and ok.any():
            dm = cube_lookup(maps[li], s - np.asarray(lp, np.float64), shadow_map_size)
            vis = ok & (dist <= dm * (1.0 + shadow_bias))
        else:
            vis = ok
        mask[idx[vis]] |= 1 << li
        acc += np.where(vis, cos / np.where(d2 > 0, d2, 1.0), 0.0)[:, None] * np.asarray(li_rgb, np.float64)
    rgb[idx] = np.asarray(emission, np.float64)[pid] + np.asarray(albedo, np.float64)[pid] * acc
    depth[idx] = np.minimum(th, max_distance)
    return rgb, depth, mask


# --- blend (float32) ----------------------------------------------------------------------


def _fma32(a, b, c):
    """float32 fma(a, b, c): the float32 product is exact in float64 and the
    sum is rounded once more to float32 (double rounding can differ from a
    true fma only when the float64 sum is itself inexact, which needs
    exponent gaps > 29 bits -- never for unit vectors' components here)."""
    return (a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)).astype(np.float32)


def texel_cosines(dirs32: np.ndarray):
    """float32 max(0, n_t . d_r) for the 64 colour / 256 depth texels (rows)
    and the R rays (columns), evaluated in the device's order
    ``fma(az, bz, fma(ay, by, ax * bx))`` (csrc/ps_common.cuh dot3)."""
    out = []
    d = np.asarray(dirs32, np.float32)[:, :3]
    for side in (8, 16):
        n = texel_directions(side).astype(np.float32)
        ax, ay, az = (n[:, i][:, None] for i in range(3))
        bx, by, bz = (d[:, i][None, :] for i in range(3))
        c = _fma32(az, bz, _fma32(ay, by, (ax * bx).astype(np.float32)))
        out.append(np.maximum(c, np.float32(0)))
    return out


def blend_weights(dirs32: np.ndarray, sharpness: float):
    """(Wc (64,R), Wd (256,R), inv_c (64,), inv_d (256,)) in float32.

    Plain float32 weights (no tf32 rounding): colour ``max(0, n_t . d_r)``,
    depth that cosine to the power ``sharpness`` (evaluated in float64 from
    the float32 cosine, rounded once); inv = 1 / sum over rays in float32."""
    wc, cd = texel_cosines(dirs32)
    wd = np.power(cd.astype(np.float64), np.float64(np.float32(sharpness))).astype(np.float32)
    return weights_from(wc, wd)


def weights_from(wc: np.ndarray, wd: np.ndarray):
    """The blend_weights tuple for given (64,R) / (256,R) float32 weights;
    the weight sums are exact-then-rounded (float64), inv = float32 1 / sum."""
    inv = []
    for w in (wc, wd):
        s = w.astype(np.float64).sum(axis=1).astype(np.float32)
        with np.errstate(divide="ignore"):
            inv.append(np.where(s > 0, np.float32(1) / s, np.float32(0)).astype(np.float32))
    return wc, wd, inv[0], inv[1]


def check_device_weights(w_color_dev: np.ndarray, w_depth_dev: np.ndarray, dirs32, sharpness):
    """Device weight tables ((R,64), (R,256)) against blend_weights at float32
    ulps: colour within 2 ulp (same fma order), depth within 8 ulp (CUDA
    powf is not correctly rounded).  Returns the ORACLE's own weights, so the
    blend is checked against weights the device did not produce."""
    ref = blend_weights(dirs32, sharpness)
    wc, wd = np.ascontiguousarray(w_color_dev.T), np.ascontiguousarray(w_depth_dev.T)
    for a, b, ulps in ((wc, ref[0], 2), (wd, ref[1], 8)):
        assert a.dtype == np.float32 and a.shape == b.shape
        tol = ulps * np.spacing(np.maximum(np.abs(b), np.float32(np.finfo(np.float32).tiny)))
        bad = np.abs(a.astype(np.float64) - b.astype(np.float64)) > tol
        assert not bad.any(), (f"{bad.sum()} device weights differ from the oracle by more than "
                               f"{ulps} ulp (max |diff| {np.abs(a - b).max():.3g})")
    return ref


def blend(rgb32, depth32, weights, prev_irr, prev_mom, hysteresis):
    """rgb32 (P,R,3), depth32 (P,R) float32 -> new (irr (P,64,3), mom (P,256,2)).

    The weighted ray sums are accumulated in float64 and rounded once to
    float32 (the device's 3xTF32 tensor-core sums are fp32-accurate), then
    scaled by the float32 1 / sum of weights, then blended with the previous
    state in float32: state = fma(h, prev - frame, frame), as the device."""
    wc, wd, inv_c, inv_d = weights
    rgb = np.asarray(rgb32, np.float32).astype(np.float64)
    if prev_irr is None:
        prev_irr = np.zeros((rgb.shape[0], 64, 3), np.float32)
    if prev_mom is None:
        prev_mom = np.zeros((rgb.shape[0], 256, 2), np.float32)
    dep32 = np.asarray(depth32, np.float32)
    dep = dep32.astype(np.float64)
    dep2 = (dep32 * dep32).astype(np.float64)  # d^2 is formed in float32 on the device
    wc64, wd64 = wc.astype(np.float64), wd.astype(np.float64)
    irr = np.einsum("tr,prc->ptc", wc64, rgb).astype(np.float32) * inv_c[None, :, None]
    m1 = np.einsum("tr,pr->pt", wd64, dep).astype(np.float32) * inv_d[None, :]
    m2 = np.einsum("tr,pr->pt", wd64, dep2).astype(np.float32) * inv_d[None, :]
    mom = np.stack([m1, m2], -1).astype(np.float32)
    h = np.float32(hysteresis)
    if h != 0:
        prev_irr = np.asarray(prev_irr, np.float32)
        prev_mom = np.asarray(prev_mom, np.float32)
        irr = _fma32(h, (prev_irr - irr).astype(np.float32), irr)
        mom = _fma32(h, (prev_mom - mom).astype(np.float32), mom)
    irr = np.where((inv_c == 0)[None, :, None], prev_irr, irr)
    mom = np.where((inv_d == 0)[None, :, None], prev_mom, mom)
    return irr.astype(np.float32), mom.astype(np.float32)


def blend_f64(rgb32, depth32, weights, prev_irr, prev_mom, hysteresis):
    """The same blend entirely in float64 (test of the oracle's accuracy)."""
    wc, wd = (np.asarray(w, np.float64) for w in weights[:2])
    rgb = np.asarray(rgb32, np.float32).astype(np.float64)
    dep = np.asarray(depth32, np.float32).astype(np.float64)
    sc, sd = wc.sum(1), wd.sum(1)
    with np.errstate(divide="ignore", invalid="ignore"):
        irr = np.einsum("tr,prc->ptc", wc, rgb) / sc[None, :, None]
        m1 = np.einsum("tr,pr->pt", wd, dep) / sd[None, :]
        m2 = np.einsum("tr,pr->pt", wd, dep * dep) / sd[None, :]
    mom = np.stack([m1, m2], -1)
    pi = np.zeros(irr.shape) if prev_irr is None else np.asarray(prev_irr, np.float64)
    pm = np.zeros(mom.shape) if prev_mom is None else np.asarray(prev_mom, np.float64)
    irr = irr + hysteresis * (pi - irr)
    mom = mom + hysteresis * (pm - mom)
    irr = np.where((sc == 0)[None, :, None], pi, irr)
    mom = np.where((sd == 0)[None, :, None], pm, mom)
    return irr, mom


# --- quantisation + guard band (bit-exact given the float state) ---------------------------


def quantize_color(irr32: np.ndarray, scale: float) -> np.ndarray:
    """(P,64,3) float32 -> (P,8,8) uint32 r | g<<10 | b<<20 (volume.py:226)."""
    qs = np.float32(1) / np.float32(scale) if scale > 0 else np.float32(0)
    x = np.clip(irr32.astype(np.float32) * qs, np.float32(0), np.float32(1))
    q = np.rint(x * np.float32(1023)).astype(np.uint32)
    t = q[..., 0] | (q[..., 1] << np.uint32(10)) | (q[..., 2] << np.uint32(20))
    return t.reshape(-1, 8, 8)


def quantize_moments(mom32: np.ndarray) -> np.ndarray:
    """(P,256,2) float32 -> (P,16,16,2) uint16 raw half bits."""
    return mom32.astype(np.float16).view(np.uint16).reshape(-1, 16, 16, 2)


def write_blocks(atlas: np.ndarray, kind: str, ppr: int, probe_ids, cores) -> None:
    side = so.BLOCK_SIDE[kind]
    for p, core in zip(probe_ids, cores):
        br, bc = divmod(int(p), ppr)
        atlas[br * side:(br + 1) * side, bc * side:(bc + 1) * side] = so.guard_band_block(core)
