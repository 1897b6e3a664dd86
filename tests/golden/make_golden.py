"""Generate golden vectors by running the REFERENCE implementation.

Run here (the container that has /root/reference):

    python tests/golden/make_golden.py

The reference is imported from ``$PROBESTREAM_REF`` (default
``/root/reference/pkg/src``).  Outputs are small ``.npz`` files next to this
script; they are committed so that the GPU box (which has no reference
mount) can check parity against the reference's own outputs.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = os.environ.get("PROBESTREAM_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from probestream import codec as rcodec  # noqa: E402
from probestream import packing as rpack  # noqa: E402
from probestream import selection as rsel  # noqa: E402
from probestream import varint as rvarint  # noqa: E402
from probestream import volume as rvol  # noqa: E402

OUT = Path(__file__).resolve().parent


def save(name, **arrays):
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print(f"wrote {name}.npz ({sum(a.nbytes for a in arrays.values())} raw bytes)")


# --- packing ------------------------------------------------------------------


def gen_pack():
    rng = np.random.default_rng(101)
    color = rng.integers(0, 2**32, size=(37, 53), dtype=np.uint32)
    color[0, 0] = 1023 | (0 << 10) | (512 << 20)  # test_packing.py:40-45 KAT
    color[0, 1] = (3 << 30) | 7                   # alpha dropped, :65-67
    cplanes = rpack.pack_color(color).data
    vis = rng.integers(0, 2**16, size=(13, 29, 2), dtype=np.uint16)
    vis[0, 0] = (0xFFFF, 0xFFFF)
    vis[1, 1] = (0x7FFF, 0x8000)  # NaN payload / signed zero (:100-107)
    vplanes = rpack.pack_visibility(vis).data
    arrays = dict(color=color, color_planes=cplanes, vis=vis, vis_planes=vplanes)
    # every width 1..13 (all residues of 4w mod 3), two rows each
    for w in range(1, 14):
        t = rng.integers(0, 2**16, size=(2, w, 2), dtype=np.uint16)
        arrays[f"vis_w{w}"] = t
        arrays[f"vis_w{w}_planes"] = rpack.pack_visibility(t).data
    kat = np.tile(np.array([[0x1234, 0xABCD]], dtype=np.uint16), (1, 3)).reshape(1, 3, 2)
    arrays["kat3"] = kat
    arrays["kat3_planes"] = rpack.pack_visibility(kat).data
    save("pack", **arrays)


# --- guard band ----------------------------------------------------------------


def gen_guard():
    rng = np.random.default_rng(102)
    core8 = rng.integers(0, 2**30, size=(8, 8), dtype=np.uint32)
    core16 = rng.integers(0, 2**16, size=(16, 16, 2), dtype=np.uint16)
    core4 = np.arange(16, dtype=np.uint32).reshape(4, 4)
    save(
        "guard",
        core8=core8, block10=rpack.reconstruct_guard_band(core8),
        core16=core16, block18=rpack.reconstruct_guard_band(core16),
        core4=core4, block6=rpack.reconstruct_guard_band(core4),
    )


# --- change detection -----------------------------------------------------------

DETECT_THRESHOLDS = [0.0, -1.0, 0.25, 1.0, 2.5, 7.0, 1023.0, 5000.0, float("nan"),
                     1e-3, 1e-2, 0.5, 1e-50, float("inf")]


def _edge_case_atlases(kind, n, ppr, rng):
    atlas = rvol.ProbeAtlas(kind, n, probes_per_row=ppr)
    if kind is rvol.AtlasKind.COLOR:
        atlas.texels[:] = rng.integers(0, 2**30, size=atlas.texels.shape, dtype=np.uint32)
    else:
        atlas.texels[:] = rng.integers(0, 0x7C00, size=atlas.texels.shape, dtype=np.uint16)
    last = atlas.copy()
    side = kind.block_side
    t = last.texels
    # random mutations on a subset of probes (core texels)
    for p in rng.choice(n, size=n // 5, replace=False):
        y, x = last.block_origin(int(p))
        yy, xx = y + 1 + rng.integers(0, side - 2), x + 1 + rng.integers(0, side - 2)
        if kind is rvol.AtlasKind.COLOR:
            t[yy, xx] ^= np.uint32(1 << int(rng.integers(0, 30)))
        else:
            t[yy, xx, int(rng.integers(0, 2))] ^= np.uint16(1 << int(rng.integers(0, 15)))
    specials = {}
    # guard-band-only difference marks the probe changed (exact path)
    y, x = last.block_origin(3)
    if kind is rvol.AtlasKind.COLOR:
        t[y, x + 4] ^= np.uint32(1)
        specials["guard_only"] = 3
        y, x = last.block_origin(4)
        t[y + 2, x + 2] ^= np.uint32(1 << 31)  # alpha bit only
        specials["alpha_only"] = 4
        y, x = last.block_origin(5)
        t[y + 2, x + 2] = (t[y + 2, x + 2] & ~np.uint32(0x3FF)) | np.uint32(
            (int(t[y + 2, x + 2]) & 0x3FF) ^ 0x3  # channel delta 1..3
        )
        y, x = last.block_origin(6)
        a = int(atlas.texels[y + 3, x + 3])
        r = a & 0x3FF
        t[y + 3, x + 3] = (a & ~0x3FF) | (r + 7 if r < 1000 else r - 7)  # delta exactly 7
        specials["delta7"] = 6
    else:
        t[y, x + 4, 0] ^= np.uint16(1)
        specials["guard_only"] = 3
        # +0 vs -0
        y, x = last.block_origin(4)
        atlas.texels[y + 2, x + 2, 0] = 0x0000
        t[y + 2, x + 2, 0] = 0x8000
        # identical NaN bits (unchanged) and differing NaN payloads (changed)
        y, x = last.block_origin(5)
        atlas.texels[y + 2, x + 2, 1] = 0x7E01
        t[y + 2, x + 2, 1] = 0x7E01
        y, x = last.block_origin(6)
        atlas.texels[y + 2, x + 2, 1] = 0x7E01
        t[y + 2, x + 2, 1] = 0x7E02
        # +inf vs +inf (unchanged), +inf vs -inf (changed), inf vs finite
        y, x = last.block_origin(7)
        atlas.texels[y + 2, x + 2, 0] = 0x7C00
        t[y + 2, x + 2, 0] = 0x7C00
        y, x = last.block_origin(8)
        atlas.texels[y + 2, x + 2, 0] = 0x7C00
        t[y + 2, x + 2, 0] = 0xFC00
        y, x = last.block_origin(9)
        atlas.texels[y + 2, x + 2, 0] = 0x7C00
        t[y + 2, x + 2, 0] = 0x3C00
        # NaN vs finite (delta NaN, bits differ -> changed)
        y, x = last.block_origin(10)
        atlas.texels[y + 2, x + 2, 1] = 0x7E00
        t[y + 2, x + 2, 1] = 0x3C00
        # a one-ulp change at 1.0: delta = 2^-10
        y, x = last.block_origin(11)
        atlas.texels[y + 2, x + 2, 0] = 0x3C00
        t[y + 2, x + 2, 0] = 0x3C01
    return atlas, last, specials


def gen_detect():
    rng = np.random.default_rng(103)
    arrays = {}
    for kind in (rvol.AtlasKind.COLOR, rvol.AtlasKind.VISIBILITY):
        for n, ppr in ((300, None), (77, 9), (260, None)):
            vol_active = rng.random(n) < 0.75
            vol_active[:12] = True
            vol = rvol.ProbeVolume((n, 1, 1), active=vol_active)
            atlas, last, _ = _edge_case_atlases(kind, n, ppr, rng)
            tag = f"{kind.value}_n{n}"
            arrays[f"{tag}_rendered"] = atlas.texels
            # stored as XOR against `rendered` so the archive compresses
            arrays[f"{tag}_last_xor"] = last.texels ^ atlas.texels
            arrays[f"{tag}_active"] = vol_active
            arrays[f"{tag}_ppr"] = np.int64(atlas.probes_per_row)
            for i, thr in enumerate(DETECT_THRESHOLDS):
                ids = rsel.detect_changed(atlas, last, vol, threshold=thr)
                arrays[f"{tag}_thr{i}"] = ids.astype(np.int64)
            # float32 rounding of a python-float threshold: delta = 2^-10,
            # threshold = delta - 1e-12 rounds up to delta in float32 -> NOT
            # changed
            thr = 2.0**-10 - 1e-12
            arrays[f"{tag}_thr_ulp"] = rsel.detect_changed(atlas, last, vol, threshold=thr)
            arrays[f"{tag}_thr_ulp64"] = rsel.detect_changed(
                atlas, last, vol, threshold=np.float64(thr))
    arrays["thresholds"] = np.array(DETECT_THRESHOLDS)
    # identical atlases -> empty; one texel of probe 7 -> [7]
    a = rvol.ProbeAtlas(rvol.AtlasKind.COLOR, 2048)
    kat_rng = np.random.default_rng(1103)  # regenerated by the tests from this seed
    a.texels[:] = kat_rng.integers(0, 2**30, size=a.texels.shape, dtype=np.uint32)
    b = a.copy()
    vol = rvol.ProbeVolume((16, 8, 16))
    arrays["kat_identical"] = rsel.detect_changed(a, b, vol)
    y, x = b.probe_core(7).shape
    b.probe_core(7)[2, 3] ^= np.uint32(1)
    arrays["kat_probe7"] = rsel.detect_changed(a, b, vol)
    arrays["kat2048_seed"] = np.int64(1103)
    save("detect", **arrays)


# --- selection --------------------------------------------------------------------


def gen_select():
    rng = np.random.default_rng(104)
    arrays = {}
    cases = []
    for case in range(12):
        n = int(rng.integers(20, 400))
        active = rng.random(n) < 0.8
        vol = rvol.ProbeVolume((n, 1, 1), active=active)
        changed = rng.choice(n, size=int(rng.integers(0, n)), replace=True)
        pvs = rng.choice(n, size=int(rng.integers(0, n)), replace=False)
        seq = rng.integers(-5, 30, size=n).astype(np.int64)
        if case % 3 == 0:
            seq[:] = 7  # all equally stale -> id order
        cur = int(rng.integers(30, 40))
        for bi, budget in enumerate([None, 0, 1, 5, -2, 10**6]):
            out = rsel.select_for_client(changed, pvs, vol, seq, cur, budget)
            arrays[f"c{case}_b{bi}"] = np.array(out, dtype=np.int64)
        arrays[f"c{case}_active"] = active
        arrays[f"c{case}_changed"] = changed.astype(np.int64)
        arrays[f"c{case}_pvs"] = pvs.astype(np.int64)
        arrays[f"c{case}_seq"] = seq
        arrays[f"c{case}_cur"] = np.int64(cur)
        cases.append(case)
    arrays["budgets"] = np.array([-1, 0, 1, 5, -2, 10**6])  # -1 encodes None
    arrays["ncases"] = np.int64(len(cases))
    # SPEC.md:298-301 KATs
    vol = rvol.ProbeVolume((16, 1, 1))
    arrays["kat_a"] = np.array(rsel.select_for_client([1, 2], [2, 3], vol, np.zeros(16, int), 5))
    arrays["kat_b"] = np.array(rsel.select_for_client([4, 9], [4, 9], vol, np.zeros(16, int), 5, budget=1))
    save("select", **arrays)


# --- slot cache + update atlas --------------------------------------------------


def gen_slots():
    rng = np.random.default_rng(105)
    arrays = {}
    for kind in (rvol.AtlasKind.COLOR, rvol.AtlasKind.VISIBILITY):
        n = 60
        src = rvol.ProbeAtlas(kind, n, probes_per_row=7)
        if kind is rvol.AtlasKind.COLOR:
            src.texels[:] = rng.integers(0, 2**32, size=src.texels.shape, dtype=np.uint32)
        else:
            src.texels[:] = rng.integers(0, 2**16, size=src.texels.shape, dtype=np.uint16)
        src0 = src.texels.copy()
        slot_count = 17
        layout = rpack.UpdateAtlasLayout(slot_count, kind.core_side, slots_per_row=5)
        texels = None
        steps = 25
        for step in range(steps):
            k = int(rng.integers(0, slot_count + 1))
            sel = rng.choice(n, size=k, replace=False)
            if step % 4 == 1:  # duplicates and unsorted input
                sel = np.concatenate([sel, sel[: k // 2]])
            # mutate the source between steps so slot contents are traceable
            row = int(rng.integers(0, src.texels.shape[0]))
            if kind is rvol.AtlasKind.COLOR:
                src.texels[row, :] ^= np.uint32(step + 1)
            else:
                src.texels[row, :, 0] ^= np.uint16(step + 1)
            arrays[f"{kind.value}_s{step}_row"] = np.int64(row)
            texels, entries = rpack.build_update_atlas(sel, layout, src, texels)
            arrays[f"{kind.value}_s{step}_sel"] = np.asarray(sel, dtype=np.int64)
            arrays[f"{kind.value}_s{step}_entries"] = np.array(entries, dtype=np.int64).reshape(-1, 2)
            if step % 6 == 5 or step == steps - 1:
                arrays[f"{kind.value}_s{step}_texels"] = texels.copy()
            ps = np.full(n, -1, np.int64)
            for p, s in layout.probe_slot.items():
                ps[p] = s
            arrays[f"{kind.value}_s{step}_probe_slot"] = ps
        arrays[f"{kind.value}_steps"] = np.int64(steps)
        arrays[f"{kind.value}_src0"] = src0
        arrays[f"{kind.value}_ppr"] = np.int64(7)
    # overflow raises before mutation
    layout = rpack.UpdateAtlasLayout(2, 8)
    try:
        layout.assign([1, 2, 3])
        arrays["overflow_raised"] = np.int64(0)
    except rpack.SlotOverflowError:
        arrays["overflow_raised"] = np.int64(1)
    save("slots", **arrays)


# --- temporal delta via the codec -------------------------------------------------


def _parse_modes(payload: bytes, planes: int, h: int, w: int):
    """Walk an LPF1 P-frame payload and return the per-block mode bytes."""
    pos = 0
    by, bx = -(-h // 16), -(-w // 16)
    modes = np.zeros((planes, by, bx), np.uint8)
    for p in range(planes):
        for j in range(by):
            for i in range(bx):
                m = payload[pos]
                pos += 1
                modes[p, j, i] = m
                if m != rcodec.MODE_SKIP:
                    length, pos = rvarint.decode_uvarint(payload, pos)
                    pos += length
    assert pos == len(payload)
    return modes


def _residual_via_codec(cur, prev):
    """Residual as the reference codec defines it: decode its own DELTA
    payload back to signed values (codec.py:211-224)."""
    out = np.empty(cur.shape, np.int64)
    for p in range(cur.shape[0]):
        blob = rcodec._encode_delta(cur[p], prev[p])
        stream = rcodec.entropy_decode(blob)
        vals, _ = rvarint.decode_uvarint_array(stream, cur[p].size)
        out[p] = rvarint.unzigzag(vals).reshape(cur[p].shape)
    return out


def gen_delta():
    rng = np.random.default_rng(106)
    arrays = {}
    for kind, dtype, hi in ((rpack.PlaneKind.COLOR_10IN16, np.uint16, 1024),
                            (rpack.PlaneKind.VISIBILITY_BYTES, np.uint8, 256)):
        h, w = 45, 70  # clipped edge blocks in both axes
        prev = rng.integers(0, hi, size=(3, h, w), dtype=dtype)
        cur = prev.copy()
        # mutate a few scattered elements so most blocks stay SKIP
        for _ in range(9):
            p, y, x = rng.integers(0, 3), rng.integers(0, h), rng.integers(0, w)
            cur[p, y, x] = (int(cur[p, y, x]) + int(rng.integers(1, hi))) % hi
        enc = rcodec.CodecStreamState(1, role="encoder", gop_length=30)
        rcodec.encode_frame(rpack.PlaneSet(kind, prev.copy()), enc)
        frame = rcodec.encode_frame(rpack.PlaneSet(kind, cur.copy()), enc)
        assert not frame.key
        modes = _parse_modes(frame.payload, 3, h, w)
        tag = "color" if dtype == np.uint16 else "vis"
        arrays[f"{tag}_prev"] = prev
        arrays[f"{tag}_cur"] = cur
        arrays[f"{tag}_skip"] = (modes == rcodec.MODE_SKIP).astype(np.uint8)
        arrays[f"{tag}_residual"] = _residual_via_codec(cur, prev)
    save("delta", **arrays)


# --- directions, fibonacci sphere, raycast ---------------------------------------


def gen_geometry():
    rng = np.random.default_rng(107)
    arrays = {
        "texdir8": rvol.texel_directions(8),
        "texdir16": rvol.texel_directions(16),
        "fib64": rsel.fibonacci_sphere(64),
        "fib256": rsel.fibonacci_sphere(256),
    }
    # a small triangle soup + rays from a few origins, incl. grazing edges
    tris = rng.uniform(-1, 1, size=(40, 3, 3))
    # a shared edge pair (two triangles of a quad) to exercise edge rules
    tris[0] = [[-0.5, -0.5, 0.3], [0.5, -0.5, 0.3], [0.5, 0.5, 0.3]]
    tris[1] = [[-0.5, -0.5, 0.3], [0.5, 0.5, 0.3], [-0.5, 0.5, 0.3]]
    scene = rsel.SceneGeometry(None, tris)
    origins = rng.uniform(-0.3, 0.3, size=(6, 3))
    dirs = rsel.fibonacci_sphere(200)
    ray_o = np.repeat(origins, len(dirs), axis=0)
    ray_d = np.tile(dirs, (len(origins), 1))
    # rays straight down onto the quad diagonal
    extra_o = np.array([[0.0, 0.0, 1.0], [0.25, 0.25, 1.0], [-0.5, -0.5, 1.0]])
    extra_d = np.array([[0.0, 0.0, -1.0]] * 3)
    ray_o = np.concatenate([ray_o, extra_o])
    ray_d = np.concatenate([ray_d, extra_d])
    hit, t, pts, nrm = scene.raycast(ray_o, ray_d)
    arrays.update(tris=tris, ray_o=ray_o, ray_d=ray_d, hit=hit, t=t, normal=nrm)
    save("geometry", **arrays)


def gen_pvs():
    """pvs_probes on triangle scenes (selection.py:384-407) with the frustum +
    fibonacci ray set, plus cage_probes on random points."""
    sys.path.insert(0, str(OUT.parents[1]))
    from paper_2103_05875_b200 import scene as S  # geometry construction only

    rng = np.random.default_rng(108)
    arrays = {}
    scenes = {"cornell": (S.cornell_box(), (8, 8, 8)),
              "hall": (S.interior_hall(detail=0.12), (16, 8, 16))}
    case = 0
    for name, (sc, dims) in scenes.items():
        vol_ours = S.volume_for(sc, dims)
        active = rng.random(int(np.prod(dims))) < 0.85
        vol = rvol.ProbeVolume(dims, vol_ours.origin, vol_ours.spacing, active=active)
        geo = rsel.SceneGeometry(None, sc.vertices)
        (x0, y0, z0), (x1, y1, z1) = sc.bounds
        for k in range(4):
            pos = np.array([x0, y0, z0]) + rng.random(3) * (np.array([x1, y1, z1]) - np.array([x0, y0, z0]))
            fwd = rng.normal(size=3)
            pose = rsel.CameraPose(pos, fwd, fov_y_deg=float(rng.uniform(50, 100)),
                                   aspect=float(rng.uniform(1.0, 1.8)))
            params = rsel.SelectionParams(raster_cols=24, raster_rows=16, sphere_rays=300)
            rays = rsel.pvs_rays(pose, params)
            ids = rsel.pvs_probes(pose, geo, vol, params)
            arrays[f"c{case}_tris"] = sc.vertices if k == 0 else np.zeros(0)
            arrays[f"c{case}_scene"] = np.array(name)
            arrays[f"c{case}_dims"] = np.array(dims)
            arrays[f"c{case}_origin"] = np.array(vol.origin)
            arrays[f"c{case}_spacing"] = np.array(vol.spacing)
            arrays[f"c{case}_active"] = active
            arrays[f"c{case}_pose"] = np.concatenate([pose.position, fwd, pose.up,
                                                      [pose.fov_y_deg, pose.aspect]])
            arrays[f"c{case}_rays"] = rays
            arrays[f"c{case}_ids"] = ids.astype(np.int64)
            case += 1
    arrays["ncases"] = np.int64(case)
    # cage_probes on random points incl. outside the volume (clamping)
    vol = rvol.ProbeVolume((5, 4, 3), (0.5, -1.0, 2.0), (0.7, 1.1, 0.9))
    pts = rng.uniform(-3, 8, size=(500, 3))
    arrays["cage_points"] = pts
    arrays["cage_ids"] = rsel.cage_probes(pts, vol)
    save("pvs", **{k: v for k, v in arrays.items() if not (k.endswith("_tris") and v.size == 0)})


def gen_codec():
    """encode_frame byte streams (codec.py:335-366) over short sequences of
    colour and visibility plane sets: key frames with intra prediction,
    P-frames with SKIP / DELTA / RAW blocks, clipped edge blocks, zero runs."""
    rng = np.random.default_rng(109)
    arrays = {}
    seqs = 0
    for kind, dtype, hi, shape in ((rpack.PlaneKind.COLOR_10IN16, np.uint16, 1024, (3, 37, 53)),
                                   (rpack.PlaneKind.VISIBILITY_BYTES, np.uint8, 256, (3, 45, 70)),
                                   (rpack.PlaneKind.COLOR_10IN16, np.uint16, 1024, (3, 64, 64)),
                                   (rpack.PlaneKind.VISIBILITY_BYTES, np.uint8, 256, (3, 16, 16))):
        enc = rcodec.CodecStreamState(seqs + 1, role="encoder", gop_length=4)
        # smooth-ish content so DELTA wins somewhere, plus zero areas for runs
        base = (np.add.outer(np.arange(shape[1]), np.arange(shape[2])) % hi).astype(dtype)
        cur = np.stack([base, (base // 3).astype(dtype), np.zeros_like(base)])
        cur[2, : shape[1] // 2] = rng.integers(0, hi, size=(shape[1] // 2, shape[2]), dtype=dtype)
        frames = []
        for f in range(6):
            if f > 0:
                m = rng.random(shape) < (0.02 if f % 2 else 0.3)
                cur = cur.copy()
                cur[m] = ((cur[m].astype(np.int64) + rng.integers(1, 5, size=int(m.sum()))) % hi).astype(dtype)
                if f == 3:
                    cur[1, :16, :16] = 0  # zero runs
            frame = rcodec.encode_frame(rpack.PlaneSet(kind, cur.copy()), enc, force_key=(f == 5))
            arrays[f"s{seqs}_f{f}_planes"] = cur.copy()
            arrays[f"s{seqs}_f{f}_bytes"] = np.frombuffer(frame.to_bytes(), np.uint8)
            arrays[f"s{seqs}_f{f}_key"] = np.int64(frame.key)
        arrays[f"s{seqs}_frames"] = np.int64(6)
        arrays[f"s{seqs}_gop"] = np.int64(4)
        arrays[f"s{seqs}_stream"] = np.int64(seqs + 1)
        seqs += 1
    arrays["nseq"] = np.int64(seqs)
    # entropy coder KATs
    for i, data in enumerate([b"", b"\x00" * 4096, b"\x01\x00\x02\x00\x03", bytes(range(256)) * 3,
                              b"\x00\x00\x05" * 100]):
        arrays[f"ent{i}_in"] = np.frombuffer(data, np.uint8)
        arrays[f"ent{i}_out"] = np.frombuffer(rcodec.entropy_encode(data), np.uint8)
    arrays["nent"] = np.int64(5)
    save("codec", **arrays)


def _ref_index_buffer(entries):
    """SPEC.md:355-362 composed from the reference's own varint primitives
    (varint.py:16-19 zigzag, :27-38 encode_uvarint): count, then per entry
    the slot delta and the zig-zagged probe delta (both from 0)."""
    out = bytearray(rvarint.encode_uvarint(len(entries)))
    ps = pp = 0
    for slot, probe in entries:
        out += rvarint.encode_uvarint(slot - ps)
        out += rvarint.encode_uvarint(int(rvarint.zigzag(np.array([probe - pp]))[0]))
        ps, pp = slot, probe
    return bytes(out)


def gen_index():
    """Index buffers (§8(f)4) built from the reference's varint / zig-zag, and
    the primitives themselves on edge values."""
    rng = np.random.default_rng(113)
    arrays = {}
    lists = [[], [(0, 5), (1, 9)], [(i, 1000 + i) for i in range(400)],
             [(0, 131071), (1, 0), (7, 65536), (300, 65535)]]
    for n in (1, 17, 130, 4096):
        slots = np.sort(rng.choice(10 * n, size=n, replace=False))
        lists.append(list(zip(slots.tolist(), rng.integers(0, 131072, size=n).tolist())))
    for i, e in enumerate(lists):
        arrays[f"e{i}"] = np.asarray(e, np.int64).reshape(-1, 2)
        arrays[f"b{i}"] = np.frombuffer(_ref_index_buffer(e), np.uint8)
    arrays["n"] = np.int64(len(lists))
    vals = np.array([0, 1, -1, 63, -64, 64, -65, 8191, -8192, 2**31 - 1, -2**31, 2**40, -2**40],
                    np.int64)
    arrays["zz_in"] = vals
    arrays["zz_out"] = rvarint.zigzag(vals)
    uv = [0, 1, 127, 128, 255, 300, 16383, 16384, 2**21, 2**28 - 1, 2**35, 2**56 + 3]
    arrays["uv_in"] = np.array(uv, np.uint64)
    blob = b"".join(rvarint.encode_uvarint(v) for v in uv)
    arrays["uv_lens"] = np.array([len(rvarint.encode_uvarint(v)) for v in uv], np.int64)
    arrays["uv_out"] = np.frombuffer(blob, np.uint8)
    save("index", **arrays)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()[f"gen_{name}"]()
        sys.exit(0)
    gen_index()
    gen_codec()
    gen_pvs()
    gen_pack()
    gen_guard()
    gen_detect()
    gen_select()
    gen_slots()
    gen_delta()
    gen_geometry()
