"""numpy restatement of the reference's bit-exact stream operations.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__``).  Each function names the
reference lines it restates; the restatements are written independently of
the reference code (different decomposition, same arithmetic) and are pinned
against fixtures the reference itself produced (``tests/golden``).

Atlas conventions (``volume.py:147-218``): one block of ``side x side``
texels per probe, row-major by probe id with ``probes_per_row`` blocks per
atlas row; colour texels are ``uint32 (H, W)``, visibility texels are raw
half bits ``uint16 (H, W, 2)``.
"""

from __future__ import annotations

import math

import numpy as np

COLOR, VISIBILITY = "color", "visibility"
BLOCK_SIDE = {COLOR: 10, VISIBILITY: 18}
CODEC_BLOCK = 16  # codec.py:35


def block_side(kind: str) -> int:
    return BLOCK_SIDE[kind]


def default_probes_per_row(n: int) -> int:
    # volume.py:61-65
    return 16 if n <= 256 else math.ceil(math.sqrt(n))


def atlas_shape(kind: str, n: int, ppr: int) -> tuple:
    # volume.py:168-176
    side = BLOCK_SIDE[kind]
    rows = -(-n // ppr)
    shape = (rows * side, ppr * side)
    return shape if kind == COLOR else shape + (2,)


def blocks_by_probe(texels: np.ndarray, kind: str, ppr: int) -> np.ndarray:
    """(probe, side, side[, 2]) array in probe order, padding blocks included.

    Restates ``selection._per_probe_blocks`` (selection.py:273-281) by
    explicit block slicing instead of a reshape/transpose view.
    """
    side = BLOCK_SIDE[kind]
    rows = texels.shape[0] // side
    out = np.empty((rows * ppr, side, side) + texels.shape[2:], texels.dtype)
    for br in range(rows):
        band = texels[br * side:(br + 1) * side]
        for bc in range(ppr):
            out[br * ppr + bc] = band[:, bc * side:(bc + 1) * side]
    return out


# --- stage (3): change detection -------------------------------------------


def detect_changed(rendered: np.ndarray, last_sent: np.ndarray, kind: str,
                   probe_count: int, ppr: int, active: np.ndarray,
                   threshold=0.0) -> np.ndarray:
    """Ascending int64 ids of active probes whose block changed.

    Restates selection.py:284-323:
      * threshold <= 0: any bit of the full block (guard band and colour
        alpha bits included) differs (:306-307);
      * colour, threshold > 0: max over the three 10-bit channels of
        |a - b| compared ``> threshold`` (:308-314, alpha ignored);
      * visibility, threshold > 0: |f32(a) - f32(b)| > threshold where the
        python-float threshold takes part as float32 (numpy 2 weak scalar
        promotion), OR (delta is NaN AND the half bits differ) (:316-321);
      * AND the active flags, flatnonzero (:322-323).
    """
    a = blocks_by_probe(rendered, kind, ppr)[:probe_count]
    b = blocks_by_probe(last_sent, kind, ppr)[:probe_count]
    flat_a = a.reshape(probe_count, -1)
    flat_b = b.reshape(probe_count, -1)
    if threshold <= 0.0:
        hit = np.any(flat_a != flat_b, axis=1)
    else:  # also taken by a NaN threshold, as in the reference
        hit = _threshold_hit(flat_a, flat_b, kind, threshold)
    hit = hit & np.asarray(active, dtype=bool)
    return np.nonzero(hit)[0].astype(np.int64)


def _threshold_hit(fa, fb, kind, threshold):
    if kind == COLOR:
        worst = np.zeros(fa.shape, dtype=np.int64)
        for sh in (20, 10, 0):
            ca = ((fa >> np.uint32(sh)) & np.uint32(1023)).astype(np.int64)
            cb = ((fb >> np.uint32(sh)) & np.uint32(1023)).astype(np.int64)
            worst = np.maximum(worst, np.abs(ca - cb))
        return np.any(worst > threshold, axis=1)
    fa32 = fa.view(np.float16).astype(np.float32)
    fb32 = fb.view(np.float16).astype(np.float32)
    with np.errstate(invalid="ignore"):
        delta = np.abs(fa32 - fb32)
    # same promotion as the reference: a python scalar is weak (compared as
    # float32), a numpy float64 scalar promotes the comparison to float64
    over = delta > threshold
    nan_diff = np.isnan(delta) & (fa != fb)
    return np.any(over | nan_diff, axis=1)


# --- stage (3): budgeted selection -----------------------------------------


def select_for_client(changed, pvs, active, last_sent_seq, current_seq,
                      budget=None) -> list:
    """Restates selection.py:413-437.

    ids = unique(changed) that are in pvs and active; order by staleness
    ``current_seq - last_sent_seq[p]`` descending, then id ascending; keep the
    first ``budget`` (python slice semantics, so a negative budget drops from
    the end).
    """
    pvs_ids = set(int(x) for x in np.asarray(pvs).reshape(-1).tolist())
    keep = []
    for p in np.unique(np.asarray(changed, dtype=np.int64).reshape(-1)).tolist():
        if p in pvs_ids and bool(active[p]):
            keep.append(p)
    keep.sort(key=lambda p: (int(last_sent_seq[p]) - int(current_seq), p))
    if budget is not None:
        keep = keep[:budget]
    return keep


# --- stage (4): slot cache --------------------------------------------------


class SlotOverflow(RuntimeError):
    pass


class SlotCache:
    """Restates ``UpdateAtlasLayout`` slot bookkeeping (packing.py:243-317).

    The reference keeps a min-heap of free slots that is only ever popped,
    so the free set is always the contiguous tail ``[used, slot_count)``;
    this restatement keeps the counter instead.  Eviction takes the cached
    probe outside the current selection with the smallest
    ``(last_selected, slot)`` (:307-317).
    """

    def __init__(self, slot_count: int, core_side: int, slots_per_row=None):
        if slot_count < 1:
            raise ValueError("slot_count must be >= 1")
        self.slot_count = slot_count
        self.core_side = core_side
        self.slots_per_row = slots_per_row or math.ceil(math.sqrt(slot_count))
        self.slot_rows = -(-slot_count // self.slots_per_row)
        self.probe_slot: dict[int, int] = {}
        self.slot_probe: dict[int, int] = {}
        self.last_selected: dict[int, int] = {}
        self.used = 0
        self.tick = 0

    def texel_shape(self, kind: str) -> tuple:
        hw = (self.slot_rows * self.core_side, self.slots_per_row * self.core_side)
        return hw if kind == COLOR else hw + (2,)

    def slot_yx(self, slot: int) -> tuple:
        r, c = divmod(slot, self.slots_per_row)
        return r * self.core_side, c * self.core_side

    def assign(self, probes) -> list:
        chosen = sorted({int(p) for p in probes})
        if len(chosen) > self.slot_count:
            raise SlotOverflow("selection larger than the slot count")
        self.tick += 1
        chosen_set = set(chosen)
        fresh = [p for p in chosen if p not in self.probe_slot]
        n_free = self.slot_count - self.used
        direct = fresh[:n_free]
        evicting = fresh[n_free:]
        for i, p in enumerate(direct):
            self._bind(p, self.used + i)
        self.used += len(direct)
        if evicting:
            victims = sorted(
                (self.last_selected.get(q, 0), s, q)
                for q, s in self.probe_slot.items() if q not in chosen_set
            )
            if len(victims) < len(evicting):
                raise SlotOverflow("no evictable slot")
            for p, (_, s, q) in zip(evicting, victims):
                del self.probe_slot[q]
                self._bind(p, s)
        for p in chosen:
            self.last_selected[p] = self.tick
        return sorted((self.probe_slot[p], p) for p in chosen)

    def _bind(self, p, s):
        self.probe_slot[p] = s
        self.slot_probe[s] = p


def build_update_atlas(selected, cache: SlotCache, source: np.ndarray, kind: str,
                       ppr: int, update_texels=None):
    """Restates packing.py:320-338: stripped cores into their slots."""
    side = BLOCK_SIDE[kind]
    if update_texels is None:
        update_texels = np.zeros(cache.texel_shape(kind), source.dtype)
    entries = cache.assign(selected)
    core = side - 2
    for slot, probe in entries:
        br, bc = divmod(probe, ppr)
        y0, x0 = br * side + 1, bc * side + 1
        sy, sx = cache.slot_yx(slot)
        update_texels[sy:sy + core, sx:sx + core] = source[y0:y0 + core, x0:x0 + core]
    return update_texels, entries


# --- guard band (packing.py:174-196) ----------------------------------------


def guard_band_block(core: np.ndarray) -> np.ndarray:
    """Octahedral wrap rule: border edges copy the adjacent core row/column
    reversed; corners copy the diagonally opposite core corner."""
    n = core.shape[0]
    blk = np.zeros((n + 2, n + 2) + core.shape[2:], core.dtype)
    blk[1:n + 1, 1:n + 1] = core
    rev = slice(None, None, -1)
    blk[0, 1:n + 1] = core[0][rev]
    blk[n + 1, 1:n + 1] = core[n - 1][rev]
    blk[1:n + 1, 0] = core[rev, 0]
    blk[1:n + 1, n + 1] = core[rev, n - 1]
    blk[0, 0] = core[n - 1, n - 1]
    blk[0, n + 1] = core[n - 1, 0]
    blk[n + 1, 0] = core[0, n - 1]
    blk[n + 1, n + 1] = core[0, 0]
    return blk


# --- stage (4): plane packing -----------------------------------------------


def pack_color(texels: np.ndarray) -> np.ndarray:
    """packing.py:73-89: R,G,B 10-bit fields -> three uint16 planes."""
    t = np.asarray(texels, dtype=np.uint32)
    out = np.empty((3,) + t.shape, np.uint16)
    for plane in range(3):
        out[plane] = (t >> np.uint32(10 * plane)) & np.uint32(0x3FF)
    return out


def unpack_color(planes: np.ndarray) -> np.ndarray:
    p = planes.astype(np.uint32)
    return p[0] | (p[1] << np.uint32(10)) | (p[2] << np.uint32(20))


def widened_width(w: int) -> int:
    # packing.py:105-109 (ceil(4w/3) in integer arithmetic)
    return (4 * w + 2) // 3


def pack_visibility(texels: np.ndarray) -> np.ndarray:
    """packing.py:112-133: per row, the big-endian byte stream of the
    (R, G) halves is dealt round-robin into Y, U, V; zero padded."""
    t = np.asarray(texels, dtype=np.uint16)
    h, w, _ = t.shape
    ww = widened_width(w)
    stream = np.zeros((h, 3 * ww), np.uint8)
    # big-endian bytes of each half, texel by texel
    be = t.astype(">u2").view(np.uint8).reshape(h, 4 * w)
    stream[:, :4 * w] = be
    out = np.empty((3, h, ww), np.uint8)
    for plane in range(3):
        out[plane] = stream[:, plane::3]
    return out


def unpack_visibility(planes: np.ndarray, w: int) -> np.ndarray:
    _, h, ww = planes.shape
    stream = np.empty((h, 3 * ww), np.uint8)
    for plane in range(3):
        stream[:, plane::3] = planes[plane]
    be = np.ascontiguousarray(stream[:, :4 * w]).view(">u2").reshape(h, w, 2)
    return be.astype(np.uint16)


def pack_texels(texels, kind):
    return pack_color(texels) if kind == COLOR else pack_visibility(texels)


# --- stage (4): temporal delta (codec.py:207-215, 250-272) -------------------


def temporal_delta(cur: np.ndarray, prev: np.ndarray):
    """Residual ``(cur - prev) mod 2^bits`` in the plane dtype and the SKIP
    map: 1 where the 16x16 codec block (edge blocks clipped, codec.py:250-257)
    is bit-identical to the reference block (codec.py:264-272)."""
    assert cur.shape == prev.shape and cur.dtype == prev.dtype
    residual = (cur - prev).astype(cur.dtype)  # wraps modulo 2^bits
    c, h, w = cur.shape
    by, bx = -(-h // CODEC_BLOCK), -(-w // CODEC_BLOCK)
    # pad the difference mask up to whole blocks (padding never differs), then
    # reduce every 16x16 tile
    diff = np.zeros((c, by * CODEC_BLOCK, bx * CODEC_BLOCK), bool)
    diff[:, :h, :w] = cur != prev
    tiles = diff.reshape(c, by, CODEC_BLOCK, bx, CODEC_BLOCK)
    skip = (~tiles.any(axis=(2, 4))).astype(np.uint8)
    return residual, skip
