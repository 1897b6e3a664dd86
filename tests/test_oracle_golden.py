"""Pin the CPU oracle against golden vectors produced by the reference.

These run without a GPU; they are what lets the oracle stand in for the
reference on the GPU box (which has no /root/reference mount).
"""

import numpy as np
import pytest

from oracle import stream_ops as so

THRESHOLDS_PY = None


def _thresholds(golden):
    return [float(x) for x in golden("detect")["thresholds"]]


def test_pack_color_matches_reference(golden):
    g = golden("pack")
    assert np.array_equal(so.pack_color(g["color"]), g["color_planes"])
    assert so.pack_color(g["color"]).dtype == np.uint16


def test_pack_visibility_matches_reference(golden):
    g = golden("pack")
    assert np.array_equal(so.pack_visibility(g["vis"]), g["vis_planes"])
    assert np.array_equal(so.pack_visibility(g["kat3"]), g["kat3_planes"])
    for w in range(1, 14):
        got = so.pack_visibility(g[f"vis_w{w}"])
        assert np.array_equal(got, g[f"vis_w{w}_planes"]), w
        assert np.array_equal(so.unpack_visibility(got, w), g[f"vis_w{w}"])


def test_widened_width():
    import math
    for x in range(0, 3000):
        assert so.widened_width(x) == math.ceil(4 * x / 3)


def test_guard_band_matches_reference(golden):
    g = golden("guard")
    assert np.array_equal(so.guard_band_block(g["core8"]), g["block10"])
    assert np.array_equal(so.guard_band_block(g["core16"]), g["block18"])
    assert np.array_equal(so.guard_band_block(g["core4"]), g["block6"])
    assert list(g["block6"][0, 1:-1]) == [3, 2, 1, 0]


@pytest.mark.parametrize("kind", ["color", "visibility"])
@pytest.mark.parametrize("n", [300, 77, 260])
def test_detect_changed_matches_reference(golden, kind, n):
    g = golden("detect")
    tag = f"{kind}_n{n}"
    rendered = g[f"{tag}_rendered"]
    last = rendered ^ g[f"{tag}_last_xor"]
    active = g[f"{tag}_active"]
    ppr = int(g[f"{tag}_ppr"])
    for i, thr in enumerate(_thresholds(golden)):
        got = so.detect_changed(rendered, last, kind, n, ppr, active, thr)
        assert np.array_equal(got, g[f"{tag}_thr{i}"]), (kind, n, thr)
    thr = 2.0**-10 - 1e-12
    assert np.array_equal(so.detect_changed(rendered, last, kind, n, ppr, active, thr),
                          g[f"{tag}_thr_ulp"])
    assert np.array_equal(
        so.detect_changed(rendered, last, kind, n, ppr, active, np.float64(thr)),
        g[f"{tag}_thr_ulp64"])


def test_detect_kats(golden):
    g = golden("detect")
    rng = np.random.default_rng(int(g["kat2048_seed"]))
    ppr = so.default_probes_per_row(2048)
    a = rng.integers(0, 2**30, size=so.atlas_shape("color", 2048, ppr), dtype=np.uint32)
    b = a.copy()
    act = np.ones(2048, bool)
    assert so.detect_changed(a, b, "color", 2048, ppr, act).size == 0
    assert g["kat_identical"].size == 0
    br, bc = divmod(7, ppr)
    b[br * 10 + 1 + 2, bc * 10 + 1 + 3] ^= np.uint32(1)
    assert list(so.detect_changed(a, b, "color", 2048, ppr, act)) == list(g["kat_probe7"]) == [7]


def test_select_matches_reference(golden):
    g = golden("select")
    budgets = [None if b == -1 else int(b) for b in g["budgets"]]
    for c in range(int(g["ncases"])):
        for bi, budget in enumerate(budgets):
            got = so.select_for_client(g[f"c{c}_changed"], g[f"c{c}_pvs"], g[f"c{c}_active"],
                                       g[f"c{c}_seq"], int(g[f"c{c}_cur"]), budget)
            assert got == list(g[f"c{c}_b{bi}"]), (c, budget)
    assert list(g["kat_a"]) == [2]
    assert list(g["kat_b"]) == [4]


@pytest.mark.parametrize("kind", ["color", "visibility"])
def test_slot_cache_and_update_atlas_match_reference(golden, kind):
    g = golden("slots")
    src = g[f"{kind}_src0"].copy()
    ppr = int(g[f"{kind}_ppr"])
    core = 8 if kind == "color" else 16
    cache = so.SlotCache(17, core, slots_per_row=5)
    texels = None
    for s in range(int(g[f"{kind}_steps"])):
        row = int(g[f"{kind}_s{s}_row"])
        if kind == "color":
            src[row, :] ^= np.uint32(s + 1)
        else:
            src[row, :, 0] ^= np.uint16(s + 1)
        texels, entries = so.build_update_atlas(g[f"{kind}_s{s}_sel"], cache, src, kind, ppr, texels)
        assert np.array_equal(np.array(entries, np.int64).reshape(-1, 2), g[f"{kind}_s{s}_entries"])
        ps = np.full(g[f"{kind}_s{s}_probe_slot"].shape, -1, np.int64)
        for p, sl in cache.probe_slot.items():
            ps[p] = sl
        assert np.array_equal(ps, g[f"{kind}_s{s}_probe_slot"]), s
        if f"{kind}_s{s}_texels" in g:
            assert np.array_equal(texels, g[f"{kind}_s{s}_texels"]), s


def test_slot_lru_kat():
    # test_packing.py:226-233
    c = so.SlotCache(2, 8)
    c.assign([1])
    c.assign([2])
    c.assign([2])
    assert c.assign([3]) == [(0, 3)]
    assert c.probe_slot == {2: 1, 3: 0}
    with pytest.raises(so.SlotOverflow):
        so.SlotCache(2, 8).assign([1, 2, 3])


@pytest.mark.parametrize("tag", ["color", "vis"])
def test_temporal_delta_matches_codec(golden, tag):
    g = golden("delta")
    res, skip = so.temporal_delta(g[f"{tag}_cur"], g[f"{tag}_prev"])
    assert np.array_equal(skip, g[f"{tag}_skip"])
    signed = np.int16 if tag == "color" else np.int8
    assert np.array_equal(res.view(signed).astype(np.int64), g[f"{tag}_residual"])
