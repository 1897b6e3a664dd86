"""GPU parity for stages (3) and (4): detect / select / slot cache / build /
pack / temporal delta, through the C ABI, against the oracle and the
reference's golden vectors.  Bit-exact everywhere."""

import math

import numpy as np
import pytest
import torch

from oracle import stream_ops as so

pytestmark = pytest.mark.gpu

DEV = "cuda"


@pytest.fixture(scope="module")
def ps():
    from paper_2103_05875_b200 import build_native

    build_native.build()
    import paper_2103_05875_b200 as pkg
    from paper_2103_05875_b200 import delta, packing, selection

    return pkg, packing, selection, delta


# --- packing -------------------------------------------------------------------------


def test_pack_golden(ps, golden):
    _, packing, _, _ = ps
    g = golden("pack")
    got = packing.pack_color(g["color"])
    assert isinstance(got.data, np.ndarray)
    assert np.array_equal(got.data, g["color_planes"])
    assert np.array_equal(packing.pack_visibility(g["vis"]).data, g["vis_planes"])
    assert np.array_equal(packing.pack_visibility(g["kat3"]).data, g["kat3_planes"])
    for w in range(1, 14):
        planes = packing.pack_visibility(g[f"vis_w{w}"])
        assert np.array_equal(planes.data, g[f"vis_w{w}_planes"]), w
        assert np.array_equal(packing.unpack_visibility(planes, w), g[f"vis_w{w}"])


@pytest.mark.parametrize("h,w", [(1, 1), (7, 13), (16, 16), (33, 50), (64, 64), (100, 257),
                                 (17, 2904), (1, 4096)])
def test_pack_color_random(ps, h, w):
    _, packing, _, _ = ps
    rng = np.random.default_rng(h * 1000 + w)
    t = rng.integers(0, 2**32, size=(h, w), dtype=np.uint32)
    want = so.pack_color(t)
    assert np.array_equal(packing.pack_color(t).data, want)
    dt = torch.from_numpy(t).to(DEV)
    got = packing.pack_color(dt)
    assert got.data.is_cuda
    assert np.array_equal(got.data.cpu().numpy(), want)
    # strided region (a column window of a wider atlas)
    if w > 4:
        big = rng.integers(0, 2**32, size=(h, w + 9), dtype=np.uint32)
        region = torch.from_numpy(big).to(DEV)[:, 3:3 + w]
        assert np.array_equal(packing.pack_color(region).data.cpu().numpy(),
                              so.pack_color(big[:, 3:3 + w]))
    back = packing.unpack_color(packing.pack_color(t))
    assert np.array_equal(back, t & np.uint32(0x3FFFFFFF))


@pytest.mark.parametrize("h,w", [(1, 1), (1, 2), (3, 5), (16, 12), (18, 18), (20, 48),
                                 (33, 100), (16, 5808), (5, 2048)])
def test_pack_visibility_random(ps, h, w):
    _, packing, _, _ = ps
    rng = np.random.default_rng(h * 7919 + w)
    t = rng.integers(0, 2**16, size=(h, w, 2), dtype=np.uint16)
    t[0, 0] = (0xFFFF, 0x7FFF)
    want = so.pack_visibility(t)
    got = packing.pack_visibility(t)
    assert got.data.shape == (3, h, math.ceil(4 * w / 3))
    assert np.array_equal(got.data, want)
    dt = torch.from_numpy(t).to(DEV)
    assert np.array_equal(packing.pack_visibility(dt).data.cpu().numpy(), want)
    assert np.array_equal(packing.unpack_visibility(got, w), t)
    if w > 3:
        big = rng.integers(0, 2**16, size=(h, w + 5, 2), dtype=np.uint16)
        region = torch.from_numpy(big).to(DEV)[:, 2:2 + w]
        assert np.array_equal(packing.pack_visibility(region).data.cpu().numpy(),
                              so.pack_visibility(big[:, 2:2 + w]))


def test_pack_errors(ps):
    _, packing, _, _ = ps
    with pytest.raises(ValueError):
        packing.pack_color(np.zeros((2, 2, 2), np.uint32))
    with pytest.raises(ValueError):
        packing.pack_visibility(np.zeros((2, 2), np.uint16))
    with pytest.raises(ValueError):
        packing.unpack_visibility(packing.pack_visibility(np.zeros((2, 3, 2), np.uint16)), 4)
    empty = packing.pack_color(np.zeros((0, 5), np.uint32))
    assert empty.data.shape == (3, 0, 5)


# --- temporal delta -------------------------------------------------------------------


@pytest.mark.parametrize("tag", ["color", "vis"])
def test_delta_golden(ps, golden, tag):
    _, packing, _, delta = ps
    g = golden("delta")
    kind = packing.PlaneKind.COLOR_10IN16 if tag == "color" else packing.PlaneKind.VISIBILITY_BYTES
    res, skip = delta.temporal_delta(packing.PlaneSet(kind, g[f"{tag}_cur"]),
                                     packing.PlaneSet(kind, g[f"{tag}_prev"]))
    assert np.array_equal(skip, g[f"{tag}_skip"])
    signed = np.int16 if tag == "color" else np.int8
    assert np.array_equal(res.view(signed).astype(np.int64), g[f"{tag}_residual"])
    # key frame: nothing is SKIP
    _, skip0 = delta.temporal_delta(packing.PlaneSet(kind, g[f"{tag}_cur"]), None)
    assert not skip0.any()


@pytest.mark.parametrize("kind", ["color", "visibility"])
@pytest.mark.parametrize("slots", [1, 5, 9, 17, 363, 1000, 1089, 4096, 16384, 131072])
def test_pack_delta_matches_pack_then_delta(ps, kind, slots):
    """Every row-alignment class of the visibility planes: 16-byte aligned
    rows (slots 9: one CTA in x; 1,089: 704-byte rows, several CTAs; 131,072:
    the C4 update atlas, 7,744-byte rows, partial last slot row) and
    unaligned ones (5, 17, 363, 1,000, 4,096, 16,384)."""
    pkg, packing, _, delta = ps
    rng = np.random.default_rng(slots)
    core = 8 if kind == "color" else 16
    spr = math.ceil(math.sqrt(slots))
    rows = math.ceil(slots / spr)
    shape = (rows * core, spr * core) + (() if kind == "color" else (2,))
    dt = np.uint32 if kind == "color" else np.uint16
    hi = 2**32 if kind == "color" else 2**16
    prev_tex = rng.integers(0, hi, size=shape, dtype=dt)
    cur_tex = prev_tex.copy()
    flat = cur_tex.reshape(-1)
    pick = rng.choice(flat.size, size=max(1, flat.size // 50), replace=False)
    flat[pick] = rng.integers(0, hi, size=pick.size, dtype=dt)
    prev_planes = so.pack_texels(prev_tex, kind)
    want_planes = so.pack_texels(cur_tex, kind)
    want_res, want_skip = so.temporal_delta(want_planes, prev_planes)
    planes, res, skip = delta.pack_delta(torch.from_numpy(cur_tex).to(DEV), kind,
                                         torch.from_numpy(prev_planes).to(DEV))
    assert np.array_equal(planes.cpu().numpy(), want_planes)
    assert np.array_equal(res.cpu().numpy(), want_res)
    assert np.array_equal(skip.cpu().numpy(), want_skip)
    # key frame
    planes0, _, skip0 = delta.pack_delta(torch.from_numpy(cur_tex).to(DEV), kind, None)
    assert np.array_equal(planes0.cpu().numpy(), want_planes)
    assert not skip0.cpu().numpy().any()


@pytest.mark.parametrize("slots", [17, 363, 4096, 16384])
def test_pack_delta_sparse_skip_unaligned_rows(ps, slots):
    """Visibility planes with rows that are not 16-byte aligned (the flat
    16-byte-word kernel): a handful of changed texels, so the SKIP map is
    mostly 1 and every cleared block is pinned -- including blocks reached
    only through a word that straddles two plane rows."""
    _, _, _, delta = ps
    rng = np.random.default_rng(slots + 7)
    spr = math.ceil(math.sqrt(slots))
    rows = math.ceil(slots / spr)
    shape = (rows * 16, spr * 16, 2)
    prev_tex = rng.integers(0, 2**16, size=shape, dtype=np.uint16)
    cur_tex = prev_tex.copy()
    h, w = shape[0], shape[1]
    pw = (4 * w + 2) // 3
    # texels at the ends of rows (straddling words) plus random ones
    for r in rng.choice(h, size=min(h, 12), replace=False):
        cur_tex[r, w - 1, rng.integers(0, 2)] ^= np.uint16(1 << int(rng.integers(0, 16)))
        cur_tex[r, 0, rng.integers(0, 2)] ^= np.uint16(1 << int(rng.integers(0, 16)))
    for _ in range(20):
        cur_tex[rng.integers(0, h), rng.integers(0, w), rng.integers(0, 2)] ^= np.uint16(0x8000)
    prev_planes = so.pack_texels(prev_tex, "visibility")
    want_planes = so.pack_texels(cur_tex, "visibility")
    want_res, want_skip = so.temporal_delta(want_planes, prev_planes)
    assert (pw * 1) % 16 != 0 and want_skip.mean() > 0.5
    planes, res, skip = delta.pack_delta(torch.from_numpy(cur_tex).to(DEV), "visibility",
                                         torch.from_numpy(prev_planes).to(DEV))
    assert np.array_equal(planes.cpu().numpy(), want_planes)
    assert np.array_equal(res.cpu().numpy(), want_res)
    assert np.array_equal(skip.cpu().numpy(), want_skip)


# --- detect -----------------------------------------------------------------------------


@pytest.mark.parametrize("kind", ["color", "visibility"])
@pytest.mark.parametrize("n", [300, 77, 260])
def test_detect_golden(ps, golden, kind, n):
    pkg, _, selection, _ = ps
    g = golden("detect")
    tag = f"{kind}_n{n}"
    rendered = g[f"{tag}_rendered"]
    last = rendered ^ g[f"{tag}_last_xor"]
    ppr = int(g[f"{tag}_ppr"])
    vol = pkg.ProbeVolume((n, 1, 1), active=g[f"{tag}_active"])
    ra = pkg.ProbeAtlas(kind, n, ppr, rendered)
    la = pkg.ProbeAtlas(kind, n, ppr, last)
    for i, thr in enumerate(g["thresholds"]):
        got = selection.detect_changed(ra, la, vol, float(thr))
        assert got.dtype == np.int64
        assert np.array_equal(got, g[f"{tag}_thr{i}"]), (kind, n, thr)
    thr = 2.0**-10 - 1e-12
    assert np.array_equal(selection.detect_changed(ra, la, vol, thr), g[f"{tag}_thr_ulp"])
    assert np.array_equal(selection.detect_changed(ra, la, vol, np.float64(thr)),
                          g[f"{tag}_thr_ulp64"])
    # device tensors in, device tensor out
    rd, ld = ra.to(DEV), la.to(DEV)
    got = selection.detect_changed(rd, ld, vol)
    assert got.is_cuda and np.array_equal(got.cpu().numpy(), g[f"{tag}_thr0"])


def test_detect_layout_errors(ps):
    pkg, _, selection, _ = ps
    a = pkg.ProbeAtlas("color", 20)
    vol = pkg.ProbeVolume((20, 1, 1))
    with pytest.raises(pkg.LayoutMismatchError):
        selection.detect_changed(a, pkg.ProbeAtlas("visibility", 20), vol)
    with pytest.raises(pkg.LayoutMismatchError):
        selection.detect_changed(a, pkg.ProbeAtlas("color", 20, 5), vol)
    with pytest.raises(pkg.LayoutMismatchError):
        selection.detect_changed(a, a.copy(), pkg.ProbeVolume((21, 1, 1)))
    assert selection.detect_changed(a, a.copy(), vol).size == 0


@pytest.mark.parametrize("kind", ["color", "visibility"])
@pytest.mark.parametrize("frac", [1.0, 0.1, 0.001])
def test_detect_full_size_property(ps, kind, frac):
    """C4 size (131,072 probes): the exact path returns exactly the mutated
    set AND active (size-independent property), and the threshold path
    agrees with the oracle on a 75%-active volume."""
    pkg, _, selection, _ = ps
    n = 64 * 32 * 64
    rng = np.random.default_rng(int(frac * 1000) + (kind == "color"))
    vol = pkg.ProbeVolume((64, 32, 64), active=rng.random(n) < 0.75)
    a = pkg.ProbeAtlas(kind, n, device=DEV)
    if kind == "color":
        a.texels.view(torch.int32).random_(0, 2**30)
    else:
        a.texels.view(torch.int16).random_(0, 0x7C00)
    b = a.copy()
    k = max(1, int(n * frac))
    mutated = np.sort(rng.choice(n, size=k, replace=False))
    side = a.kind.block_side
    ppr = a.probes_per_row
    rows = torch.from_numpy((mutated // ppr) * side + 1 + rng.integers(0, side - 2, size=k)).to(DEV)
    cols = torch.from_numpy((mutated % ppr) * side + 1 + rng.integers(0, side - 2, size=k)).to(DEV)
    bt = b.texels.view(torch.int32) if kind == "color" else b.texels.view(torch.int16)[..., 0]
    bt[rows, cols] ^= 1
    got = selection.detect_changed(a, b, vol).cpu().numpy()
    want = mutated[vol.active[mutated]]
    assert np.array_equal(got, want)


# --- select -----------------------------------------------------------------------------


def test_select_golden(ps, golden):
    pkg, _, selection, _ = ps
    g = golden("select")
    budgets = [None if b == -1 else int(b) for b in g["budgets"]]
    for c in range(int(g["ncases"])):
        n = len(g[f"c{c}_active"])
        vol = pkg.ProbeVolume((n, 1, 1), active=g[f"c{c}_active"])
        for bi, budget in enumerate(budgets):
            got = selection.select_for_client(g[f"c{c}_changed"], g[f"c{c}_pvs"], vol,
                                              g[f"c{c}_seq"], int(g[f"c{c}_cur"]), budget)
            assert got == list(g[f"c{c}_b{bi}"]), (c, budget)
    vol = pkg.ProbeVolume((16, 1, 1))
    assert selection.select_for_client([1, 2], [2, 3], vol, np.zeros(16, int), 5) == [2]
    assert selection.select_for_client([4, 9], [4, 9], vol, np.zeros(16, int), 5, budget=1) == [4]
    assert selection.select_for_client([], [1], vol, np.zeros(16, int), 5) == []


def test_select_index_error_only_when_in_both(ps):
    pkg, _, selection, _ = ps
    vol = pkg.ProbeVolume((8, 1, 1))
    seq = np.zeros(8, int)
    assert selection.select_for_client([1, 99], [1], vol, seq, 1) == [1]
    with pytest.raises(IndexError):
        selection.select_for_client([1, 99], [99], vol, seq, 1)


def test_select_full_size(ps):
    pkg, _, selection, _ = ps
    n = 131072
    rng = np.random.default_rng(9)
    active = rng.random(n) < 0.8
    vol = pkg.ProbeVolume((64, 32, 64), active=active)
    changed = rng.choice(n, size=n // 2, replace=False)
    pvs = rng.choice(n, size=n // 2, replace=False)
    seq = rng.integers(-100, 100, size=n)
    for budget in (None, 1000, 0, -5):
        got = selection.select_for_client(changed, pvs, vol, seq, 200, budget)
        want = so.select_for_client(changed, pvs, active, seq, 200, budget)
        assert got == want


def test_select_unordered_is_the_same_set(ps):
    """ordered=False (the server chain's fast path, no budget) returns exactly
    the selected set in ascending id order."""
    pkg, _, selection, _ = ps
    n = 131072
    rng = np.random.default_rng(10)
    active = rng.random(n) < 0.8
    vol = pkg.ProbeVolume((64, 32, 64), active=active)
    changed = rng.choice(n, size=n // 3, replace=False)
    seq = torch.from_numpy(rng.integers(-100, 100, size=n)).to(DEV)
    bits, _ = selection.ids_to_bits(changed, n, torch.device(DEV))
    ids, cnt = selection.select_device(bits, None, vol, seq, 200, None, ordered=False)
    k = int(cnt.item())
    want = so.select_for_client(changed, np.arange(n), active, seq.cpu().numpy(), 200, None)
    assert ids[:k].cpu().tolist() == sorted(want)


# --- slot cache + build ---------------------------------------------------------------


@pytest.mark.parametrize("kind", ["color", "visibility"])
def test_slots_golden(ps, golden, kind):
    pkg, packing, _, _ = ps
    g = golden("slots")
    src = g[f"{kind}_src0"].copy()
    ppr = int(g[f"{kind}_ppr"])
    n = 60
    core = 8 if kind == "color" else 16
    layout = packing.UpdateAtlasLayout(17, core, slots_per_row=5)
    texels = None
    for s in range(int(g[f"{kind}_steps"])):
        row = int(g[f"{kind}_s{s}_row"])
        if kind == "color":
            src[row, :] ^= np.uint32(s + 1)
        else:
            src[row, :, 0] ^= np.uint16(s + 1)
        atlas = pkg.ProbeAtlas(kind, n, ppr, src)
        texels, entries = packing.build_update_atlas(g[f"{kind}_s{s}_sel"], layout, atlas, texels)
        assert np.array_equal(np.array(entries, np.int64).reshape(-1, 2),
                              g[f"{kind}_s{s}_entries"]), s
        ps_ = np.full(n, -1, np.int64)
        for p, sl in layout.probe_slot.items():
            ps_[p] = sl
        assert np.array_equal(ps_, g[f"{kind}_s{s}_probe_slot"]), s
        if f"{kind}_s{s}_texels" in g:
            assert np.array_equal(texels, g[f"{kind}_s{s}_texels"]), s


def test_slot_kats(ps):
    _, packing, _, _ = ps
    layout = packing.UpdateAtlasLayout(2, 8)
    layout.assign([1])
    layout.assign([2])
    layout.assign([2])
    assert layout.assign([3]) == [(0, 3)]
    assert layout.probe_slot == {2: 1, 3: 0}
    with pytest.raises(packing.SlotOverflowError):
        packing.UpdateAtlasLayout(2, 8).assign([1, 2, 3])
    a, b = packing.UpdateAtlasLayout(4, 8), packing.UpdateAtlasLayout(4, 8)
    for sel in [[3, 1], [1], [7, 3, 2], [9], [1, 9]]:
        assert a.assign(sel) == b.assign(list(reversed(sel)))


def test_slots_overflow_does_not_mutate(ps):
    _, packing, _, _ = ps
    layout = packing.UpdateAtlasLayout(3, 8, probe_count=10)
    first = layout.assign([4, 5])
    with pytest.raises(packing.SlotOverflowError):
        layout.assign(torch.tensor([1, 2, 3, 6], device=DEV))
    assert layout.probe_slot == {4: 0, 5: 1}
    assert layout.assign([4, 5]) == first


@pytest.mark.parametrize("slots,n", [(50, 200), (1000, 3000), (4096, 4096)])
def test_slot_random_sequences_vs_oracle(ps, slots, n):
    _, packing, _, _ = ps
    rng = np.random.default_rng(slots + n)
    dev_layout = packing.UpdateAtlasLayout(slots, 8, probe_count=n)
    ref = so.SlotCache(slots, 8)
    for step in range(12):
        k = int(rng.integers(0, slots + 1))
        sel = rng.choice(n, size=k, replace=False)
        assert dev_layout.assign(torch.from_numpy(sel).to(DEV)) == ref.assign(sel), step
    assert dev_layout.probe_slot == ref.probe_slot


def _bits_of(ids, n):
    words = np.zeros((n + 31) // 32, np.uint32)
    for p in ids:
        words[p >> 5] |= np.uint32(1) << np.uint32(p & 31)
    return torch.from_numpy(words.view(np.int32)).to(DEV)


@pytest.mark.parametrize("n,slots", [(1, 1), (37, 37), (5000, 5000), (20000, 24000),
                                     (131072, 131072)])
def test_assign_bits_vs_oracle(ps, n, slots):
    """ps_assign_slots_bits (bitmap in, two look-back kernels) == the reference
    slot cache (packing.py:283-305) == ps_assign_slots on the same sequence:
    entries, probe_slot, slot_probe, last_selected and the tick, with and
    without a PVS mask, across tile boundaries (8192 probes per tile)."""
    _, packing, _, _ = ps
    rng = np.random.default_rng(n + slots)
    a = packing.UpdateAtlasLayout(slots, 8, probe_count=n)
    b = packing.UpdateAtlasLayout(slots, 8, probe_count=n)
    ref = so.SlotCache(slots, 8)
    steps = 6 if n < 100000 else 3
    for step in range(steps):
        frac = [1.0, 0.3, 0.0, 0.9, 0.01, 1.0][step]
        sel = np.flatnonzero(rng.random(n) < frac)
        pvs = None
        if step == 3:
            pv = np.flatnonzero(rng.random(n) < 0.5)
            pvs = _bits_of(pv, n)
            sel_eff = np.intersect1d(sel, pv)
        else:
            sel_eff = sel
        entries, count = a.assign_bits_device(_bits_of(sel, n), pvs)
        got = [tuple(r) for r in entries[: int(count.item())].cpu().tolist()]
        want = ref.assign(sel_eff)
        assert got == [tuple(map(int, e)) for e in want], step
        assert b.assign(torch.from_numpy(sel_eff).to(DEV)) == got, step
        assert torch.equal(a._probe_slot, b._probe_slot)
        assert torch.equal(a._slot_probe, b._slot_probe)
        assert torch.equal(a._last_selected, b._last_selected)
        assert torch.equal(a._meta[:2], b._meta[:2])
        plan = a._plan.cpu().tolist()
        assert plan[0] == len(sel_eff) and plan[6] == step + 1
    assert a.probe_slot == ref.probe_slot


def test_assign_bits_needs_a_slot_per_probe(ps):
    _, packing, _, _ = ps
    layout = packing.UpdateAtlasLayout(10, 8, probe_count=20)
    with pytest.raises(ValueError):
        layout.assign_bits_device(_bits_of([1, 2], 20))
