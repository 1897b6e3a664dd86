"""The drop-in boundary with the reference's OWN objects.

``detect_changed`` / ``select_for_client`` / ``build_update_atlas`` /
``pack_texels`` of the package are called with
  (a) stand-in classes carrying exactly the attributes of the reference's
      ``ProbeVolume`` (volume.py:68-144) and ``ProbeAtlas`` (:147-218) -- no
      package-specific attribute such as a device cache -- and
  (b) the real reference classes, imported from ``baseline/_ref`` (the
      driver's offline install, present on the GPU box) or
      ``$PROBESTREAM_REF``, side by side with the reference functions
      themselves, i.e. the INTEGRATION.md §1 module-level swap.
numpy in, numpy / list out, bit-exact."""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field

import numpy as np
import pytest

from oracle import stream_ops as so

import _reference

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ps():
    from paper_2103_05875_b200 import build_native

    build_native.build()
    from paper_2103_05875_b200 import packing, selection

    return packing, selection


# --- (a) stand-ins with exactly the reference's attributes ----------------------------


class StandInKind(enum.Enum):  # volume.py:33-58 (a different enum class than ours)
    COLOR = "color"
    VISIBILITY = "visibility"

    @property
    def block_side(self):
        return 10 if self is StandInKind.COLOR else 18

    @property
    def core_side(self):
        return self.block_side - 2


@dataclass(frozen=True)
class StandInVolume:  # volume.py:68-98: dims, origin, spacing, read-only active flags
    dims: tuple
    origin: tuple = (0.0, 0.0, 0.0)
    spacing: tuple = (1.0, 1.0, 1.0)
    active: np.ndarray = field(default=None, repr=False)

    def __post_init__(self):
        n = self.dims[0] * self.dims[1] * self.dims[2]
        flags = np.ones(n, bool) if self.active is None else np.asarray(self.active, bool).copy()
        flags.setflags(write=False)
        object.__setattr__(self, "active", flags)

    @property
    def probe_count(self):
        return self.dims[0] * self.dims[1] * self.dims[2]


class StandInAtlas:  # volume.py:147-184
    def __init__(self, kind, probe_count, probes_per_row=None, texels=None):
        self.kind = kind
        self.probe_count = probe_count
        self.probes_per_row = probes_per_row or (16 if probe_count <= 256
                                                 else math.ceil(math.sqrt(probe_count)))
        side = kind.block_side
        self.block_rows = math.ceil(probe_count / self.probes_per_row)
        shape = (self.block_rows * side, self.probes_per_row * side)
        dt = np.uint32
        if kind is StandInKind.VISIBILITY:
            shape, dt = shape + (2,), np.uint16
        self.texels = np.zeros(shape, dt) if texels is None else np.asarray(texels, dt)


def _random_pair(rng, kind_name, n, ppr, frac):
    shape = so.atlas_shape(kind_name, n, ppr)
    if kind_name == "color":
        cur = rng.integers(0, 2**30, size=shape, dtype=np.uint32)
    else:
        cur = rng.integers(0, 0x7C00, size=shape, dtype=np.uint16)
    prev = cur.copy()
    side = so.block_side(kind_name)
    for p in np.nonzero(rng.random(n) < frac)[0]:
        r, c = divmod(int(p), ppr)
        y, x = r * side + rng.integers(0, side), c * side + rng.integers(0, side)
        prev[y, x] ^= 1
    return cur, prev


@pytest.mark.parametrize("kind_name", ["color", "visibility"])
def test_standin_objects_through_the_chain(ps, kind_name):
    packing, selection = ps
    rng = np.random.default_rng(5)
    dims = (16, 8, 16)
    n = 2048
    active = rng.random(n) < 0.75
    vol = StandInVolume(dims, active=active)
    assert not hasattr(vol, "active_device")
    kind = StandInKind(kind_name)
    ppr = math.ceil(math.sqrt(n))
    cache = so.SlotCache(1024, kind.core_side)
    layout = packing.UpdateAtlasLayout(1024, kind.core_side)
    upd_ref = upd = None
    seq = np.full(n, -1, np.int64)
    for frame in range(3):
        cur, prev = _random_pair(rng, kind_name, n, ppr, 0.4)
        a, b = StandInAtlas(kind, n, ppr, cur), StandInAtlas(kind, n, ppr, prev)
        for thr in (0.0, 3.0 if kind_name == "color" else 1e-3):
            got = selection.detect_changed(a, b, vol, thr)
            want = so.detect_changed(cur, prev, kind_name, n, ppr, active, thr)
            assert isinstance(got, np.ndarray) and got.dtype == np.int64
            assert np.array_equal(got, want)
        changed = selection.detect_changed(a, b, vol)
        pvs = np.nonzero(rng.random(n) < 0.8)[0]
        sel = selection.select_for_client(changed, pvs, vol, seq, frame, budget=700)
        assert isinstance(sel, list)
        assert sel == so.select_for_client(changed, pvs, active, seq, frame, 700)
        seq[sel] = frame
        upd, entries = packing.build_update_atlas(sel, layout, a, upd)
        upd_ref, entries_ref = so.build_update_atlas(sel, cache, cur, kind_name, ppr, upd_ref)
        assert entries == entries_ref
        assert np.array_equal(upd, upd_ref)
        planes = packing.pack_texels(upd, kind)
        assert np.array_equal(planes.data, so.pack_texels(upd_ref, kind_name))


# --- (b) the real reference package, side by side ---------------------------------------


@pytest.fixture(scope="module")
def ref():
    mod = _reference.load()
    if mod is None:
        pytest.skip("reference probestream not importable (no baseline/_ref / PROBESTREAM_REF)")
    import probestream.packing  # noqa: F401
    import probestream.selection  # noqa: F401
    import probestream.volume  # noqa: F401

    return mod


@pytest.mark.parametrize("kind_name", ["color", "visibility"])
def test_reference_objects_and_functions_side_by_side(ps, ref, kind_name):
    """the package's functions replace the reference's
    module functions and are fed the reference's own ProbeVolume /
    ProbeAtlas / AtlasKind; outputs equal the reference functions' outputs."""
    packing, selection = ps
    rv, rs, rp = ref.volume, ref.selection, ref.packing
    rng = np.random.default_rng(11)
    dims = (12, 8, 12)
    n = 12 * 8 * 12
    vol = rv.ProbeVolume(dims, active=rng.random(n) < 0.75)
    kind = rv.AtlasKind(kind_name)
    ppr = rv.default_probes_per_row(n)
    slot_count = 500  # < changed count over 3 frames: eviction happens
    ref_layout = rp.UpdateAtlasLayout(slot_count, kind.core_side)
    our_layout = packing.UpdateAtlasLayout(slot_count, kind.core_side)
    ref_upd = our_upd = None
    seq = np.full(n, -1, np.int64)
    for frame in range(4):
        cur, prev = _random_pair(rng, kind_name, n, ppr, 0.5)
        a, b = rv.ProbeAtlas(kind, n, ppr, cur), rv.ProbeAtlas(kind, n, ppr, prev)
        thr = 0.0 if frame % 2 == 0 else (2.0 if kind_name == "color" else 1e-3)
        want = rs.detect_changed(a, b, vol, thr)
        got = selection.detect_changed(a, b, vol, thr)
        assert got.dtype == want.dtype and np.array_equal(got, want)
        pvs = rng.choice(n, size=n // 2, replace=False)
        budget = None if frame == 0 else 300
        want_sel = rs.select_for_client(want, pvs, vol, seq, frame, budget)
        got_sel = selection.select_for_client(got, pvs, vol, seq, frame, budget)
        assert got_sel == want_sel
        seq[np.asarray(want_sel, np.int64)] = frame
        ref_upd, ref_entries = rp.build_update_atlas(want_sel, ref_layout, a, ref_upd)
        our_upd, our_entries = packing.build_update_atlas(got_sel, our_layout, a, our_upd)
        assert our_entries == ref_entries
        assert np.array_equal(our_upd, ref_upd)
        assert our_layout.probe_slot == ref_layout.probe_slot
        rpl = rp.pack_texels(ref_upd, kind)
        opl = packing.pack_texels(our_upd, kind)
        assert opl.kind.value == rpl.kind.value
        assert np.array_equal(opl.data, rpl.data)


def test_reference_layout_mismatch_error_is_a_value_error(ps, ref):
    """LayoutMismatchError (selection.py:25) semantics across the swap."""
    packing, selection = ps
    rv = ref.volume
    vol = rv.ProbeVolume((4, 4, 4))
    a = rv.ProbeAtlas(rv.AtlasKind.COLOR, 64)
    b = rv.ProbeAtlas(rv.AtlasKind.VISIBILITY, 64)
    with pytest.raises(ValueError):
        selection.detect_changed(a, b, vol)
    with pytest.raises(ref.selection.LayoutMismatchError):
        ref.selection.detect_changed(a, b, vol)
