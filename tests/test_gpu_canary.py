"""Out-of-bounds write checks with canary guard zones (compute-sanitizer is
closed on the GPU pool): every output buffer of the main
kernels is a view into a larger allocation whose margins hold a byte
pattern; after the kernels run (edge-case shapes: partial tiles, probe
counts that are not multiples of 32 / 8192, misaligned plane rows, key and
P frames) the margins must be intact.  Called through the C ABI or with the
package's buffers swapped for guarded views."""

from __future__ import annotations

import ctypes
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
DEV = "cuda"
PAD = 4096  # bytes of guard zone on each side
CANARY = 0xA5


class Guarded:
    """A tensor view with PAD canary bytes before and after it."""

    def __init__(self, shape, dtype, fill=None):
        n = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
        self.raw = torch.full((PAD + n + PAD,), CANARY, dtype=torch.uint8, device=DEV)
        self.view = self.raw[PAD:PAD + n].view(dtype).view(shape)
        if fill is not None:
            self.view.copy_(fill)

    def intact(self) -> bool:
        torch.cuda.synchronize()
        return bool((self.raw[:PAD] == CANARY).all()) and bool((self.raw[-PAD:] == CANARY).all())


@pytest.fixture(scope="module")
def pkg():
    from paper_2103_05875_b200 import build_native

    build_native.build()
    from paper_2103_05875_b200 import _native as N

    return N


def stream():
    return torch.cuda.current_stream().cuda_stream


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("n", [1, 37, 8193, 20000])
def test_detect_assign_build_pack_stay_in_bounds(pkg, kind, n):
    N = pkg
    lib = N.lib()
    rng = np.random.default_rng(n + kind)
    side = 10 if kind == 0 else 18
    core = side - 2
    ppr = 16 if n <= 256 else math.ceil(math.sqrt(n))
    rows = math.ceil(n / ppr)
    shape = (rows * side, ppr * side)
    rendered = torch.from_numpy(rng.integers(0, 2**31, size=shape, dtype=np.uint32)).to(DEV)
    last = Guarded(shape, torch.int32, rendered.view(torch.int32) ^ 1)
    active = torch.from_numpy((rng.random(n) < 0.8).astype(np.uint8)).to(DEV)
    words = (n + 31) // 32
    bits = Guarded((words,), torch.int32)
    ids = Guarded((n,), torch.int64)
    count = Guarded((1,), torch.int64)
    ws = torch.empty(lib.ps_detect_workspace_bytes(n), dtype=torch.uint8, device=DEV)
    N.call("ps_detect_changed", kind, rendered.data_ptr(), last.view.data_ptr(), n, ppr, rows,
           active.data_ptr(), 0.0, 0, bits.view.data_ptr(), ids.view.data_ptr(),
           count.view.data_ptr(), ws.data_ptr(), ws.numel(), stream())
    assert bits.intact() and ids.intact() and count.intact()
    # slot cache from the bitmap, then build + commit, then pack + delta
    slots = n
    spr = math.ceil(math.sqrt(slots))
    probe_slot = Guarded((n,), torch.int32, torch.full((n,), -1, dtype=torch.int32))
    slot_probe = Guarded((slots,), torch.int32, torch.full((slots,), -1, dtype=torch.int32))
    last_sel = Guarded((n,), torch.int64, torch.zeros(n, dtype=torch.int64))
    meta = Guarded((4,), torch.int64, torch.zeros(4, dtype=torch.int64))
    entries = Guarded((slots, 2), torch.int64)
    ecount = Guarded((1,), torch.int64)
    plan = Guarded((8,), torch.int64)
    aws = torch.empty(lib.ps_assign_bits_workspace_bytes(n, slots), dtype=torch.uint8, device=DEV)
    for _ in range(2):
        N.call("ps_assign_slots_bits", bits.view.data_ptr(), None, n, slots,
               probe_slot.view.data_ptr(), slot_probe.view.data_ptr(), last_sel.view.data_ptr(),
               meta.view.data_ptr(), entries.view.data_ptr(), ecount.view.data_ptr(),
               plan.view.data_ptr(), None, aws.data_ptr(), aws.numel(), stream())
    for g in (probe_slot, slot_probe, last_sel, meta, entries, ecount, plan):
        assert g.intact()
    srows = math.ceil(slots / spr)
    ushape = (srows * core, spr * core)
    upd = Guarded(ushape, torch.int32, torch.zeros(ushape, dtype=torch.int32))
    seq = Guarded((n,), torch.int64, torch.zeros(n, dtype=torch.int64))
    N.call("ps_build_update", kind, rendered.data_ptr(), n, ppr, entries.view.data_ptr(),
           ecount.view.data_ptr(), slots, spr, upd.view.data_ptr(), ushape[1],
           last.view.data_ptr(), seq.view.data_ptr(), 3, None, stream())
    assert upd.intact() and last.intact() and seq.intact()
    h = ushape[0]
    w = ushape[1]  # texels per row (one 32-bit word each, both kinds)
    pw, eb = (w, 2) if kind == 0 else ((4 * w + 2) // 3, 1)
    pdt = torch.int16 if eb == 2 else torch.uint8
    prev = Guarded((3, h, pw), pdt, torch.zeros((3, h, pw), dtype=pdt))
    cur = Guarded((3, h, pw), pdt)
    res = Guarded((3, h, pw), pdt)
    sk = Guarded((3, -(-h // 16), -(-pw // 16)), torch.uint8)
    for p in (None, prev.view.data_ptr()):  # key frame, then P frame
        N.call("ps_pack_delta", kind, upd.view.data_ptr(), h, w, w, cur.view.data_ptr(), p,
               res.view.data_ptr(), sk.view.data_ptr(), None, stream())
        for g in (cur, res, sk, prev):
            assert g.intact()


def test_trace_blend_stay_in_bounds(pkg):
    """Trace + shading + tcgen05 blend + atlas blocks on a volume whose probe
    count (105) is not a multiple of the blend's 32-probe CTA or a warp."""
    from paper_2103_05875_b200 import scene as S
    from paper_2103_05875_b200.probes import ProbeUpdater

    sc = S.cornell_box()
    vol = S.volume_for(sc, (7, 5, 3))
    upd = ProbeUpdater(vol, sc.device(), rays_per_probe=64, shadows="map")
    guards = []

    def guard(t):
        g = Guarded(tuple(t.shape), t.dtype, t)
        guards.append(g)
        return g.view

    upd.records = guard(upd.records)
    upd.irradiance = guard(upd.irradiance)
    upd.moments = guard(upd.moments)
    for bufs in (upd._color_bufs, upd._vis_bufs):
        for atlas in bufs:
            atlas.texels = guard(atlas.texels)
    for f in range(3):
        upd.update(f, S.moving_light(sc, f).lights)
    torch.cuda.synchronize()
    assert all(g.intact() for g in guards)
