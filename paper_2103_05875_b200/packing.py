"""Plane packing, guard band and the update-atlas slot cache on the GPU.

Drop-in mirror of ``probestream.packing`` (packing.py in the reference):
same names, argument meaning, return types and exceptions.  numpy inputs are
staged to the device and results come back as numpy (the reference's
contract); CUDA-tensor inputs stay on the device and results are CUDA
tensors (the zero-copy fast path).  Every transform runs in the CUDA library
(``csrc/ps_pack.cu``, ``csrc/ps_select.cu``); there is no CPU fallback.

* ``pack_color`` / ``unpack_color``              packing.py:73-99
* ``widened_width`` / ``pack_visibility`` / ...  packing.py:105-163
* ``strip_guard_band`` / ``reconstruct_guard_band`` packing.py:174-202
* ``UpdateAtlasLayout`` / ``build_update_atlas``  packing.py:231-338
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .errors import SlotOverflowError
from .volume import AtlasKind, ProbeAtlas, kind_of

__all__ = [
    "PlaneKind", "PlaneSet", "pack_color", "unpack_color", "widened_width", "pack_visibility",
    "unpack_visibility", "pack_texels", "unpack_texels", "strip_guard_band",
    "reconstruct_guard_band", "guard_band_valid", "SlotOverflowError", "UpdateAtlasLayout",
    "build_update_atlas", "apply_update_entries",
]


class PlaneKind(enum.Enum):
    COLOR_10IN16 = "color-10in16"
    VISIBILITY_BYTES = "visibility-bytes"

    @property
    def dtype(self):
        return np.uint16 if self is PlaneKind.COLOR_10IN16 else np.uint8

    @property
    def torch_dtype(self):
        return torch.uint16 if self is PlaneKind.COLOR_10IN16 else torch.uint8


@dataclass
class PlaneSet:
    """Three equally sized planes (Y, U, V); ``data`` is numpy or a CUDA tensor."""

    kind: PlaneKind
    data: object

    def __post_init__(self) -> None:
        shape = tuple(self.data.shape)
        if len(shape) != 3 or shape[0] != 3:
            raise ValueError(f"plane data must be (3, h, w), got {shape}")
        want = self.kind.torch_dtype if D.is_tensor(self.data) else np.dtype(self.kind.dtype)
        if self.data.dtype != want:
            raise ValueError(f"plane dtype {self.data.dtype} does not match {self.kind}")

    @property
    def height(self) -> int:
        return self.data.shape[1]

    @property
    def width(self) -> int:
        return self.data.shape[2]

    @property
    def element_bits(self) -> int:
        return 16 if self.kind is PlaneKind.COLOR_10IN16 else 8

    def copy(self) -> "PlaneSet":
        return PlaneSet(self.kind, self.data.clone() if D.is_tensor(self.data) else self.data.copy())

    def numpy(self) -> np.ndarray:
        return D.to_numpy(self.data) if D.is_tensor(self.data) else self.data

    def equals(self, other: "PlaneSet") -> bool:
        return self.kind == other.kind and np.array_equal(self.numpy(), other.numpy())


# --- helpers ------------------------------------------------------------------------


def _stage(texels, np_dtype, torch_dtype):
    """Return (device tensor, was_numpy)."""
    if D.is_tensor(texels):
        t = texels if texels.is_cuda else texels.to(D.device_of())
        if t.dtype != torch_dtype:
            if t.dtype in (torch.int32, torch.int16) and t.element_size() == torch_dtype.itemsize:
                t = t.view(torch_dtype)
            else:
                t = t.to(torch_dtype)
        return t, False
    arr = np.ascontiguousarray(np.asarray(texels, dtype=np_dtype))
    return torch.from_numpy(arr).to(D.device_of()), True


def _row_stride(t: torch.Tensor, inner: int) -> tuple:
    """Row stride in texels for a (h, w[, 2]) region; makes it contiguous if needed."""
    if t.dim() == 2:
        if t.stride(1) != 1 and t.shape[1] > 1:
            t = t.contiguous()
        return t, t.stride(0) if t.shape[0] > 1 else t.shape[1]
    if t.stride(2) != 1 or (t.shape[1] > 1 and t.stride(1) != 2) or t.stride(0) % 2:
        t = t.contiguous()
    return t, (t.stride(0) // 2) if t.shape[0] > 1 else t.shape[1]


# --- colour packing (packing.py:73-99) --------------------------------------------


def pack_color(texels) -> PlaneSet:
    """Packed 32-bit colour texels -> uint16 Y/U/V planes (R->Y, G->U, B->V)."""
    if len(getattr(texels, "shape", np.shape(texels))) != 2:
        raise ValueError("color texel region must be 2-D")
    t, was_np = _stage(texels, np.uint32, torch.uint32)
    t, stride = _row_stride(t, 1)
    h, w = t.shape
    out = torch.empty((3, h, w), dtype=torch.uint16, device=t.device)
    if h and w:
        N.call("ps_pack_color", t.data_ptr(), h, w, stride, out.data_ptr(), D.stream_ptr(t.device))
    return PlaneSet(PlaneKind.COLOR_10IN16, D.to_numpy(out) if was_np else out)


def unpack_color(planes: PlaneSet):
    if planes.kind is not PlaneKind.COLOR_10IN16:
        raise ValueError("expected color plane set")
    data, was_np = _stage(planes.data, np.uint16, torch.uint16)
    data = data.contiguous()
    if bool((data.view(torch.int16) & -1024).any()):  # any bit above the 10-bit range
        raise ValueError("color plane element exceeds 10-bit range")
    _, h, w = data.shape
    out = torch.empty((h, w), dtype=torch.uint32, device=data.device)
    if h and w:
        N.call("ps_unpack_color", data.data_ptr(), h, w, out.data_ptr(), D.stream_ptr(data.device))
    return D.to_numpy(out) if was_np else out


# --- visibility packing (packing.py:105-151) -----------------------------------------


def widened_width(texel_width: int) -> int:
    if texel_width < 0:
        raise ValueError("width must be >= 0")
    return (4 * texel_width + 2) // 3


def pack_visibility(texels) -> PlaneSet:
    """RG16F texels -> three uint8 planes by row-wise MSB-first byte distribution."""
    shape = tuple(getattr(texels, "shape", np.shape(texels)))
    if len(shape) != 3 or shape[2] != 2:
        raise ValueError("visibility texel region must be (h, w, 2)")
    t, was_np = _stage(texels, np.uint16, torch.uint16)
    t, stride = _row_stride(t, 2)
    h, w, _ = t.shape
    out = torch.empty((3, h, widened_width(w)), dtype=torch.uint8, device=t.device)
    if h and w:
        N.call("ps_pack_visibility", t.data_ptr(), h, w, stride, out.data_ptr(),
               D.stream_ptr(t.device))
    return PlaneSet(PlaneKind.VISIBILITY_BYTES, D.to_numpy(out) if was_np else out)


def unpack_visibility(planes: PlaneSet, texel_width: int):
    if planes.kind is not PlaneKind.VISIBILITY_BYTES:
        raise ValueError("expected visibility plane set")
    if widened_width(texel_width) != planes.width:
        raise ValueError(f"plane width {planes.width} does not match {texel_width} texels per row")
    data, was_np = _stage(planes.data, np.uint8, torch.uint8)
    data = data.contiguous()
    h = data.shape[1]
    out = torch.empty((h, texel_width, 2), dtype=torch.uint16, device=data.device)
    if h and texel_width:
        N.call("ps_unpack_visibility", data.data_ptr(), h, texel_width, out.data_ptr(),
               D.stream_ptr(data.device))
    return D.to_numpy(out) if was_np else out


def pack_texels(texels, kind) -> PlaneSet:
    return pack_color(texels) if kind_of(kind) is AtlasKind.COLOR else pack_visibility(texels)


def unpack_texels(planes: PlaneSet, kind, texel_width: int):
    if kind_of(kind) is AtlasKind.COLOR:
        return unpack_color(planes)
    return unpack_visibility(planes, texel_width)


# --- guard band (packing.py:174-202) -------------------------------------------------
# Per-block host utilities kept for API parity; the hot path applies the same
# rule inside the probe-update kernel and the client apply kernel.


def strip_guard_band(block):
    if block.shape[0] != block.shape[1] or block.shape[0] < 3:
        raise ValueError(f"probe block must be square with side >= 3, got {tuple(block.shape)}")
    core = block[1:-1, 1:-1]
    return core.clone() if D.is_tensor(core) else core.copy()


def reconstruct_guard_band(core, out=None):
    n = core.shape[0]
    if core.shape[1] != n or n < 1:
        raise ValueError(f"core must be square, got {tuple(core.shape)}")
    if out is None:
        shape = (n + 2, n + 2) + tuple(core.shape[2:])
        out = (torch.empty(shape, dtype=core.dtype, device=core.device) if D.is_tensor(core)
               else np.empty(shape, dtype=core.dtype))
    flip = (lambda x, d: torch.flip(x, (d,))) if D.is_tensor(core) else (lambda x, d: np.flip(x, d))
    out[1:-1, 1:-1] = core
    out[0, 1:-1] = flip(core[0], 0)
    out[-1, 1:-1] = flip(core[-1], 0)
    out[1:-1, 0] = flip(core[:, 0], 0)
    out[1:-1, -1] = flip(core[:, -1], 0)
    out[0, 0] = core[-1, -1]
    out[0, -1] = core[-1, 0]
    out[-1, 0] = core[0, -1]
    out[-1, -1] = core[0, 0]
    return out


def _signed(t):
    """Same-width signed view (unsigned torch dtypes support few ops)."""
    return t.view({torch.uint16: torch.int16, torch.uint32: torch.int32}.get(t.dtype, t.dtype))


def guard_band_valid(block) -> bool:
    rebuilt = reconstruct_guard_band(block[1:-1, 1:-1])
    if D.is_tensor(block):
        return bool(torch.equal(_signed(rebuilt), _signed(block)))
    return bool(np.array_equal(rebuilt, block))


# --- update-atlas slot cache (packing.py:231-317) --------------------------------------


class UpdateAtlasLayout:
    """Slot allocator for the probe update texture, state resident on the GPU.

    Same contract as the reference: cached probes keep their slot; uncached
    probes take the lowest free slot in ascending id order; with no free slot
    the cached probe outside the selection with the oldest
    ``(last_selected, slot)`` is evicted; overflow raises before any
    mutation.  The state machine runs as scan + sort kernels
    (``ps_assign_slots``) so twin layouts replay identically.

    ``probe_count`` bounds the probe ids the device state can hold; when it
    is not given it grows to fit the ids seen (host inputs) or the source
    atlas (``build_update_atlas``).
    """

    def __init__(self, slot_count: int, core_side: int, slots_per_row: int | None = None,
                 probe_count: int | None = None, device=None) -> None:
        if slot_count < 1:
            raise ValueError("slot_count must be >= 1")
        self.slot_count = slot_count
        self.core_side = core_side
        self.slots_per_row = slots_per_row or math.ceil(math.sqrt(slot_count))
        self.slot_rows = math.ceil(slot_count / self.slots_per_row)
        self._device = torch.device(device) if device is not None else None
        self._cap = 0
        self._probe_slot = None
        self._slot_probe = None
        self._last_selected = None
        self._meta = None
        self._status = None
        self._entries = None
        self._entry_count = None
        if probe_count:
            self._ensure(probe_count)

    # geometry (packing.py:259-281)
    @property
    def width(self) -> int:
        return self.slots_per_row * self.core_side

    @property
    def height(self) -> int:
        return self.slot_rows * self.core_side

    def texel_shape(self, kind) -> tuple:
        if kind_of(kind) is AtlasKind.COLOR:
            return (self.height, self.width)
        return (self.height, self.width, 2)

    def slot_origin(self, slot: int) -> tuple:
        if not (0 <= slot < self.slot_count):
            raise IndexError(f"slot {slot} outside [0, {self.slot_count})")
        r, c = divmod(slot, self.slots_per_row)
        return r * self.core_side, c * self.core_side

    def slot_region(self, texels, slot: int):
        y, x = self.slot_origin(slot)
        s = self.core_side
        return texels[y:y + s, x:x + s]

    # device state
    @property
    def device(self) -> torch.device:
        if self._device is None:
            self._device = D.device_of()
        return self._device

    @property
    def probe_capacity(self) -> int:
        return self._cap

    def _ensure(self, need: int) -> None:
        if need <= self._cap:
            return
        dev = self.device
        cap = max(need, 1)
        ps = torch.full((cap,), -1, dtype=torch.int32, device=dev)
        ls = torch.zeros((cap,), dtype=torch.int64, device=dev)
        if self._probe_slot is not None:
            ps[: self._cap] = self._probe_slot
            ls[: self._cap] = self._last_selected
        else:
            self._slot_probe = torch.full((self.slot_count,), -1, dtype=torch.int32, device=dev)
            self._meta = torch.zeros(4, dtype=torch.int64, device=dev)
            self._status = torch.zeros(1, dtype=torch.int32, device=dev)
            self._entries = torch.empty((self.slot_count, 2), dtype=torch.int64, device=dev)
            self._entry_count = torch.zeros(1, dtype=torch.int64, device=dev)
        self._probe_slot, self._last_selected, self._cap = ps, ls, cap

    def assign_device(self, ids: torch.Tensor, count: torch.Tensor | None = None):
        """Stream-ordered assign: ids int64 CUDA tensor (first ``count`` valid
        when ``count`` is a device scalar).  Returns (entries (S, 2) int64,
        entry_count (1,) int64) device tensors; no host synchronisation.
        Errors are latched in ``self._status`` (see ``raise_pending``)."""
        if self._cap == 0:
            raise ValueError("layout has no probe capacity; pass probe_count")
        ids = ids.to(torch.int64).contiguous()
        nbytes = N.lib().ps_assign_workspace_bytes(self._cap, self.slot_count)
        ws = getattr(self, "_ws", None)
        if ws is None or ws.numel() < nbytes:
            # the layout owns its scratch (sized for its capacity, which only
            # grows before the first device assign)
            ws = self._ws = D.workspace(nbytes, self.device)
        N.call("ps_assign_slots", ids.data_ptr(), D.ptr(count), int(ids.numel()), self._cap,
               self.slot_count, self._probe_slot.data_ptr(), self._slot_probe.data_ptr(),
               self._last_selected.data_ptr(), self._meta.data_ptr(), self._entries.data_ptr(),
               self._entry_count.data_ptr(), self._status.data_ptr(), ws.data_ptr(), ws.numel(),
               D.stream_ptr(self.device))
        return self._entries, self._entry_count

    def assign_bits_device(self, sel_bits: torch.Tensor, pvs_bits: torch.Tensor | None = None):
        """Stream-ordered assign of the probes whose bit is set in ``sel_bits``
        (int32 words over the layout's probe capacity, ANDed with ``pvs_bits``
        when given) -- the same state machine as ``assign`` in two kernels
        (ps_assign_slots_bits), for layouts with a slot per probe
        (slot_count >= probe capacity: no eviction is reachable).  Returns
        (entries, entry_count) device tensors; no host synchronisation."""
        n = self._cap
        if n == 0:
            raise ValueError("layout has no probe capacity; pass probe_count")
        if self.slot_count < n:
            raise ValueError("assign_bits_device needs slot_count >= probe capacity; "
                             "use assign_device")
        if getattr(self, "_ws_bits", None) is None:
            lib = N.lib()
            self._ws_bits = D.workspace(lib.ps_assign_bits_workspace_bytes(n, self.slot_count),
                                        self.device)
            self._plan = torch.zeros(8, dtype=torch.int64, device=self.device)
        N.call("ps_assign_slots_bits", sel_bits.data_ptr(), D.ptr(pvs_bits), n, self.slot_count,
               self._probe_slot.data_ptr(), self._slot_probe.data_ptr(),
               self._last_selected.data_ptr(), self._meta.data_ptr(), self._entries.data_ptr(),
               self._entry_count.data_ptr(), self._plan.data_ptr(), None,
               self._ws_bits.data_ptr(), self._ws_bits.numel(), D.stream_ptr(self.device))
        return self._entries, self._entry_count

    def raise_pending(self) -> None:
        st = int(self._status.item()) if self._status is not None else 0
        if st:
            self._status.zero_()
            if st & N.PS_DEV_SLOT_OVERFLOW:
                raise SlotOverflowError("selection larger than the slot count; "
                                        "budget the selection upstream")
            if st & N.PS_DEV_INDEX:
                raise IndexError("probe id outside the layout's probe range")

    def assign(self, probes) -> list:
        """Assign slots for a selected probe set; returns (slot, probe) pairs
        sorted by slot.  Mutates the cache (packing.py:283-305)."""
        if D.is_tensor(probes):
            ids = probes.to(torch.int64)
            if ids.numel():
                lo, hi = int(ids.min()), int(ids.max())
                if lo < 0:
                    raise IndexError(f"probe id {lo} is negative")
                self._ensure(hi + 1)
        else:
            host = np.asarray(list(probes) if not isinstance(probes, np.ndarray) else probes,
                              dtype=np.int64).reshape(-1)
            uniq = np.unique(host)
            if len(uniq) > self.slot_count:  # reject before mutation (packing.py:287-291)
                raise SlotOverflowError(f"{len(uniq)} probes selected for {self.slot_count} "
                                        "slots; budget the selection upstream")
            if len(uniq) and uniq[0] < 0:
                raise IndexError(f"probe id {int(uniq[0])} is negative")
            self._ensure(int(uniq[-1]) + 1 if len(uniq) else 1)
            ids = torch.from_numpy(host).to(self.device)
        entries, count = self.assign_device(ids)
        self.raise_pending()
        n = int(count.item())
        e = entries[:n].cpu()
        return list(zip(e[:, 0].tolist(), e[:, 1].tolist()))

    # dict views for API parity with the reference attributes
    @property
    def probe_slot(self) -> dict:
        if self._cap == 0:
            return {}
        ps = self._probe_slot.cpu().numpy()
        ids = np.nonzero(ps >= 0)[0]
        return {int(p): int(ps[p]) for p in ids}

    @property
    def slot_probe(self) -> dict:
        if self._cap == 0:
            return {}
        sp = self._slot_probe.cpu().numpy()
        return {int(s): int(sp[s]) for s in np.nonzero(sp >= 0)[0]}

    @property
    def last_selected(self) -> dict:
        if self._cap == 0:
            return {}
        ls = self._last_selected.cpu().numpy()
        return {int(p): int(ls[p]) for p in np.nonzero(ls > 0)[0]}


def _atlas_parts(source):
    kind = kind_of(source.kind)
    return kind, int(source.probe_count), int(source.probes_per_row)


def build_update_atlas(selected, layout: UpdateAtlasLayout, source, update_texels=None):
    """Write selected probes' stripped cores into their slots (packing.py:320-338).

    ``update_texels`` persists across calls and is mutated in place; slots of
    unselected cached probes keep their contents.  Returns the texel array
    and the (slot, probe) entries sorted by slot.
    """
    kind, n, ppr = _atlas_parts(source)
    src_t, src_np = _stage(source.texels, source.dtype if hasattr(source, "dtype") else
                           (np.uint32 if kind is AtlasKind.COLOR else np.uint16),
                           torch.uint32 if kind is AtlasKind.COLOR else torch.uint16)
    src_t = src_t.contiguous()
    dev = src_t.device
    if layout._device is None:
        layout._device = dev
    layout._ensure(n)
    shape = layout.texel_shape(kind)
    tdt = torch.uint32 if kind is AtlasKind.COLOR else torch.uint16
    out_np = None
    if update_texels is None:
        upd = torch.zeros(shape, dtype=tdt, device=dev)
        if src_np:
            out_np = np.zeros(shape, dtype=np.uint32 if kind is AtlasKind.COLOR else np.uint16)
    elif D.is_tensor(update_texels):
        if tuple(update_texels.shape) != shape:
            raise ValueError(f"update texels {tuple(update_texels.shape)} != layout {shape}")
        upd = update_texels
    else:
        if update_texels.shape != shape:
            raise ValueError(f"update texels {update_texels.shape} != layout {shape}")
        out_np = update_texels
        upd = torch.from_numpy(np.ascontiguousarray(update_texels)).to(dev)
    if not upd.is_contiguous():
        raise ValueError("update texels must be contiguous")
    if D.is_tensor(selected):
        ids = selected.to(device=dev, dtype=torch.int64)
        if ids.numel() and (int(ids.min()) < 0 or int(ids.max()) >= n):
            raise IndexError("selected probe outside the source atlas")
    else:
        host = np.asarray(selected if isinstance(selected, (np.ndarray, list, tuple))
                          else list(selected), dtype=np.int64).reshape(-1)
        uniq = np.unique(host)
        if len(uniq) > layout.slot_count:
            raise SlotOverflowError(f"{len(uniq)} probes selected for {layout.slot_count} "
                                    "slots; budget the selection upstream")
        if len(uniq) and (uniq[0] < 0 or uniq[-1] >= n):
            raise IndexError("selected probe outside the source atlas")
        ids = torch.from_numpy(host).to(dev)
    entries, count = layout.assign_device(ids)
    layout.raise_pending()
    N.call("ps_build_update", kind.native, src_t.data_ptr(), n, ppr, entries.data_ptr(),
           count.data_ptr(), layout.slot_count, layout.slots_per_row, upd.data_ptr(),
           shape[1], None, None, 0, None, D.stream_ptr(dev))
    k = int(count.item())
    e = entries[:k].cpu()
    ent = list(zip(e[:, 0].tolist(), e[:, 1].tolist()))  # [(slot, probe), ...] by slot
    if out_np is not None:
        out_np[...] = D.to_numpy(upd)
        return out_np, ent
    return upd, ent


def apply_update_entries_device(entries: torch.Tensor, entry_count: torch.Tensor,
                                update_texels: torch.Tensor, layout: UpdateAtlasLayout,
                                target) -> None:
    """Stream-ordered client apply: (slot, probe) int64 entries (first
    ``entry_count`` valid) from the update atlas into ``target`` (a device
    ProbeAtlas), guard bands rebuilt on the GPU."""
    kind = kind_of(target.kind)
    N.call("ps_apply_entries", kind.native, update_texels.data_ptr(), update_texels.shape[1],
           layout.slots_per_row, entries.data_ptr(), entry_count.data_ptr(), entries.shape[0],
           target.texels.data_ptr(), target.probes_per_row, D.stream_ptr(update_texels.device))


def apply_update_entries(entries, update_texels, layout: UpdateAtlasLayout, target) -> None:
    """Client-side apply (packing.py:341-350): slot cores into target blocks
    with rebuilt guard bands (mutates ``target``)."""
    kind = kind_of(target.kind)
    tdt = torch.uint32 if kind is AtlasKind.COLOR else torch.uint16
    npd = np.uint32 if kind is AtlasKind.COLOR else np.uint16
    dev = D.device_of(update_texels, target.texels)
    ent = torch.as_tensor(np.asarray(list(entries), dtype=np.int64).reshape(-1, 2), device=dev)
    cnt = torch.tensor([ent.shape[0]], dtype=torch.int64, device=dev)
    upd = (update_texels.contiguous() if D.is_tensor(update_texels)
           else torch.from_numpy(np.ascontiguousarray(update_texels, dtype=npd)).to(dev))
    on_host = not D.is_tensor(target.texels)
    dst = (torch.from_numpy(np.ascontiguousarray(target.texels)).to(dev) if on_host
           else target.texels)
    if not dst.is_contiguous():
        raise ValueError("target atlas texels must be contiguous")
    if ent.shape[0]:
        if int(ent[:, 1].min()) < 0 or int(ent[:, 1].max()) >= target.probe_count:
            raise IndexError("entry probe outside the target atlas")
        if int(ent[:, 0].min()) < 0 or int(ent[:, 0].max()) >= layout.slot_count:
            raise IndexError("entry slot outside the layout")
        view = type("A", (), {"kind": kind, "texels": dst, "probes_per_row": target.probes_per_row})
        apply_update_entries_device(ent, cnt, upd.view(tdt) if upd.dtype != tdt else upd, layout, view)
    if on_host:
        target.texels[...] = D.to_numpy(dst)
