"""Change detection and budgeted selection on the GPU.

Drop-in mirror of ``probestream.selection.detect_changed`` (selection.py:284-323)
and ``select_for_client`` (selection.py:413-437).  numpy atlases are staged to
the device and the reference's return types come back (int64 numpy ids,
python list); CUDA-tensor atlases return CUDA tensors.  The kernels live in
``csrc/ps_detect.cu`` and ``csrc/ps_select.cu``.

``*_device`` variants keep everything stream-ordered (bitmaps and
device-side counts, no host synchronisation) for the frame pipeline.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .errors import LayoutMismatchError
from .volume import AtlasKind, kind_of

__all__ = ["LayoutMismatchError", "detect_changed", "detect_changed_device",
           "select_for_client", "select_device", "ids_to_bits", "bits_to_ids"]


def _threshold_args(threshold):
    """(value, is_f64): a numpy float64 scalar promotes the reference's
    visibility comparison to float64; python scalars are weak (float32)."""
    is64 = isinstance(threshold, (np.float64, np.longdouble))
    return float(threshold), int(is64)


def _atlas_tensor(atlas, device):
    kind = kind_of(atlas.kind)
    tdt = torch.uint32 if kind is AtlasKind.COLOR else torch.uint16
    t = atlas.texels
    if D.is_tensor(t):
        t = t.to(device) if t.device != device else t
        if t.dtype != tdt:
            t = t.view(tdt) if t.element_size() == tdt.itemsize else t.to(tdt)
        return t.contiguous(), False
    npd = np.uint32 if kind is AtlasKind.COLOR else np.uint16
    return torch.from_numpy(np.ascontiguousarray(np.asarray(t, dtype=npd))).to(device), True


def _check_layout(rendered, last_sent, volume):
    # selection.py:295-302
    if (kind_of(rendered.kind) != kind_of(last_sent.kind)
            or rendered.probe_count != last_sent.probe_count
            or rendered.probes_per_row != last_sent.probes_per_row):
        raise LayoutMismatchError("atlases do not share a layout")
    if rendered.probe_count != volume.probe_count:
        raise LayoutMismatchError("atlas probe count does not match volume")


def detect_changed_device(rendered, last_sent, volume, threshold=0.0, *, bits=None,
                          ids=None, count=None, with_ids=True, workspace_slot="detect",
                          probe_range=None, active=None):
    """Stream-ordered detection.  Returns (changed_bits uint32[(N+31)/32],
    ids int64[N] (first ``count`` valid) or None, count int64[1] or None).
    ``probe_range`` restricts the test to a z-slab [begin, end)."""
    _check_layout(rendered, last_sent, volume)
    dev = D.device_of(rendered.texels, last_sent.texels)
    a, _ = _atlas_tensor(rendered, dev)
    b, _ = _atlas_tensor(last_sent, dev)
    n = rendered.probe_count
    ppr = rendered.probes_per_row
    block_rows = -(-n // ppr)
    side = kind_of(rendered.kind).block_side
    if a.shape[0] != block_rows * side or a.shape[1] != ppr * side:
        raise LayoutMismatchError("atlas texels do not match the layout")
    words = (n + 31) // 32
    if bits is None:
        bits = torch.empty(words, dtype=torch.int32, device=dev)
    if with_ids:
        if ids is None:
            ids = torch.empty(n, dtype=torch.int64, device=dev)
        if count is None:
            count = torch.empty(1, dtype=torch.int64, device=dev)
    ws = D.Workspace.get(N.lib().ps_detect_workspace_bytes(n), dev, workspace_slot)
    thr, is64 = _threshold_args(threshold)
    if active is None:
        active = D.active_flags(volume, dev)
    begin, end = probe_range if probe_range is not None else (0, n)
    N.call("ps_detect_changed_range", kind_of(rendered.kind).native, a.data_ptr(), b.data_ptr(),
           n, ppr, block_rows, begin, end, active.data_ptr(), thr, is64, bits.data_ptr(),
           D.ptr(ids) if with_ids else None, D.ptr(count) if with_ids else None,
           ws.data_ptr(), ws.numel(), D.stream_ptr(dev))
    return bits, (ids if with_ids else None), (count if with_ids else None)


def detect_changed(rendered, last_sent, volume, threshold: float = 0.0):
    """Probe ids whose blocks differ from their last transmitted state.

    Threshold 0 is an exact comparison: any bit difference marks the probe.
    Inactive probes are never reported.
    """
    _check_layout(rendered, last_sent, volume)
    was_np = not (D.is_tensor(rendered.texels) or D.is_tensor(last_sent.texels))
    _, ids, count = detect_changed_device(rendered, last_sent, volume, threshold)
    k = int(count.item())
    out = ids[:k]
    return D.to_numpy(out) if was_np else out


# --- id list <-> bitmap ---------------------------------------------------------------


def ids_to_bits(ids, probe_count: int, device=None, count=None, status=None):
    dev = device or D.device_of(ids)
    t = D.to_device(ids, torch.int64, dev).reshape(-1)
    bits = torch.zeros((probe_count + 31) // 32, dtype=torch.int32, device=dev)
    if status is None:
        status = torch.zeros(1, dtype=torch.int32, device=dev)
    if t.numel():
        N.call("ps_ids_to_bits", t.data_ptr(), D.ptr(count), int(t.numel()), probe_count,
               bits.data_ptr(), status.data_ptr(), D.stream_ptr(dev))
    return bits, status


def bits_to_ids(bits, probe_count: int):
    dev = bits.device
    ids = torch.empty(probe_count, dtype=torch.int64, device=dev)
    count = torch.empty(1, dtype=torch.int64, device=dev)
    ws = D.Workspace.get(N.lib().ps_compact_workspace_bytes(probe_count), dev, "compact")
    N.call("ps_bits_to_ids", bits.data_ptr(), probe_count, ids.data_ptr(), count.data_ptr(),
           ws.data_ptr(), ws.numel(), D.stream_ptr(dev))
    return ids, count


# --- budgeted selection ----------------------------------------------------------------


def select_device(changed_bits, pvs_bits, volume, last_sent_seq, current_seq: int,
                  budget=None, *, out_ids=None, out_count=None, workspace_slot="select",
                  ordered: bool = True, active=None):
    """Stream-ordered selection over bitmaps; pvs_bits None means every probe.
    Returns (ids int64[N], count int64[1]) with the first count ids valid, in
    staleness order (``ordered``) or, without a budget, ascending id order --
    the same set, for callers that only need the set."""
    dev = changed_bits.device
    n = volume.probe_count
    seq = D.to_device(last_sent_seq, torch.int64, dev)
    if seq.numel() < n:
        raise IndexError("last_sent_seq shorter than the probe count")
    if out_ids is None:
        out_ids = torch.empty(n, dtype=torch.int64, device=dev)
    if out_count is None:
        out_count = torch.empty(1, dtype=torch.int64, device=dev)
    ws = D.Workspace.get(N.lib().ps_select_workspace_bytes(n), dev, workspace_slot)
    has_budget = budget is not None
    if active is None:
        active = D.active_flags(volume, dev)
    N.call("ps_select", changed_bits.data_ptr(), D.ptr(pvs_bits), active.data_ptr(),
           seq.data_ptr(), int(current_seq), n, int(has_budget), int(budget) if has_budget else 0, int(bool(ordered)), out_ids.data_ptr(),
           out_count.data_ptr(), ws.data_ptr(), ws.numel(), D.stream_ptr(dev))
    return out_ids, out_count


def _host_index_check(changed, pvs, n):
    """The reference only indexes ``volume.active[p]`` for ids present in both
    sets (selection.py:428-433), so an out-of-range id raises IndexError only
    there.  (Negative ids wrap in numpy; the drop-in rejects them.)"""
    c = np.unique(np.asarray(changed, dtype=np.int64).reshape(-1))
    p = np.unique(np.asarray(pvs, dtype=np.int64).reshape(-1))
    both = np.intersect1d(c, p)
    bad = both[(both < 0) | (both >= n)]
    if bad.size:
        raise IndexError(f"index {int(bad[0])} is out of bounds for {n} probes")


def select_for_client(changed, pvs, volume, last_sent_seq, current_seq: int, budget=None):
    """Order the sendable set by staleness and truncate to the budget.

    Staleness is update sequences since last transmission (never-sent probes
    are the most stale); ties break on ascending probe id.
    """
    n = volume.probe_count
    dev = D.device_of(changed, pvs, last_sent_seq)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    cb, status = ids_to_bits(changed, n, dev, status=status)
    pb, status = ids_to_bits(pvs, n, dev, status=status)
    if int(status.item()) & N.PS_DEV_INDEX:
        to_np = (lambda x: D.to_numpy(x) if D.is_tensor(x) else x)
        _host_index_check(to_np(changed), to_np(pvs), n)
    ids, count = select_device(cb, pb, volume, last_sent_seq, current_seq, budget)
    k = int(count.item())
    return ids[:k].cpu().tolist()


# --- potentially visible set (selection.py:174-249, 329-407) --------------------------

RAY_EPS = 1e-6  # selection.py:22


class CameraPose:
    """Client camera (selection.py:177-222): position, unit forward, up, fov, aspect."""

    def __init__(self, position, forward, up=(0.0, 1.0, 0.0), fov_y_deg: float = 90.0,
                 aspect: float = 1.0):
        self.position = np.asarray(position, dtype=np.float64)
        f = np.asarray(forward, dtype=np.float64)
        length = np.linalg.norm(f)
        if length < 1e-9:
            raise ValueError("camera forward vector must be nonzero")
        self.forward = f / length
        self.up = np.asarray(up, dtype=np.float64)
        self.fov_y_deg = fov_y_deg
        self.aspect = aspect

    def basis(self):
        f = self.forward
        right = np.cross(f, self.up)
        for fallback in (np.array([1.0, 0.0, 0.0]), np.array([0.0, 0.0, 1.0])):
            if np.linalg.norm(right) >= 1e-9:
                break
            right = np.cross(f, fallback)  # up parallel to forward
        right = right / np.linalg.norm(right)
        return f, right, np.cross(right, f)


class SelectionParams:
    """selection.py:255-267."""

    def __init__(self, change_threshold: float = 0.0, sphere_rays: int = 1024,
                 raster_cols: int = 64, raster_rows: int = 64, budget=None):
        if raster_cols * raster_rows < 1 and sphere_rays < 1:
            raise ValueError("at least one ray is required")
        if budget is not None and budget < 0:
            raise ValueError("budget must be >= 0")
        self.change_threshold = change_threshold
        self.sphere_rays = sphere_rays
        self.raster_cols = raster_cols
        self.raster_rows = raster_rows
        self.budget = budget


def frustum_directions(pose: CameraPose, cols: int, rows: int) -> np.ndarray:
    """Unit directions through the centres of a cols x rows frustum grid."""
    f, r, u = pose.basis()
    ty = np.tan(np.radians(pose.fov_y_deg) / 2.0)
    tx = ty * pose.aspect
    sx = (np.arange(cols) + 0.5) / cols * 2.0 - 1.0
    sy = (np.arange(rows) + 0.5) / rows * 2.0 - 1.0
    gx, gy = np.meshgrid(sx, sy, indexing="xy")
    d = f[None, :] + (gx.reshape(-1, 1) * tx) * r[None, :] + (gy.reshape(-1, 1) * ty) * u[None, :]
    return d / np.linalg.norm(d, axis=1, keepdims=True)


def fibonacci_sphere(count: int) -> np.ndarray:
    from .probes import fibonacci_sphere as _fib

    return _fib(count)


def pvs_rays(pose: CameraPose, params: SelectionParams) -> np.ndarray:
    parts = []
    if params.raster_cols > 0 and params.raster_rows > 0:
        parts.append(frustum_directions(pose, params.raster_cols, params.raster_rows))
    if params.sphere_rays > 0:
        parts.append(fibonacci_sphere(params.sphere_rays))
    return np.concatenate(parts) if parts else np.zeros((0, 3))


def cage_probes(points, volume) -> np.ndarray:
    """The 8 corner probe ids of the cell enclosing each point (clamped);
    host helper for small point sets -- the GPU PVS kernel does the same per
    hit point."""
    p = np.atleast_2d(np.asarray(points, dtype=np.float64))
    dims = np.asarray(volume.dims)
    rel = (p - np.asarray(volume.origin)) / np.asarray(volume.spacing)
    low = np.clip(np.floor(rel).astype(np.int64), 0, np.maximum(dims - 2, 0))
    nx, ny, _ = volume.dims
    out = np.empty((len(p), 8), dtype=np.int64)
    col = 0
    for dk in (0, 1):
        for dj in (0, 1):
            for di in (0, 1):
                ijk = np.minimum(low + np.array([di, dj, dk]), dims - 1)
                out[:, col] = ijk[:, 0] + nx * (ijk[:, 1] + ny * ijk[:, 2])
                col += 1
    return out


def probes_for_point(point, volume) -> set:
    return set(int(p) for p in cage_probes(np.asarray(point), volume)[0])


_PVS_SCENES: dict = {}


def _pvs_scene(scene, device):
    """DeviceScene + float64 vertex table for a scene (cached per object)."""
    from .scene import DeviceScene, Scene

    key = (id(scene), str(device))
    hit = _PVS_SCENES.get(key)
    if hit is not None and hit[0] is scene:
        return hit[1], hit[2]
    if isinstance(scene, DeviceScene):
        ds = scene
        verts = ds.scene.vertices
    else:
        if not isinstance(scene, Scene):  # the reference's SceneGeometry
            boxes = getattr(scene, "boxes", np.zeros((0, 2, 3)))
            if len(boxes):
                raise ValueError("the GPU PVS supports triangle scenes; triangulate boxes")
            tris = np.asarray(scene.triangles, dtype=np.float64).reshape(-1, 3, 3)
            n = len(tris)
            scene = Scene(tris, np.zeros((n, 3), np.float32), np.zeros((n, 3), np.float32))
        ds = scene.device(device)
        verts = scene.vertices
    v64 = torch.from_numpy(np.ascontiguousarray(verts, dtype=np.float64)).to(device)
    _PVS_SCENES[key] = (scene, ds, v64)
    return ds, v64


def pvs_probes_device(pose: CameraPose, scene, volume, params: SelectionParams, rays=None,
                      *, bits=None, ids=None, count=None):
    """Stream-ordered PVS: returns (active-masked bitmap, ids, count) on the device."""
    dev = D.device_of()
    if rays is None:
        rays = pvs_rays(pose, params)
    rays = np.ascontiguousarray(np.asarray(rays, dtype=np.float64).reshape(-1, 3))
    ds, v64 = _pvs_scene(scene, dev)
    n = volume.probe_count
    if bits is None:
        bits = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
    if ids is None:
        ids = torch.empty(n, dtype=torch.int64, device=dev)
    if count is None:
        count = torch.empty(1, dtype=torch.int64, device=dev)
    d_rays = torch.from_numpy(rays).to(dev) if len(rays) else torch.zeros((1, 3), dtype=torch.float64, device=dev)
    # camera / volume placement are host scalars of the call (C doubles)
    cam = np.ascontiguousarray(np.asarray(pose.position, dtype=np.float64).reshape(3))
    vo = np.ascontiguousarray(np.asarray(volume.origin, dtype=np.float64).reshape(3))
    vs = np.ascontiguousarray(np.asarray(volume.spacing, dtype=np.float64).reshape(3))
    ws = D.Workspace.get(N.lib().ps_pvs_workspace_bytes(n), dev, "pvs")
    nx, ny, nz = volume.dims
    N.call("ps_pvs", ds.nodes.data_ptr(), ds.width, ds.tris.data_ptr(), v64.data_ptr(),
           d_rays.data_ptr(), len(rays), cam.ctypes.data, nx, ny, nz, vo.ctypes.data, vs.ctypes.data,
           D.active_flags(volume, dev).data_ptr(), bits.data_ptr(), ids.data_ptr(), count.data_ptr(),
           ws.data_ptr(), ws.numel(), D.stream_ptr(dev))
    return bits, ids, count


def pvs_probes(pose: CameraPose, scene, volume, params: SelectionParams, rays=None) -> np.ndarray:
    """Active probes that could shade any point visible from the camera
    (selection.py:384-407); ascending int64 ids."""
    _, ids, count = pvs_probes_device(pose, scene, volume, params, rays)
    return D.to_numpy(ids[: int(count.item())])
