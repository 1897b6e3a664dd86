"""Stages (1)+(2): per-probe ray generation, BVH tracing and the DDGI blend.

New API surface (the reference has no implementation of these stages,
SURVEY F3/F4); it emits the reference's atlas types so stages (3)+(4)
consume its output unchanged.  The algorithm, fixed here and restated
independently by ``oracle/ddgi.py``:

Ray set (host, float64 -> float32): the base set is
``fibonacci_sphere(R)`` (selection.py:241-249) in a fixed coherence order
(sorted by the Morton code of its octahedral uv, so a warp's 32 rays cover a
small solid angle); frame ``f`` rotates it by the uniformly random rotation
drawn from ``np.random.default_rng(seed + f)`` (unit quaternion from 4
normals).  Every probe uses the same rotated set, as in DDGI.

Tracing (device): ray origin = probe position (volume.py:127-138), nearest
hit with the reference raycast semantics (selection.py:66-149).  A hit is
shaded ``emission + albedo * sum_l I_l * cos / d^2 * V_l`` with the normal
facing the ray and the light seen from ``s = hit + bias * n``; a miss
returns the sky colour.  Depth = ``min(t, max_distance)`` (miss:
``max_distance``).  ``V_l`` (``shadows``):
  "map"  -- default, as the paper's server (shadow-mapped direct light,
            PAPER.md:370): each frame a cube distance map of side S is traced
            from every light (face f: axis f//2, sign -1 if f odd; texel
            (i, j) looks along e_a*sign + e_b*u + e_c*w, u = (i+.5)/S*2-1,
            w = (j+.5)/S*2-1, b, c = a+1, a+2 mod 3); V = |light - s| <=
            map[face, texel of (s - light)] * (1 + shadow_bias);
  "rays" -- an exact any-hit shadow ray s -> light;
  "none" -- V = 1.

Blend (device): colour texel t (8x8, texel_directions) averages radiance
with weights ``max(0, n_t . d_r)``; depth texel t (16x16) averages depth and
depth^2 with ``max(0, n_t . d_r)^sharpness`` (plain float32 weights); the
tensor-core blend (csrc/ps_blend_tc.cu) is fp32-accurate by 3xTF32 (weights
and ray channels split hi + lo); state = fma(h, prev - frame, frame) (h = 0
on the first frame); a texel no ray reaches keeps its state.
Output: colour unorm10 of ``state / irradiance_scale`` (round to nearest
even), visibility raw float16 halves; border texels by the guard-band rule
(packing.py:180-196).
"""

from __future__ import annotations

import ctypes
import functools
import math
import os

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .scene import DeviceScene, Scene
from .volume import AtlasKind, ProbeAtlas, ProbeVolume, oct_encode, texel_directions


def fibonacci_sphere(count: int) -> np.ndarray:
    """selection.py:241-249 (float64)."""
    if count < 1:
        return np.zeros((0, 3))
    i = np.arange(count, dtype=np.float64) + 0.5
    z = 1.0 - 2.0 * i / count
    rad = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    th = np.pi * (1.0 + np.sqrt(5.0)) * i
    return np.stack([rad * np.cos(th), rad * np.sin(th), z], axis=1)


def _morton2(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    def spread(v):
        v = v.astype(np.uint32) & np.uint32(0xFFFF)
        v = (v | (v << np.uint32(8))) & np.uint32(0x00FF00FF)
        v = (v | (v << np.uint32(4))) & np.uint32(0x0F0F0F0F)
        v = (v | (v << np.uint32(2))) & np.uint32(0x33333333)
        v = (v | (v << np.uint32(1))) & np.uint32(0x55555555)
        return v
    return spread(x) | (spread(y) << np.uint32(1))


@functools.lru_cache(maxsize=8)
def _base_ray_set(count: int) -> np.ndarray:
    fib = fibonacci_sphere(count)
    uv = oct_encode(fib, validate=False)
    q = np.clip((uv * 1024.0).astype(np.int64), 0, 1023)
    order = np.argsort(_morton2(q[:, 0], q[:, 1]), kind="stable")
    out = fib[order]
    out.setflags(write=False)
    return out


def base_ray_set(count: int) -> np.ndarray:
    """fibonacci_sphere(count) reordered by octahedral Morton code (float64)."""
    return _base_ray_set(int(count)).copy()


def frame_rotation(seed: int, frame: int) -> np.ndarray:
    """Uniform random rotation for a frame: unit quaternion from 4 normals."""
    q = np.random.default_rng(seed + frame).normal(size=4)
    w, x, y, z = q / np.linalg.norm(q)
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
        [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
        [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)],
    ])


def frame_ray_directions(count: int, seed: int, frame: int) -> np.ndarray:
    """(count, 4) float32 table [dx dy dz 0] for a frame."""
    d = _base_ray_set(int(count)) @ frame_rotation(seed, frame).T
    out = np.zeros((count, 4), np.float32)
    out[:, :3] = d
    return out


def texel_direction_table() -> np.ndarray:
    """(320, 4) float32: 64 colour texel directions then 256 depth ones."""
    out = np.zeros((320, 4), np.float32)
    out[:64, :3] = texel_directions(8).reshape(-1, 3)
    out[64:, :3] = texel_directions(16).reshape(-1, 3)
    return out


EARLY_SHADOWS = os.environ.get("PS_EARLY_SHADOWS", "1") != "0"


class ProbeUpdater:
    """Owns the float probe state and the two output atlases on one GPU and
    updates a contiguous probe range per frame (``probe_range`` = a z-slab
    when sharded across GPUs).  ``update`` launches two kernels and never
    synchronises."""

    def __init__(self, volume: ProbeVolume, scene: Scene | DeviceScene, rays_per_probe: int = 256,
                 hysteresis: float = 0.97, sharpness: float = 50.0, max_distance: float | None = None,
                 irradiance_scale: float = 1.0, shadows="map", normal_bias: float | None = None,
                 seed: int = 0, probe_range=None, probes_per_row: int | None = None,
                 device=None, record_rays: bool = False, shadow_map_size: int = 256,
                 shadow_bias: float = 0.02, atlas_buffers: int = 1, reserve_sms: int = 0):
        self.volume = volume
        self.device = torch.device(device) if device is not None else D.device_of()
        self.dscene = scene if isinstance(scene, DeviceScene) else scene.device(self.device)
        sc = self.dscene.scene
        (x0, y0, z0), (x1, y1, z1) = sc.bounds
        diag = math.sqrt((x1 - x0) ** 2 + (y1 - y0) ** 2 + (z1 - z0) ** 2)
        self.rays_per_probe = int(rays_per_probe)
        self.hysteresis = float(hysteresis)
        self.sharpness = float(sharpness)
        self.max_distance = float(max_distance if max_distance is not None else diag)
        self.irradiance_scale = float(irradiance_scale)
        # shadows: "map" (cube distance maps traced from each light, the
        # paper's shadow-mapped server), "rays" (exact shadow rays), "none";
        # booleans map True -> "rays", False -> "none"
        if shadows is True:
            shadows = "rays"
        elif shadows is False or shadows is None:
            shadows = "none"
        self.shadow_mode = {"none": N.PS_SHADOW_NONE, "rays": N.PS_SHADOW_RAYS,
                            "map": N.PS_SHADOW_MAP}[shadows]
        self.shadows = shadows
        self.shadow_map_size = int(shadow_map_size)
        self.shadow_bias = float(shadow_bias)
        self.reserve_sms = int(reserve_sms)
        self.normal_bias = float(normal_bias if normal_bias is not None else 1e-3 * diag)
        self.seed = int(seed)
        n = volume.probe_count
        self.probe_begin, self.probe_end = probe_range if probe_range is not None else (0, n)
        nloc = self.probe_end - self.probe_begin
        dev = self.device
        self.irradiance = torch.zeros((max(nloc, 1), 64, 3), dtype=torch.float32, device=dev)
        self.moments = torch.zeros((max(nloc, 1), 256, 2), dtype=torch.float32, device=dev)
        # atlas_buffers = 2 lets frame f+1 be traced while the streaming
        # stages still read frame f's atlases (server overlap)
        self._color_bufs = [ProbeAtlas(AtlasKind.COLOR, n, probes_per_row, device=dev)
                            for _ in range(atlas_buffers)]
        self._vis_bufs = [ProbeAtlas(AtlasKind.VISIBILITY, n, probes_per_row, device=dev)
                          for _ in range(atlas_buffers)]
        self.color, self.visibility = self._color_bufs[0], self._vis_bufs[0]
        R = self.rays_per_probe
        self.texdir = torch.from_numpy(texel_direction_table()).to(dev)
        self.w_color = torch.empty((R, 64), dtype=torch.float32, device=dev)
        self.w_depth = torch.empty((R, 256), dtype=torch.float32, device=dev)
        self.inv_wsum = torch.empty(320, dtype=torch.float32, device=dev)
        # tensor-core blend operand image (rays % 8 == 0); None -> CUDA-core blend
        nimg = N.lib().ps_blend_weight_image_floats(R)
        self.w_image = torch.empty(nimg, dtype=torch.float32, device=dev) if nimg else None
        self.ray_dirs = torch.empty((R, 4), dtype=torch.float32, device=dev)
        # double-buffered pinned staging for the per-frame ray table
        self._pinned_dirs = [torch.empty((R, 4), dtype=torch.float32).pin_memory() for _ in range(2)]
        self._pinned_evt = [None, None]
        self.ray_records = (torch.empty((max(nloc, 1) * R, 8), dtype=torch.float32, device=dev)
                            if record_rays else None)
        self.records = torch.empty((max(nloc, 1) * R, 4), dtype=torch.float32, device=dev)
        self.work_counter = torch.zeros(1, dtype=torch.int32, device=dev)
        S = self.shadow_map_size
        self.shadow_maps = (torch.empty((self.dscene.MAX_LIGHTS, 6, S, S), dtype=torch.float32,
                                        device=dev) if self.shadow_mode == N.PS_SHADOW_MAP else None)
        self.frames_done = 0
        # CUDA-graph replay (enable_graphs): one graph per frame parity; the
        # ray table and lights still go H2D every frame, from per-parity
        # pinned buffers the graph's copy nodes read
        self.graphs = None
        self._graph_evt = [None, None]
        self._pinned_lights = None
        # sharded shadow maps (set by the sharded frame): (rank, world, group);
        # each rank traces a slice of the map texels and the slices are
        # all-gathered before the probe rays are traced
        self.shadow_split = None
        # peer-memory variant (set_shadow_peers): the slice is stored straight
        # into every rank's mapped maps, ordered by flags -- no collective
        self.shadow_peer = None

    def enable_graphs(self, on: bool = True) -> None:
        self.graphs = {} if on else None
        # early shadow maps (graphed, unsharded): frame f+1's lights copy and
        # shadow maps replay on a side stream as soon as frame f's trace is
        # done, so they overlap frame f's blend; the trace of f+1 waits for
        # them.  PS_EARLY_SHADOWS=0 keeps them inside the frame graph (tuning)
        self._early = (on and self.shadow_mode == N.PS_SHADOW_MAP and EARLY_SHADOWS)
        self._shadow_stream = torch.cuda.Stream(self.device) if self._early else None
        self._trace_done = None

    def set_shadow_peers(self, rank: int, world: int, group=None) -> None:
        """Shard the shadow-map pass over the process group through peer
        memory: two-parity maps mapped into every rank (CUDA IPC), the shadow
        kernel stores its texel slice into all of them, then a release flag per
        rank and an acquire wait before the probe rays are traced."""
        from .distributed import PeerBuffers

        if self.shadow_mode != N.PS_SHADOW_MAP or world < 2:
            return
        dev = self.device
        maps2 = torch.empty((2,) + tuple(self.shadow_maps.shape), dtype=torch.float32, device=dev)
        flags = torch.zeros(world, dtype=torch.int64, device=dev)
        pb = PeerBuffers({"maps": maps2, "flags": flags}, rank, world, group)
        per = self.shadow_maps.numel() * 4
        ptr = lambda xs: torch.tensor(xs, dtype=torch.int64, device=dev)
        self.shadow_peer = {
            "maps2": maps2, "flags": flags, "pb": pb,
            "dst": [ptr([m + k * per for m in pb.ptrs["maps"]]) for k in range(2)],
            "sig": ptr([f + rank * 8 for f in pb.ptrs["flags"]]),
            "state": torch.zeros(3, dtype=torch.int64, device=dev),
        }
        self.shadow_split = (rank, world, group)

    def _shadow_slice(self):
        """(begin, end, chunk) of this rank's map texels, or None when unsharded."""
        if (self.shadow_split is None or self.shadow_mode != N.PS_SHADOW_MAP
                or self.dscene.light_count == 0):
            return None
        rank, world = self.shadow_split[:2]
        S = self.shadow_map_size
        total = self.dscene.light_count * 6 * S * S
        chunk = -(-total // world)
        if chunk * world > self.shadow_maps.numel():
            return None  # no room for the padded gather: every rank traces all texels
        return rank * chunk, min((rank + 1) * chunk, total), chunk

    def _params(self, hysteresis: float, passes: int = 0, texels=None, shadow_maps=None,
                shadow_dst=None, ndst: int = 0) -> N.TraceParams:
        v, s = self.volume, self.dscene
        p = N.TraceParams()
        p.nx, p.ny, p.nz = v.dims
        p.probe_begin, p.probe_end = self.probe_begin, self.probe_end
        p.origin = (ctypes.c_double * 3)(*map(float, v.origin))
        p.spacing = (ctypes.c_double * 3)(*map(float, v.spacing))
        p.ray_dirs = self.ray_dirs.data_ptr()
        p.rays_per_probe = self.rays_per_probe
        p.nodes, p.tris, p.materials = s.nodes.data_ptr(), s.tris.data_ptr(), s.materials.data_ptr()
        p.bvh_width = s.width
        p.light_count = s.light_count
        p.lights = s.lights.data_ptr()
        p.sky = (ctypes.c_float * 3)(*map(float, s.scene.sky))
        p.max_distance = self.max_distance
        p.normal_bias = self.normal_bias
        p.shadow_mode = self.shadow_mode
        p.shadow_map_size = self.shadow_map_size
        maps = shadow_maps if shadow_maps is not None else self.shadow_maps
        p.shadow_maps = maps.data_ptr() if maps is not None else None
        p.shadow_dst = D.ptr(shadow_dst)
        p.shadow_ndst = ndst
        p.shadow_bias = self.shadow_bias
        p.passes = passes
        if texels is not None:
            p.shadow_texel_begin, p.shadow_texel_end = texels
        p.records = self.records.data_ptr()
        p.work_counter = self.work_counter.data_ptr()
        p.reserve_sms = self.reserve_sms
        p.w_color, p.w_depth, p.inv_wsum = (self.w_color.data_ptr(), self.w_depth.data_ptr(),
                                            self.inv_wsum.data_ptr())
        p.w_image = D.ptr(self.w_image)
        p.hysteresis = hysteresis
        p.irradiance_scale = self.irradiance_scale
        p.irradiance, p.moments = self.irradiance.data_ptr(), self.moments.data_ptr()
        p.color_atlas = self.color.texels.data_ptr()
        p.vis_atlas = self.visibility.texels.data_ptr()
        p.probes_per_row_color = self.color.probes_per_row
        p.probes_per_row_vis = self.visibility.probes_per_row
        p.ray_records = self.ray_records.data_ptr() if self.ray_records is not None else None
        return p

    def _wait_pinned(self, k: int) -> None:
        """Host waits until the copy (eager or graph replay) that last read
        pinned ray buffer k has completed."""
        for evs in (self._pinned_evt, self._graph_evt):
            if evs[k] is not None:
                evs[k].synchronize()

    def upload_rays(self, frame: int) -> None:
        k = frame & 1
        self._wait_pinned(k)
        self._pinned_dirs[k].numpy()[...] = frame_ray_directions(self.rays_per_probe, self.seed, frame)
        self.ray_dirs.copy_(self._pinned_dirs[k], non_blocking=True)
        evt = torch.cuda.Event()
        evt.record(torch.cuda.current_stream(self.device))
        self._pinned_evt[k] = evt

    def _issue(self, hysteresis: float) -> None:
        """Weights + shadow maps + trace + blend on the current stream."""
        sl = self._shadow_slice()
        if self.shadow_peer is not None and sl is not None:
            self._issue_peer(hysteresis, sl)
            return
        self._issue_pre(hysteresis, sl)
        if sl is not None:
            self._gather_shadow(sl)
            self._issue_post(hysteresis)

    def _issue_peer(self, hysteresis: float, sl) -> None:
        """Weights, this rank's shadow slice into every rank's maps (parity k),
        flag, wait for all slices, trace + blend: kernels only."""
        sp = self.shadow_peer
        stream = D.stream_ptr(self.device)
        k = self.frames_done & 1
        rank, world = self.shadow_split[:2]
        N.call("ps_blend_weights", self.ray_dirs.data_ptr(), self.rays_per_probe,
               self.texdir.data_ptr(), self.sharpness, self.w_color.data_ptr(),
               self.w_depth.data_ptr(), self.inv_wsum.data_ptr(), D.ptr(self.w_image), stream)
        N.call("ps_frame_advance", sp["state"].data_ptr(), 1 << 30, stream)
        b, e, _ = sl
        if e > b:
            params = self._params(hysteresis, passes=1, texels=(b, e), shadow_maps=sp["maps2"][k],
                                  shadow_dst=sp["dst"][k], ndst=world)
            N.call("ps_trace_blend", ctypes.byref(params), stream)
        seq = sp["state"][0:1]
        N.call("ps_peer_signal", sp["sig"].data_ptr(), world, 0, seq.data_ptr(), 1, stream)
        from .distributed import peer_wait

        peer_wait(sp["flags"].data_ptr(), world, 0, seq.data_ptr(), self.device, stream)
        params = self._params(hysteresis, passes=6, shadow_maps=sp["maps2"][k])
        N.call("ps_trace_blend", ctypes.byref(params), stream)

    def _issue_pre(self, hysteresis: float, sl) -> None:
        """Weights, then everything (unsharded) or this rank's shadow-map slice."""
        stream = D.stream_ptr(self.device)
        N.call("ps_blend_weights", self.ray_dirs.data_ptr(), self.rays_per_probe,
               self.texdir.data_ptr(), self.sharpness, self.w_color.data_ptr(),
               self.w_depth.data_ptr(), self.inv_wsum.data_ptr(), D.ptr(self.w_image), stream)
        if sl is None:
            params = self._params(hysteresis)
        else:
            b, e, _ = sl
            if e <= b:
                return  # empty slice: this rank only receives
            params = self._params(hysteresis, passes=1, texels=(b, e))
        N.call("ps_trace_blend", ctypes.byref(params), stream)

    def _issue_post(self, hysteresis: float) -> None:
        params = self._params(hysteresis, passes=6)
        N.call("ps_trace_blend", ctypes.byref(params), D.stream_ptr(self.device))

    def _gather_shadow(self, sl) -> None:
        """In-place all-gather of the ranks' map slices (NCCL, current stream)."""
        import torch.distributed as dist

        rank, world, group = self.shadow_split
        _, _, chunk = sl
        flat = self.shadow_maps.view(-1)
        dist.all_gather_into_tensor(flat[:chunk * world], flat[rank * chunk:(rank + 1) * chunk],
                                    group=group)

    def _update_graphed(self, frame: int, lights):
        k = self.frames_done & 1
        self._wait_pinned(k)
        s = self.dscene
        if self._pinned_lights is None:
            self._pinned_lights = [torch.zeros((s.MAX_LIGHTS, 6), dtype=torch.float32).pin_memory()
                                   for _ in range(2)]
        if lights is not None:
            arr = np.array([list(l.position) + list(l.intensity) for l in lights],
                           np.float32).reshape(-1, 6)
            if len(arr) > s.MAX_LIGHTS:
                raise ValueError(f"at most {s.MAX_LIGHTS} lights")
            s.light_count = len(arr)
            s.light_host = arr
        self._pinned_lights[k].numpy()[: s.light_count] = s.light_host
        self._pinned_dirs[k].numpy()[...] = frame_ray_directions(self.rays_per_probe, self.seed, frame)
        kb = self.frames_done % len(self._color_bufs)
        self.color, self.visibility = self._color_bufs[kb], self._vis_bufs[kb]
        sl = self._shadow_slice()
        key = (k, kb, s.light_count)
        g = self.graphs.get(key)
        if g is None and self.shadow_peer is not None and sl is not None:
            g = [torch.cuda.CUDAGraph()]  # peer shadow maps: no collective, one graph
            with torch.cuda.graph(g[0], capture_error_mode="thread_local"):
                self.ray_dirs.copy_(self._pinned_dirs[k], non_blocking=True)
                s.lights.copy_(self._pinned_lights[k], non_blocking=True)
                self._issue_peer(self.hysteresis, sl)
            self.graphs[key] = g
        if g is None and not (self._early and sl is None and self.shadow_peer is None):
            # unsharded: one graph; sharded shadow maps: graph (inputs, weights, map
            # slice) -> eager NCCL all-gather -> graph (trace, blend)
            g = [torch.cuda.CUDAGraph()] + ([torch.cuda.CUDAGraph()] if sl is not None else [])
            with torch.cuda.graph(g[0], capture_error_mode="thread_local"):
                self.ray_dirs.copy_(self._pinned_dirs[k], non_blocking=True)
                s.lights.copy_(self._pinned_lights[k], non_blocking=True)
                self._issue_pre(self.hysteresis, sl)
            if sl is not None:
                with torch.cuda.graph(g[1], capture_error_mode="thread_local"):
                    self._issue_post(self.hysteresis)
            self.graphs[key] = g
        if g is None and self._early and sl is None and self.shadow_peer is None:
            g = self._capture_early(k)
            self.graphs[key] = g
        if isinstance(g, dict):
            self._replay_early(g)
        else:
            g[0].replay()
            if len(g) > 1:
                self._gather_shadow(sl)
                g[1].replay()
        evt = torch.cuda.Event()
        evt.record(torch.cuda.current_stream(self.device))
        self._graph_evt[k] = evt
        self.frames_done += 1
        return self.color, self.visibility

    def _capture_early(self, k: int) -> dict:
        """Three graphs for pinned parity k: shadow (lights H2D + shadow maps),
        trace (ray table H2D + weights + trace), blend."""
        s, h = self.dscene, self.hysteresis
        g = {"shadow": torch.cuda.CUDAGraph(), "trace": torch.cuda.CUDAGraph(),
             "blend": torch.cuda.CUDAGraph()}
        with torch.cuda.graph(g["shadow"], capture_error_mode="thread_local"):
            s.lights.copy_(self._pinned_lights[k], non_blocking=True)
            N.call("ps_trace_blend", ctypes.byref(self._params(h, passes=1)),
                   D.stream_ptr(self.device))
        with torch.cuda.graph(g["trace"], capture_error_mode="thread_local"):
            self.ray_dirs.copy_(self._pinned_dirs[k], non_blocking=True)
            stream = D.stream_ptr(self.device)
            N.call("ps_blend_weights", self.ray_dirs.data_ptr(), self.rays_per_probe,
                   self.texdir.data_ptr(), self.sharpness, self.w_color.data_ptr(),
                   self.w_depth.data_ptr(), self.inv_wsum.data_ptr(), D.ptr(self.w_image), stream)
            N.call("ps_trace_blend", ctypes.byref(self._params(h, passes=2)), stream)
        with torch.cuda.graph(g["blend"], capture_error_mode="thread_local"):
            N.call("ps_trace_blend", ctypes.byref(self._params(h, passes=4)),
                   D.stream_ptr(self.device))
        return g

    def _replay_early(self, g: dict) -> None:
        main = torch.cuda.current_stream(self.device)
        side = self._shadow_stream
        # the maps and the lights buffer are free once the last trace is done
        if self._trace_done is not None:
            side.wait_event(self._trace_done)
        else:
            side.wait_stream(main)
        with torch.cuda.stream(side):
            g["shadow"].replay()
        shadows_done = torch.cuda.Event()
        shadows_done.record(side)
        main.wait_event(shadows_done)
        g["trace"].replay()
        self._trace_done = torch.cuda.Event()
        self._trace_done.record(main)
        g["blend"].replay()

    def update(self, frame: int | None = None, lights=None):
        """Trace + blend one frame; returns (colour atlas, visibility atlas)."""
        if frame is None:
            frame = self.frames_done
        if self.graphs is not None and self.frames_done >= 1:
            return self._update_graphed(frame, lights)
        if lights is not None:
            self.dscene.set_lights(lights)
        self.upload_rays(frame)
        h = 0.0 if self.frames_done == 0 else self.hysteresis
        k = self.frames_done % len(self._color_bufs)
        self.color, self.visibility = self._color_bufs[k], self._vis_bufs[k]
        self._issue(h)
        self.frames_done += 1
        return self.color, self.visibility

    def pass_times_ms(self, reps: int = 3) -> dict:
        """Device time of the shadow-map pass (unsharded maps only), the
        probe-ray pass and the blend pass alone (CUDA events around
        ps_trace_blend with passes = 1 / 2 / 4 on the current frame's inputs).
        Re-running the blend advances the float state, so call this only
        after the frames being measured."""
        stream = D.stream_ptr(self.device)
        out = {}
        shadow = self.shadow_peer["maps2"][(self.frames_done - 1) & 1] if self.shadow_peer else None
        runs = (("shadow_maps", 1),) if self.shadows == "map" and not self.shadow_peer else ()
        for name, passes in runs + (("trace", 2), ("blend", 4)):
            params = self._params(self.hysteresis, passes=passes, shadow_maps=shadow)
            N.call("ps_trace_blend", ctypes.byref(params), stream)  # warm
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                N.call("ps_trace_blend", ctypes.byref(params), stream)
            b.record()
            b.synchronize()
            out[name] = a.elapsed_time(b) / reps
        return out

    @property
    def rays_per_frame(self) -> int:
        return (self.probe_end - self.probe_begin) * self.rays_per_probe


def update_probes(volume: ProbeVolume, scene, state: ProbeUpdater | None = None, frame: int = 0,
                  rays_per_probe: int = 256, hysteresis: float = 0.97, **kwargs):
    """Functional entry point: returns (colour atlas,
    visibility atlas, state); pass the returned state back next frame."""
    if state is None:
        state = ProbeUpdater(volume, scene, rays_per_probe=rays_per_probe, hysteresis=hysteresis,
                             **kwargs)
    color, vis = state.update(frame)
    return color, vis, state
