"""Synthetic scenes for the probe ray tracer and their device upload.

The reference ships no scenes (its harness, which would generate them, is
absent: SURVEY F2/F3), so BASELINE.json's configurations are built here,
deterministically from a seed:

* ``cornell_box()``      -- config 1: unit room of axis-aligned wall boxes plus
                            two blocks and a ceiling point light (the boxes are
                            triangulated; the reference raycast treats boxes and
                            triangles alike, selection.py:66-149).
* ``interior_hall()``    -- config 2/4: a ~260k-triangle Sponza-scale hall with
                            tessellated columns, arches, a gallery, curtains,
                            statues and a skylight.

Triangles are float64 ``(T, 3, 3)``; each carries an albedo and an emission.
``DeviceScene`` holds the BVH (built on the host by ``ps_bvh_build``) and the
per-triangle material / normal table on the GPU.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N


@dataclass
class PointLight:
    position: tuple
    intensity: tuple  # rgb, radiant intensity (falls off with 1/d^2)


@dataclass
class Scene:
    vertices: np.ndarray            # (T, 3, 3) float64
    albedo: np.ndarray              # (T, 3)
    emission: np.ndarray            # (T, 3)
    lights: list = field(default_factory=list)
    sky: tuple = (0.0, 0.0, 0.0)
    bounds: tuple = ((0.0, 0.0, 0.0), (1.0, 1.0, 1.0))

    @property
    def triangle_count(self) -> int:
        return len(self.vertices)

    def face_normals(self) -> np.ndarray:
        v = self.vertices
        n = np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0])
        return n / np.maximum(np.linalg.norm(n, axis=1, keepdims=True), 1e-30)

    def with_lights(self, lights) -> "Scene":
        return Scene(self.vertices, self.albedo, self.emission, list(lights), self.sky, self.bounds)

    def light_array(self) -> np.ndarray:
        if not self.lights:
            return np.zeros((0, 6), np.float32)
        return np.array([list(l.position) + list(l.intensity) for l in self.lights], np.float32)

    def material_table(self) -> np.ndarray:
        """(T, 12) float32: albedo rgb 0, emission rgb 0, unit normal xyz 0."""
        m = np.zeros((self.triangle_count, 12), np.float32)
        m[:, 0:3] = self.albedo
        m[:, 4:7] = self.emission
        m[:, 8:11] = self.face_normals()
        return m

    def device(self, device=None, leaf_size: int = 2, width: int | None = None) -> "DeviceScene":
        """BVH layouts: 2 = BVH2, 4 = BVH4 (fp32 boxes), 5 = BVH4 with fp16
        boxes (64-byte nodes), 3 = BVH4 with fp16 boxes relative to an fp16
        node origin and compact child references (64-byte nodes), 8 = BVH8
        with 8-bit quantised boxes (96-byte nodes); default from
        PS_BVH_WIDTH or DEFAULT_BVH_WIDTH."""
        import os

        if width is None:
            width = int(os.environ.get("PS_BVH_WIDTH", DEFAULT_BVH_WIDTH))
            if (width == 5 and len(self.vertices)
                    and np.abs(self.vertices - bvh_frame_origin(self.vertices)).max() > FP16_SAFE):
                width = 4  # fp16 boxes would lose too much precision
        return DeviceScene(self, device, leaf_size, width)


# fp16-box BVH4: two 256-bit loads per node instead of four; C4 trace + blend
# 5.75 -> 5.43 ms (the trace is bound by L1 wavefronts of node fetches).  Scenes
# with coordinates beyond FP16_SAFE use fp32 boxes (width 4).
DEFAULT_BVH_WIDTH = 5
FP16_SAFE = 16384.0
# PS_BVH_CENTER=0 builds the BVH in world coordinates (tuning / A-B only)
BVH_CENTER = __import__("os").environ.get("PS_BVH_CENTER", "1") != "0"


def bvh_frame_origin(vertices) -> np.ndarray:
    """Origin of the frame the BVH is built in: the centre of the triangles'
    bounds on a 1/16 grid, so |coordinates| halve for a scene in the positive
    octant and the fp16 boxes round outward at half the magnitude (C4 hall:
    trace 4.106 -> 3.996 ms, 1.411 -> 1.381 leaves and 2.806 -> 2.747 triangle
    tests per ray).  Rays are moved into this frame for the traversal only
    (ps_traverse.cuh to_bvh_frame)."""
    v = np.asarray(vertices, np.float64).reshape(-1, 3)
    if not BVH_CENTER or not len(v):
        return np.zeros(3)
    c = 0.5 * (v.min(axis=0) + v.max(axis=0))
    return np.round(c * 16.0) / 16.0


class DeviceScene:
    """BVH + triangles + materials + lights resident in HBM (replicated per GPU)."""

    def __init__(self, scene: Scene, device=None, leaf_size: int = 2, width: int = DEFAULT_BVH_WIDTH):
        import torch

        from . import _device as D

        self.scene = scene
        self.width = int(width)
        self.device = torch.device(device) if device is not None else D.device_of()
        # the BVH (boxes + triangle records) lives in a frame centred on the
        # scene; the node buffer starts with a 64-byte header holding that
        # origin, and kernels get a pointer to node 0 (ps_traverse.cuh)
        self.frame_origin = bvh_frame_origin(scene.vertices)
        verts = np.ascontiguousarray(np.asarray(scene.vertices, np.float64) -
                                     self.frame_origin.reshape(1, 1, 3), dtype=np.float64)
        sizes = N.BvhSizes()
        vp = verts.ctypes.data_as(ctypes.c_void_p)
        N.check(N.lib().ps_bvh_build_wide(vp, len(verts), leaf_size, self.width,
                                          ctypes.byref(sizes), None, None), "ps_bvh_build_wide")
        words = {2: 16, 3: 16, 4: 32, 5: 16, 8: 24}[self.width]
        nodes = np.zeros(sizes.node_count * words, np.float32)
        tris = np.zeros(sizes.tri_slots * 12, np.float32)
        N.check(N.lib().ps_bvh_build_wide(vp, len(verts), leaf_size, self.width,
                                          ctypes.byref(sizes),
                                          nodes.ctypes.data_as(ctypes.c_void_p),
                                          tris.ctypes.data_as(ctypes.c_void_p)),
                "ps_bvh_build_wide")
        # traversal stack: at most (children - 1) pushes per level (64 entries);
        # BVH8 pushes at most one node group per level (32 entries)
        if self.width == 8:
            if sizes.max_depth > 32:
                raise ValueError(f"BVH8 depth {sizes.max_depth} exceeds the traversal stack (32)")
        elif ((2 if self.width == 2 else 4) - 1) * sizes.max_depth + 1 > 64:
            raise ValueError(f"BVH depth {sizes.max_depth} exceeds the traversal stack (64)")
        self.sizes = (int(sizes.node_count), int(sizes.tri_slots), int(sizes.max_depth))
        self.host_nodes, self.host_tris = nodes, tris
        buf = np.zeros(16 + nodes.size, np.float32)
        buf[:3] = self.frame_origin
        buf[16:] = nodes
        self.node_buffer = torch.from_numpy(buf).to(self.device)
        self.nodes = self.node_buffer[16:]  # node 0; the header sits 64 bytes before it
        self.tris = torch.from_numpy(tris).to(self.device)
        self.materials = torch.from_numpy(scene.material_table()).to(self.device)
        self.set_lights(scene.lights)

    MAX_LIGHTS = 30

    def set_lights(self, lights) -> None:
        """Per-frame light update: pinned staging + async copy into a fixed
        device table (no allocation, no host sync)."""
        import torch

        arr = np.array([list(l.position) + list(l.intensity) for l in lights],
                       np.float32).reshape(-1, 6)
        if len(arr) > self.MAX_LIGHTS:
            raise ValueError(f"at most {self.MAX_LIGHTS} lights")
        if not hasattr(self, "lights"):
            self.lights = torch.zeros((self.MAX_LIGHTS, 6), dtype=torch.float32, device=self.device)
            self._light_stage = [torch.zeros((self.MAX_LIGHTS, 6), dtype=torch.float32).pin_memory()
                                 for _ in range(2)]
            self._light_evt = [None, None]
            self._light_k = 0
        k = self._light_k = 1 - self._light_k
        if self._light_evt[k] is not None:
            self._light_evt[k].synchronize()
        self._light_stage[k].numpy()[: len(arr)] = arr
        self.light_host = arr
        self.lights.copy_(self._light_stage[k], non_blocking=True)
        evt = torch.cuda.Event()
        evt.record(torch.cuda.current_stream(self.device))
        self._light_evt[k] = evt
        self.light_count = len(arr)

    @property
    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (self.nodes, self.tris, self.materials))


# --- geometry builders ------------------------------------------------------------------


def box_triangles(lo, hi) -> np.ndarray:
    """12 triangles of an axis-aligned box."""
    x0, y0, z0 = lo
    x1, y1, z1 = hi
    c = np.array([[x0, y0, z0], [x1, y0, z0], [x1, y1, z0], [x0, y1, z0],
                  [x0, y0, z1], [x1, y0, z1], [x1, y1, z1], [x0, y1, z1]], np.float64)
    faces = [(0, 1, 2, 3), (5, 4, 7, 6), (4, 0, 3, 7), (1, 5, 6, 2), (3, 2, 6, 7), (4, 5, 1, 0)]
    out = []
    for a, b, cc, d in faces:
        out.append([c[a], c[b], c[cc]])
        out.append([c[a], c[cc], c[d]])
    return np.array(out)


def grid_quad(origin, u, v, nu, nv) -> np.ndarray:
    """Tessellated parallelogram origin + s*u + t*v, s,t in [0,1]: 2*nu*nv triangles."""
    o, u, v = (np.asarray(x, np.float64) for x in (origin, u, v))
    s = np.linspace(0.0, 1.0, nu + 1)
    t = np.linspace(0.0, 1.0, nv + 1)
    P = o + s[:, None, None] * u + t[None, :, None] * v  # (nu+1, nv+1, 3)
    a, b = P[:-1, :-1], P[1:, :-1]
    c, d = P[1:, 1:], P[:-1, 1:]
    t1 = np.stack([a, b, c], axis=2).reshape(-1, 3, 3)
    t2 = np.stack([a, c, d], axis=2).reshape(-1, 3, 3)
    return np.concatenate([t1, t2])


def cylinder(center, radius, y0, y1, segments, rings) -> np.ndarray:
    cx, cz = center
    th = np.linspace(0.0, 2 * np.pi, segments + 1)
    ys = np.linspace(y0, y1, rings + 1)
    x = cx + radius * np.cos(th)
    z = cz + radius * np.sin(th)
    P = np.stack([np.broadcast_to(x[:, None], (segments + 1, rings + 1)),
                  np.broadcast_to(ys[None, :], (segments + 1, rings + 1)),
                  np.broadcast_to(z[:, None], (segments + 1, rings + 1))], axis=-1)
    a, b = P[:-1, :-1], P[1:, :-1]
    c, d = P[1:, 1:], P[:-1, 1:]
    return np.concatenate([np.stack([a, b, c], 2).reshape(-1, 3, 3),
                           np.stack([a, c, d], 2).reshape(-1, 3, 3)])


def arch(p0, p1, y_base, rise, width, segments, around) -> np.ndarray:
    """Half-circle tube from p0 to p1 (x,z) springing at y_base."""
    p0, p1 = np.asarray(p0, np.float64), np.asarray(p1, np.float64)
    mid = 0.5 * (p0 + p1)
    span = np.linalg.norm(p1 - p0) / 2
    axis = (p1 - p0) / (2 * span)
    ang = np.linspace(np.pi, 0.0, segments + 1)
    centers = np.stack([mid[0] + axis[0] * span * np.cos(ang), y_base + rise * np.sin(ang),
                        mid[1] + axis[1] * span * np.cos(ang)], axis=-1)
    # tube cross-section in the plane spanned by the radial dir and the horizontal normal
    side = np.array([-axis[1], 0.0, axis[0]])
    radial = np.stack([axis[0] * np.cos(ang) * span / max(span, 1e-9),
                       rise * np.sin(ang) / max(rise, 1e-9), axis[1] * np.cos(ang)], axis=-1)
    radial /= np.linalg.norm(radial, axis=1, keepdims=True)
    phi = np.linspace(0.0, 2 * np.pi, around + 1)
    r = width / 2
    P = (centers[:, None, :] + r * np.cos(phi)[None, :, None] * radial[:, None, :]
         + r * np.sin(phi)[None, :, None] * side[None, None, :])
    a, b = P[:-1, :-1], P[1:, :-1]
    c, d = P[1:, 1:], P[:-1, 1:]
    return np.concatenate([np.stack([a, b, c], 2).reshape(-1, 3, 3),
                           np.stack([a, c, d], 2).reshape(-1, 3, 3)])


def icosphere(center, radius, subdiv) -> np.ndarray:
    t = (1.0 + math.sqrt(5.0)) / 2.0
    verts = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t), (0, -1, -t),
             (0, 1, -t), (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4),
             (11, 10, 2), (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8),
             (3, 8, 9), (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    tris = np.array([[verts[a], verts[b], verts[c]] for a, b, c in faces], np.float64)
    tris /= np.linalg.norm(tris, axis=2, keepdims=True)
    for _ in range(subdiv):
        a, b, c = tris[:, 0], tris[:, 1], tris[:, 2]
        ab, bc, ca = a + b, b + c, c + a
        ab /= np.linalg.norm(ab, axis=1, keepdims=True)
        bc /= np.linalg.norm(bc, axis=1, keepdims=True)
        ca /= np.linalg.norm(ca, axis=1, keepdims=True)
        tris = np.concatenate([np.stack(x, 1) for x in ((a, ab, ca), (b, bc, ab), (c, ca, bc),
                                                          (ab, bc, ca))])
    return np.asarray(center, np.float64) + radius * tris


class _Builder:
    def __init__(self):
        self.parts, self.alb, self.emi = [], [], []

    def add(self, tris, albedo, emission=(0.0, 0.0, 0.0)):
        tris = np.asarray(tris, np.float64).reshape(-1, 3, 3)
        self.parts.append(tris)
        self.alb.append(np.broadcast_to(np.asarray(albedo, np.float64), (len(tris), 3)))
        self.emi.append(np.broadcast_to(np.asarray(emission, np.float64), (len(tris), 3)))

    def scene(self, lights, sky, bounds) -> Scene:
        return Scene(np.concatenate(self.parts), np.concatenate(self.alb).astype(np.float32),
                     np.concatenate(self.emi).astype(np.float32), lights, sky, bounds)


def cornell_box() -> Scene:
    """Config 1: unit room from AABB walls, a tall and a short block, a point light."""
    b = _Builder()
    th = 0.02
    white, red, green = (0.73, 0.73, 0.73), (0.65, 0.05, 0.05), (0.12, 0.45, 0.15)
    b.add(box_triangles((-th, -th, -th), (1 + th, 0.0, 1 + th)), white)        # floor
    b.add(box_triangles((-th, 1.0, -th), (1 + th, 1 + th, 1 + th)), white)     # ceiling
    b.add(box_triangles((-th, 0.0, 1.0), (1 + th, 1.0, 1 + th)), white)        # back
    b.add(box_triangles((-th, 0.0, -th), (0.0, 1.0, 1 + th)), red)             # left
    b.add(box_triangles((1.0, 0.0, -th), (1 + th, 1.0, 1 + th)), green)        # right
    b.add(box_triangles((0.53, 0.0, 0.46), (0.83, 0.6, 0.76)), white)          # tall block
    b.add(box_triangles((0.17, 0.0, 0.13), (0.47, 0.3, 0.43)), white)          # short block
    b.add(box_triangles((0.40, 0.985, 0.40), (0.60, 1.0, 0.60)), (0.8, 0.8, 0.8), (4.0, 3.6, 3.0))
    lights = [PointLight((0.5, 0.95, 0.5), (0.8, 0.75, 0.65))]
    return b.scene(lights, (0.0, 0.0, 0.0), ((0.0, 0.0, 0.0), (1.0, 1.0, 1.0)))


HALL = ((0.0, 0.0, 0.0), (32.0, 16.0, 32.0))


def interior_hall(seed: int = 0, detail: float = 1.0) -> Scene:
    """Configs 2/4: a ~260k-triangle Sponza-scale interior (seeded).

    ``detail`` scales the tessellation (1.0 -> ~260k triangles)."""
    rng = np.random.default_rng(seed)
    b = _Builder()
    (x0, y0, z0), (x1, y1, z1) = HALL
    W, H, L = x1 - x0, y1 - y0, z1 - z0
    g = max(4, int(48 * detail))
    stone, floor_c, ceil_c = (0.62, 0.58, 0.50), (0.45, 0.42, 0.38), (0.70, 0.68, 0.62)
    # floor, walls; ceiling with a central skylight opening
    b.add(grid_quad((x0, y0, z0), (0, 0, L), (W, 0, 0), g, g), floor_c)
    b.add(grid_quad((x0, y0, z0), (W, 0, 0), (0, H, 0), g, g // 2), stone)
    b.add(grid_quad((x0, y0, z1), (0, H, 0), (W, 0, 0), g // 2, g), stone)
    b.add(grid_quad((x0, y0, z0), (0, H, 0), (0, 0, L), g // 2, g), stone)
    b.add(grid_quad((x1, y0, z0), (0, 0, L), (0, H, 0), g, g // 2), stone)
    sk0, sk1 = 12.0, 20.0
    for (a0, a1, c0, c1) in ((x0, sk0, z0, z1), (sk1, x1, z0, z1), (sk0, sk1, z0, sk0), (sk0, sk1, sk1, z1)):
        b.add(grid_quad((a0, y1, c0), (a1 - a0, 0, 0), (0, 0, c1 - c0), g // 4, g // 4), ceil_c)
    # gallery floors at y = 8 along both long sides
    for gx0, gx1 in ((x0, 7.0), (25.0, x1)):
        b.add(box_triangles((gx0, 7.8, z0), (gx1, 8.2, z1)), stone)
    seg = max(8, int(40 * detail))
    rings = max(4, int(24 * detail))
    col_z = np.arange(2.0, L - 1.0, 2.5)
    for cx in (7.0, 25.0):
        for cz in col_z:
            b.add(cylinder((cx, cz), 0.45, y0, 7.8, seg, rings), (0.80, 0.78, 0.72))
            b.add(cylinder((cx, cz), 0.30, 8.2, 14.0, seg, rings), (0.80, 0.78, 0.72))
            b.add(box_triangles((cx - 0.6, 7.4, cz - 0.6), (cx + 0.6, 7.8, cz + 0.6)), stone)
        for za, zb in zip(col_z[:-1], col_z[1:]):
            b.add(arch((cx, za), (cx, zb), 5.8, 2.0, 0.4, max(8, int(40 * detail)),
                       max(4, int(12 * detail))), (0.75, 0.70, 0.62))
            b.add(arch((cx, za), (cx, zb), 12.5, 1.4, 0.3, max(8, int(32 * detail)),
                       max(4, int(10 * detail))), (0.75, 0.70, 0.62))
    # curtains hanging from the galleries (wavy tessellated sheets)
    palette = [(0.60, 0.08, 0.08), (0.10, 0.35, 0.12), (0.10, 0.14, 0.50)]
    cn = max(4, int(44 * detail))
    for i, cz in enumerate(col_z[:-1]):
        for cx, sgn in ((6.4, -1.0), (25.6, 1.0)):
            s = np.linspace(0, 1, cn + 1)
            t = np.linspace(0, 1, cn + 1)
            S, T = np.meshgrid(s, t, indexing="ij")
            X = cx + sgn * 0.15 * np.sin(S * np.pi * 6.0)
            Y = 7.6 - 5.0 * T
            Z = cz + 0.4 + 1.7 * S
            P = np.stack([X, Y, Z], -1)
            a, bb, c, d = P[:-1, :-1], P[1:, :-1], P[1:, 1:], P[:-1, 1:]
            b.add(np.concatenate([np.stack([a, bb, c], 2).reshape(-1, 3, 3),
                                  np.stack([a, c, d], 2).reshape(-1, 3, 3)]), palette[i % 3])
    # statues on the floor of the nave
    sub = 4 if detail >= 1.0 else max(1, int(4 * detail))
    for k in range(8):
        cx = 11.0 + 10.0 * rng.random()
        cz = 3.0 + 26.0 * rng.random()
        r = 0.6 + 0.5 * rng.random()
        b.add(icosphere((cx, r + 0.8, cz), r, sub), tuple(0.3 + 0.6 * rng.random(3)))
        b.add(box_triangles((cx - 0.5, 0.0, cz - 0.5), (cx + 0.5, 0.8, cz + 0.5)), stone)
    # crates
    for _ in range(int(160 * max(detail, 0.1))):
        cx, cz = x0 + 1 + (W - 2) * rng.random(), z0 + 1 + (L - 2) * rng.random()
        s = 0.2 + 0.5 * rng.random()
        b.add(box_triangles((cx - s, 0.0, cz - s), (cx + s, 2 * s, cz + s)), (0.55, 0.40, 0.25))
    lights = [PointLight((16.0, 14.0, 16.0), (120.0, 110.0, 95.0)),
              PointLight((4.0, 6.0, 8.0), (25.0, 14.0, 6.0)),
              PointLight((28.0, 6.0, 24.0), (6.0, 14.0, 25.0))]
    return b.scene(lights, (0.35, 0.45, 0.60), HALL)


def moving_light(scene: Scene, frame: int, period: int = 120) -> Scene:
    """Config 3: the first light orbits the hall centre over `period` frames."""
    (x0, y0, z0), (x1, y1, z1) = scene.bounds
    ang = 2.0 * math.pi * (frame % period) / period
    cx, cz = 0.5 * (x0 + x1), 0.5 * (z0 + z1)
    rad = 0.3 * min(x1 - x0, z1 - z0)
    first = scene.lights[0]
    moved = PointLight((cx + rad * math.cos(ang), first.position[1], cz + rad * math.sin(ang)),
                       first.intensity)
    return scene.with_lights([moved] + list(scene.lights[1:]))


def volume_for(scene: Scene, dims, margin: float = 0.5):
    """Probe volume filling the scene bounds: cell-centred grid."""
    from .volume import ProbeVolume

    (x0, y0, z0), (x1, y1, z1) = scene.bounds
    ext = np.array([x1 - x0, y1 - y0, z1 - z0])
    d = np.asarray(dims, np.float64)
    spacing = ext / d
    origin = np.array([x0, y0, z0]) + margin * spacing
    return ProbeVolume(tuple(int(x) for x in dims), tuple(origin.tolist()), tuple(spacing.tolist()))
