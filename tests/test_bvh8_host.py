"""Host BVH8 builder (csrc/ps_bvh.cpp emit_bvh8), CPU only: the quantised
layout decoded in numpy must be conservative -- every inner slot's decoded
box contains the child node's decoded boxes, every leaf slot's decoded box
contains its triangles -- and every triangle is referenced exactly once."""

import ctypes

import numpy as np
import pytest


def _build(verts, leaf_size=2):
    from paper_2103_05875_b200 import _native as N

    lib = N.lib()
    v = np.ascontiguousarray(verts, np.float64)
    sizes = N.BvhSizes()
    vp = v.ctypes.data_as(ctypes.c_void_p)
    N.check(lib.ps_bvh_build_wide(vp, len(v), leaf_size, 8, ctypes.byref(sizes), None, None), "size")
    nodes = np.zeros(sizes.node_count * 24, np.float32)
    tris = np.zeros(sizes.tri_slots * 12, np.float32)
    N.check(lib.ps_bvh_build_wide(vp, len(v), leaf_size, 8, ctypes.byref(sizes),
                                  nodes.ctypes.data_as(ctypes.c_void_p),
                                  tris.ctypes.data_as(ctypes.c_void_p)), "build")
    return nodes.reshape(-1, 24), tris.reshape(-1, 12), sizes


def _decode(node):
    w = node.view(np.uint32)
    b = node.view(np.uint8)
    p = node[:3].astype(np.float64)
    e = b[12:15].astype(np.int64) - 127
    scale = np.ldexp(1.0, e)
    imask = int(b[15])
    child_base, tri_base = int(w[4]), int(w[5])
    meta = b[24:32]
    qlo = b[32:56].reshape(3, 8).astype(np.float64)
    qhi = b[56:80].reshape(3, 8).astype(np.float64)
    lo = p[:, None] + scale[:, None] * qlo
    hi = p[:, None] + scale[:, None] * qhi
    return lo, hi, imask, child_base, tri_base, meta


@pytest.mark.parametrize("scene_name", ["cornell", "random", "hall"])
def test_bvh8_layout_is_conservative(scene_name):
    from paper_2103_05875_b200 import scene as S

    if scene_name == "cornell":
        verts = S.cornell_box().vertices
    elif scene_name == "hall":
        verts = S.interior_hall().vertices[:20000]
    else:
        rng = np.random.default_rng(0)
        c = rng.uniform(-50, 50, size=(3000, 1, 3))
        verts = c + rng.normal(scale=0.7, size=(3000, 3, 3))
    nodes, tris, sizes = _build(verts)
    seen = np.zeros(len(verts), np.int64)
    tri_v = verts.reshape(-1, 3, 3)
    rec_prim = tris[:, 3].view(np.int32)
    # depth-first over the nodes, carrying every ancestor slot box: each
    # triangle must lie inside all decoded boxes on its path
    stack = [(0, [])]
    visited = 0
    while stack:
        i, path = stack.pop()
        visited += 1
        lo, hi, imask, child_base, tri_base, meta = _decode(nodes[i])
        rank = 0
        for sl in range(8):
            empty = np.all(lo[:, sl] > hi[:, sl])
            box = (lo[:, sl], hi[:, sl])
            if imask >> sl & 1:
                stack.append((child_base + rank, path + [box]))
                rank += 1
            elif not empty:
                m = int(meta[sl])
                first, cnt = tri_base + (m & 31), m >> 5
                assert 1 <= cnt <= 2
                for k in range(cnt):
                    t = int(rec_prim[first + k])
                    seen[t] += 1
                    v = tri_v[t]
                    for blo, bhi in path + [box]:
                        assert np.all(v.min(0) >= blo) and np.all(v.max(0) <= bhi)
                    # the record holds v0 and the float edges
                    np.testing.assert_allclose(tris[first + k, 0:3], v[0], rtol=1e-6, atol=1e-6)
            else:
                assert np.all(lo[:, sl] > hi[:, sl])
    assert visited == len(nodes)
    assert np.all(seen == 1)
    assert sizes.tri_slots == len(verts)


def _build_w(verts, width, leaf_size=2):
    from paper_2103_05875_b200 import _native as N

    lib = N.lib()
    v = np.ascontiguousarray(verts, np.float64)
    sizes = N.BvhSizes()
    vp = v.ctypes.data_as(ctypes.c_void_p)
    N.check(lib.ps_bvh_build_wide(vp, len(v), leaf_size, width, ctypes.byref(sizes), None, None), "size")
    words = {3: 16, 8: 24}[width]
    nodes = np.zeros(sizes.node_count * words, np.float32)
    tris = np.zeros(sizes.tri_slots * 12, np.float32)
    N.check(lib.ps_bvh_build_wide(vp, len(v), leaf_size, width, ctypes.byref(sizes),
                                  nodes.ctypes.data_as(ctypes.c_void_p),
                                  tris.ctypes.data_as(ctypes.c_void_p)), "build")
    return nodes.reshape(-1, words), tris.reshape(-1, 12), sizes


@pytest.mark.parametrize("scene_name", ["cornell", "random", "hall"])
def test_bvh4_relative_half_layout_is_conservative(scene_name):
    """Width 3 (origin-relative fp16 BVH4, compact child refs): every
    triangle lies inside every decoded box on its path; refs are consistent."""
    from paper_2103_05875_b200 import scene as S

    if scene_name == "cornell":
        verts = S.cornell_box().vertices
    elif scene_name == "hall":
        verts = S.interior_hall().vertices[:20000]
    else:
        rng = np.random.default_rng(1)
        c = rng.uniform(-50, 50, size=(3000, 1, 3))
        verts = c + rng.normal(scale=0.7, size=(3000, 3, 3))
    nodes, tris, sizes = _build_w(verts, 3)
    tri_v = verts.reshape(-1, 3, 3)
    rec_prim = tris[:, 3].view(np.int32)
    seen = np.zeros(len(verts), np.int64)
    stack = [(0, [])]
    visited = 0
    while stack:
        i, path = stack.pop()
        visited += 1
        nd = nodes[i]
        h = nd.view(np.uint16)
        w = nd.view(np.uint32)
        org = h[24:27].view(np.float16).astype(np.float64)
        meta = int(h[27])
        child_base, tri_base = int(w[14]), int(w[15])
        planes = h[:24].view(np.float16).astype(np.float64).reshape(3, 2, 4)
        lo = org[:, None] + planes[:, 0]
        hi = org[:, None] + planes[:, 1]
        rank = 0
        for k in range(4):
            nib = meta >> (4 * k) & 15
            box = (lo[:, k], hi[:, k])
            if nib == 15:
                stack.append((child_base + rank, path + [box]))
                rank += 1
            elif nib:
                off, cnt = (nib - 1) >> 1, ((nib - 1) & 1) + 1
                for j in range(cnt):
                    t = int(rec_prim[tri_base + off + j])
                    seen[t] += 1
                    v = tri_v[t]
                    for blo, bhi in path + [box]:
                        assert np.all(v.min(0) >= blo) and np.all(v.max(0) <= bhi)
            else:
                assert np.all(np.isinf(lo[:, k])) and np.all(lo[:, k] > hi[:, k])
    assert visited == len(nodes)
    assert np.all(seen == 1)
