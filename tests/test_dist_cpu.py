"""Multi-process host logic of the slab-sharded frame on CPU (gloo,
world_size 2): slab ranges, the change-bitmap exchange, the payload gather
to the encoder rank, and an end-to-end emulation of the sharded stages 3-4
against the single-process oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import stream_ops as so


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2103_05875_b200.distributed import exchange_bitmap, gather_payloads, slab_range
    from paper_2103_05875_b200.volume import ProbeVolume

    vol = ProbeVolume((8, 4, 6))
    n = vol.probe_count
    b, e = slab_range(vol, rank, world)
    rng = np.random.default_rng(100 + rank)
    changed = np.zeros(n, bool)
    changed[b:e] = rng.random(e - b) < 0.4
    words = np.zeros((n + 31) // 32, np.uint32)
    for p in np.nonzero(changed)[0]:
        words[p >> 5] |= np.uint32(1 << (p & 31))
    bits = torch.from_numpy(words.view(np.int32).copy())
    exchange_bitmap(bits)
    slab_max = max(slab_range(vol, r, world)[1] - slab_range(vol, r, world)[0] for r in range(world))
    payload = torch.full((slab_max * 4,), rank + 1, dtype=torch.int32)
    payloads = torch.zeros((world, slab_max * 4), dtype=torch.int32) if rank == 0 else None
    if rank == 0:
        payloads[0] = payload
    gather_payloads(payload, payloads, rank, world, 0)
    results[rank] = (bits.numpy().copy(), changed, None if payloads is None else payloads.numpy().copy())
    dist.destroy_process_group()


def test_slab_ranges_cover_volume():
    from paper_2103_05875_b200.distributed import slab_range
    from paper_2103_05875_b200.volume import ProbeVolume

    for dims in ((64, 32, 64), (8, 8, 8), (5, 3, 7)):
        vol = ProbeVolume(dims)
        for world in (1, 2, 3, 4, 8):
            rs = [slab_range(vol, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == vol.probe_count
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert all((e - b) % (dims[0] * dims[1]) == 0 for b, e in rs)


def test_exchange_gloo_world2():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
    union = results[0][1] | results[1][1]
    for r in range(world):
        bits = results[r][0].view(np.uint32)
        got = np.array([(bits[p >> 5] >> (p & 31)) & 1 for p in range(len(union))], bool)
        assert np.array_equal(got, union)
    pay = results[0][2]
    assert (pay[0] == 1).all() and (pay[1] == 2).all()


def test_sharded_stages_emulation_matches_single():
    """numpy emulation of the per-rank detect / replicated select+assign /
    export / import flow gives the single-process oracle's update atlas."""
    from paper_2103_05875_b200.distributed import slab_range
    from paper_2103_05875_b200.volume import ProbeVolume

    vol = ProbeVolume((6, 4, 5))
    n = vol.probe_count
    ppr = so.default_probes_per_row(n)
    rng = np.random.default_rng(7)
    kind = "visibility"
    shp = so.atlas_shape(kind, n, ppr)
    rendered = rng.integers(0, 2**16, size=shp, dtype=np.uint16)
    last = rendered.copy()
    side = 18
    for p in rng.choice(n, size=n // 3, replace=False):
        br, bc = divmod(int(p), ppr)
        last[br * side + 3, bc * side + 4, 0] ^= 1
    act = np.ones(n, bool)
    want_ids = so.detect_changed(rendered, last, kind, n, ppr, act)
    cache = so.SlotCache(n, 16)
    want_tex, want_entries = so.build_update_atlas(want_ids, cache, rendered, kind, ppr)
    world = 3
    ranges = [slab_range(vol, r, world) for r in range(world)]
    # per-rank detect on own slab, OR of bitmaps
    union = np.zeros(n, bool)
    for b, e in ranges:
        ids = so.detect_changed(rendered, last, kind, n, ppr, act)
        union[ids[(ids >= b) & (ids < e)]] = True
    sel = np.nonzero(union)[0]
    cache2 = so.SlotCache(n, 16)
    entries = cache2.assign(sel)
    assert entries == want_entries
    # per-rank export by local index, encoder import
    slab_max = max(e - b for b, e in ranges)
    payloads = np.zeros((world, slab_max, 16, 16, 2), np.uint16)
    for r, (b, e) in enumerate(ranges):
        for slot, p in entries:
            if b <= p < e:
                br, bc = divmod(p, ppr)
                payloads[r, p - b] = rendered[br * side + 1:br * side + 17, bc * side + 1:bc * side + 17]
    tex = np.zeros(cache2.texel_shape(kind), np.uint16)
    for slot, p in entries:
        r = next(i for i, (b, e) in enumerate(ranges) if b <= p < e)
        sy, sx = cache2.slot_yx(slot)
        tex[sy:sy + 16, sx:sx + 16] = payloads[r, p - ranges[r][0]]
    assert np.array_equal(tex, want_tex)


def test_cost_balanced_ranges():
    """ranges_from_cost: whole planes, contiguous, cover the volume, every rank
    at least one plane, and near-equal cost (calibration input of
    balanced_ranges, which every rank evaluates identically)."""
    from paper_2103_05875_b200.distributed import ranges_from_cost

    plane = 64 * 32
    for world in (1, 2, 3, 4, 8):
        r = ranges_from_cost(64, plane, world, [1.0] * 64)
        assert r[0][0] == 0 and r[-1][1] == 64 * plane
        assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
        sizes = [(e - b) // plane for b, e in r]
        assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1
    cost = [1.0] * 32 + [3.0] * 32  # the far half is 3x more expensive
    r = ranges_from_cost(64, plane, 4, cost)
    sums = [sum(cost[b // plane:e // plane]) for b, e in r]
    assert max(sums) - min(sums) <= 3.0 + 1e-9
    r = ranges_from_cost(8, plane, 8, [100.0] + [1.0] * 7)
    assert [(e - b) // plane for b, e in r] == [1] * 8
    r = ranges_from_cost(8, plane, 4, [1.0] * 7 + [100.0])
    assert r[-1] == (7 * plane, 8 * plane) and min(e - b for b, e in r) >= plane


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("share", [1.0, 0.88, 0.5])
def test_slab_ranges_partition_the_volume(world, share):
    """Slabs tile [0, n) in rank order, at whole rows of nx probes (whole
    k-planes at share 1), with the encoder's reduced share when asked."""
    from paper_2103_05875_b200.distributed import slab_range

    class V:
        dims = (64, 32, 64)

    n = 64 * 32 * 64
    r = [slab_range(V, k, world, share) for k in range(world)]
    assert r[0][0] == 0 and r[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
    assert all(b % 64 == 0 and e % 64 == 0 and e > b for b, e in r)
    if share == 1.0:
        assert all(b % (64 * 32) == 0 for b, _ in r)
    else:
        sizes = [e - b for b, e in r]
        assert sizes[0] < min(sizes[1:])
        assert abs(sizes[0] / (sum(sizes[1:]) / (world - 1)) - share) < 0.05
