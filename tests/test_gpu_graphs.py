"""CUDA-graph replay of the frame pipeline: a server that replays captured
graphs (trace + blend, one stage chain per kind) must produce bit-identical
outputs and state to the eager server, frame by frame, across key frames
(device-side key flag) and budgeted selection (device-side seq stamps)."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    from paper_2103_05875_b200 import build_native

    build_native.build()
    from paper_2103_05875_b200 import _native as N
    from paper_2103_05875_b200 import scene, server

    return N, scene, server


def test_frame_advance(mods):
    N, _, _ = mods
    st = torch.tensor([4, -1, 0], dtype=torch.int64, device="cuda")
    keys = []
    for _ in range(7):
        N.call("ps_frame_advance", st.data_ptr(), 3, torch.cuda.current_stream().cuda_stream)
        keys.append(int(st[2]))
    assert st[:2].tolist() == [11, 6]
    assert keys == [1, 0, 0, 1, 0, 0, 1]
    with pytest.raises(ValueError):
        N.call("ps_frame_advance", st.data_ptr(), 0, torch.cuda.current_stream().cuda_stream)


def _same(a, b):
    return torch.equal(a.view(torch.uint8), b.view(torch.uint8))


@pytest.mark.parametrize("budget,overlap", [(None, True), (90, True), (None, False)])
def test_graphed_server_bit_identical(mods, budget, overlap):
    _, scene, server = mods
    sc = scene.cornell_box()
    vol = scene.volume_for(sc, (8, 8, 8))
    kw = dict(rays_per_probe=64, gop_length=3, budget=budget, overlap=overlap,
              irradiance_scale=2.0, shadow_map_size=64,
              slot_count=None if budget is None else 128)
    eager = server.ProbeStreamServer(vol, sc, **kw)
    graphed = server.ProbeStreamServer(vol, sc, graphs=True, **kw)
    for f in range(9):
        lights = scene.moving_light(sc, f, period=8).lights
        ref = eager.tick(f, lights)
        out = graphed.tick(f, lights)
        torch.cuda.synchronize()
        for name, a, b in zip(("color", "visibility"), out, ref):
            n = int(b.entry_count.item())
            assert a.key == b.key, (f, name)
            assert int(a.entry_count.item()) == n, (f, name)
            assert torch.equal(a.entries[:n], b.entries[:n]), (f, name)
            assert _same(a.planes, b.planes), (f, name)
            assert _same(a.skip, b.skip), (f, name)
            assert _same(a.residual, b.residual), (f, name)
        for ka, kb in ((graphed.color, eager.color), (graphed.visibility, eager.visibility)):
            assert _same(ka.last_sent.texels, kb.last_sent.texels), f
            assert torch.equal(ka.last_sent_seq, kb.last_sent_seq), f
    assert len(graphed.updater.graphs) >= 1
    assert len(graphed.color.graphs) >= 1


def test_graphed_server_async_frames_match_eager(mods):
    """Frames issued back to back without host syncs (the bench's pattern:
    early shadow maps on their side stream overlapping the previous blend,
    chains overlapping the next trace): every frame's outputs, snapshotted
    on the stream that produced them, equal the eager server's."""
    _, scene, server = mods
    sc = scene.cornell_box()
    vol = scene.volume_for(sc, (8, 8, 8))
    kw = dict(rays_per_probe=64, gop_length=4, irradiance_scale=2.0, shadow_map_size=64)
    eager = server.ProbeStreamServer(vol, sc, **kw)
    graphed = server.ProbeStreamServer(vol, sc, graphs=True, **kw)
    frames = 10
    snaps = []
    for f in range(frames):
        lights = scene.moving_light(sc, f, period=5).lights
        outs = graphed.tick(f, lights)
        snap = []
        for kind, o in zip(("color", "visibility"), outs):
            with torch.cuda.stream(graphed.output_stream(kind)):
                n = o.entry_count.clone()
                snap.append((n, o.entries.clone(), o.planes.clone(), o.residual.clone(),
                             o.skip.clone()))
        snaps.append(snap)
    graphed.join()
    torch.cuda.synchronize()
    for f in range(frames):
        lights = scene.moving_light(sc, f, period=5).lights
        ref = eager.tick(f, lights)
        eager.join()
        torch.cuda.synchronize()
        for (n, ent, planes, res, skip), b in zip(snaps[f], ref):
            m = int(b.entry_count.item())
            assert int(n.item()) == m, f
            assert torch.equal(ent[:m], b.entries[:m]), f
            assert _same(planes, b.planes), f
            assert _same(res, b.residual), f
            assert _same(skip, b.skip), f
