"""§8(f) row 3: client side on the GPU -- LPF1 decode (against the reference's
own encoded frames) and the end-to-end master invariant of the server path:
after every frame, the client's atlases rebuilt from the decoded bitstream,
the index entries and the guard-band rule equal the server's last-sent
atlases bit for bit (SPEC.md server invariants)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    from paper_2103_05875_b200 import build_native

    build_native.build()
    from paper_2103_05875_b200 import codec, packing, scene, server

    return codec, packing, scene, server


def test_decode_reference_frames(mods, golden):
    codec, packing, _, _ = mods
    g = golden("codec")
    for s in range(int(g["nseq"])):
        state = codec.CodecStreamState(int(g[f"s{s}_stream"]), role="decoder")
        for f in range(int(g[f"s{s}_frames"])):
            wire = g[f"s{s}_f{f}_bytes"].tobytes()
            import struct
            magic, flags, sid, seq, w, h, planes, bits, plen = struct.unpack_from("<4sBIIHHBBI", wire)
            frame = codec.EncodedFrame(sid, seq, bool(flags & 1), w, h, planes, bits, wire[23:23 + plen])
            out = codec.decode_frame(frame, state)
            assert np.array_equal(out.data.cpu().numpy(), g[f"s{s}_f{f}_planes"]), (s, f)


def test_encode_decode_round_trip_long(mods):
    codec, packing, _, _ = mods
    rng = np.random.default_rng(4)
    enc = codec.CodecStreamState(3, gop_length=7)
    dec = codec.CodecStreamState(3, role="decoder")
    cur = rng.integers(0, 1024, size=(3, 90, 141), dtype=np.uint16)
    for f in range(20):
        m = rng.random(cur.shape) < 0.03
        cur = cur.copy()
        cur[m] = rng.integers(0, 1024, size=int(m.sum()), dtype=np.uint16)
        frame = codec.encode_frame(packing.PlaneSet(packing.PlaneKind.COLOR_10IN16, cur), enc)
        out = codec.decode_frame(frame, dec)
        assert np.array_equal(out.data.cpu().numpy(), cur), f


def test_corrupt_frames_rejected(mods):
    codec, packing, _, _ = mods
    rng = np.random.default_rng(5)
    cur = rng.integers(0, 256, size=(3, 32, 32), dtype=np.uint8)
    enc = codec.CodecStreamState(1)
    frame = codec.encode_frame(packing.PlaneSet(packing.PlaneKind.VISIBILITY_BYTES, cur), enc)
    bad = codec.EncodedFrame(frame.stream_id, frame.frame_seq, True, frame.width, frame.height,
                             frame.plane_count, frame.element_bits, frame.payload[:-3])
    with pytest.raises(codec.CodecError):
        codec.decode_frame(bad, codec.CodecStreamState(1, role="decoder"))
    p = codec.encode_frame(packing.PlaneSet(packing.PlaneKind.VISIBILITY_BYTES, cur), enc)
    with pytest.raises(codec.MissingReferenceError):
        codec.decode_frame(p, codec.CodecStreamState(1, role="decoder"))


@pytest.mark.parametrize("config,dims,rays,budget", [("cornell", (8, 8, 8), 64, None),
                                                     ("cornell", (8, 8, 8), 64, 100),
                                                     ("hall", (16, 8, 16), 64, None)])
def test_master_invariant_end_to_end(mods, config, dims, rays, budget):
    codec, packing, scene, server = mods
    sc = scene.cornell_box() if config == "cornell" else scene.interior_hall(detail=0.2)
    vol = scene.volume_for(sc, dims)
    slots = vol.probe_count if budget is None else 128
    srv = server.ProbeStreamServer(vol, sc, rays_per_probe=rays, encode=True, gop_length=4,
                                   budget=budget, slot_count=slots, irradiance_scale=2.0)
    from paper_2103_05875_b200.volume import ProbeAtlas

    clients = {}
    for ks in (srv.color, srv.visibility):
        clients[ks.kind.value] = {
            "atlas": ProbeAtlas(ks.kind, vol.probe_count, ks.last_sent.probes_per_row, device="cuda"),
            "ref": None,
        }
    for f in range(6):
        outs = srv.tick(f, scene.moving_light(sc, f).lights)
        torch.cuda.synchronize()
        for ks, out in zip((srv.color, srv.visibility), outs):
            cl = clients[ks.kind.value]
            n = int(out.frame_len.item())
            eb = 2 if ks.kind.value == "color" else 1
            h, w = out.planes.shape[1:]
            planes, status = codec.decode_frame_device(out.frame, n - 27, None if out.key else cl["ref"],
                                                       h, w, eb)
            torch.cuda.synchronize()
            assert int(status.item()) == 0
            assert torch.equal(planes.view(torch.uint8), out.planes.view(torch.uint8)), (f, ks.kind)
            cl["ref"] = planes
            pset = packing.PlaneSet(
                packing.PlaneKind.COLOR_10IN16 if eb == 2 else packing.PlaneKind.VISIBILITY_BYTES, planes)
            tex = (packing.unpack_color(pset) if eb == 2 else
                   packing.unpack_visibility(pset, ks.update_texels.shape[1]))
            packing.apply_update_entries_device(out.entries, out.entry_count, tex, ks.layout, cl["atlas"])
            torch.cuda.synchronize()
            a = cl["atlas"].texels.view(torch.int32) if eb == 2 else cl["atlas"].texels.view(torch.int16)
            b = ks.last_sent.texels.view(torch.int32) if eb == 2 else ks.last_sent.texels.view(torch.int16)
            assert torch.equal(a, b), (config, f, ks.kind)
