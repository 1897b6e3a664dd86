#!/usr/bin/env python
"""BASELINE config 5 / SURVEY §8(d) C5: the pack/select-only streaming path
(stages 3 + 4 without tracing) over N in {4k, 16k, 32k, 64k, 128k} probes from
precomputed synthetic atlases, at changed fractions p in {1.0, 0.1, 0.01} and
with all probes or 75 % of them active.

Inputs as §8(d) specifies: colour texels ``rng.integers(0, 2**30, u32)``,
visibility halves ``rng.integers(0, 0x7C00, u16)`` (finite, non-negative);
last_sent = rendered with one texel of a fraction p of the probes mutated.
Per iteration the last-sent atlas and staleness stamps are restored and L2
is flushed (a 256 MB write) outside the timed region; the chain (detect ->
select -> assign -> build + commit -> pack + temporal delta) is timed per
stage with CUDA events, P-frames (temporal delta against the previous planes),
then timed again as one CUDA-graph replay of the whole chain (``graphed_chain_ms``,
how the server issues it).

Achieved bandwidth uses §8(d)'s algorithmic bytes: detect 801 / 2,593 B per
probe + 8 B per changed id; build + pack 896 / 3,072 B and temporal delta
768 / 2,048 B per selected probe (colour / visibility); pack_delta is also
reported on its own over the whole update atlas it rewrites every frame.
``--cpu`` adds the numpy restatement of the reference stages (1 core, best
of 3) at N <= 16,384.

    python tools/sweep_c5.py [--iters 10] [--cpu] > gpurun_out/c5.json
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

DIMS = {4096: (16, 16, 16), 16384: (32, 16, 32), 32768: (32, 32, 32), 65536: (64, 32, 32),
        131072: (64, 32, 64)}
SURVEY_BYTES = {"color": (801, 896, 768), "visibility": (2593, 3072, 2048)}
PEAK = 6546.6  # GB/s, MEASURED_PEAKS.json hbm_gbs


def synth(kind, n, ppr, p, rng):
    from oracle import stream_ops as so

    shape = so.atlas_shape(kind, n, ppr)
    if kind == "color":
        cur = rng.integers(0, 2 ** 30, size=shape, dtype=np.uint32)
    else:
        cur = rng.integers(0, 0x7C00, size=shape, dtype=np.uint16)
    last = cur.copy()
    side = so.block_side(kind)
    mut = np.flatnonzero(rng.random(n) < p)
    for q in mut:
        br, bc = divmod(int(q), ppr)
        y, x = br * side + 1 + int(rng.integers(0, side - 2)), bc * side + 1 + int(rng.integers(0, side - 2))
        if kind == "color":
            last[y, x] ^= np.uint32(1 + int(rng.integers(0, 1023)))
        else:
            last[y, x, int(rng.integers(0, 2))] ^= np.uint16(1 + int(rng.integers(0, 0x3FF)))
    return cur, last, mut


def gpu_case(n, p, active_frac, iters, seed=0):
    import torch

    from paper_2103_05875_b200.server import KindStream
    from paper_2103_05875_b200.volume import AtlasKind, ProbeAtlas, ProbeVolume

    rng = np.random.default_rng(seed)
    active = np.ones(n, bool) if active_frac >= 1.0 else rng.random(n) < active_frac
    vol = ProbeVolume(DIMS[n], active=active)
    dev = torch.device("cuda")
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    out = {"n": n, "p": p, "active": active_frac, "kinds": {}}
    for kind in (AtlasKind.COLOR, AtlasKind.VISIBILITY):
        tag = kind.value
        ks = KindStream(kind, vol, dev, gop_length=1 << 30)
        ppr = ks.last_sent.probes_per_row
        cur, last, mut = synth(tag, n, ppr, p, rng)
        rendered = ProbeAtlas(kind, n, ppr, device=dev)
        rendered.texels.copy_(torch.from_numpy(cur.view(np.int32) if tag == "color" else cur.view(np.int16)).to(dev).view(rendered.texels.dtype))
        saved = torch.from_numpy(last.view(np.int32) if tag == "color" else last.view(np.int16)).to(dev).view(rendered.texels.dtype)
        changed = int(np.sum(active[mut])) if len(mut) else 0
        times = {}
        for it in range(iters + 2):
            ks.last_sent.texels.copy_(saved)
            ks.last_sent_seq.fill_(-1)
            flush.fill_(float(it))
            torch.cuda.synchronize()
            ks.timers = {} if it >= 2 else None
            o = ks.tick(rendered, it)
            torch.cuda.synchronize()
            if it >= 2:
                for name, evs in ks.timers.items():
                    a = [e for s, e in evs if s == 0][0]
                    b = [e for s, e in evs if s == 1][0]
                    times.setdefault(name.split(".")[1], []).append(a.elapsed_time(b))
        got = int(o.entry_count.item())
        # the same chain replayed as one CUDA graph (as the server runs it):
        # whole-chain time, no per-stage events
        ks.timers = None
        ks.enable_graphs(True)
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        graphed = []
        for it in range(iters + 2):
            ks.last_sent.texels.copy_(saved)
            ks.last_sent_seq.fill_(-1)
            flush.fill_(float(it))
            torch.cuda.synchronize()
            st.record()
            og = ks.tick(rendered, iters + 2 + it)
            en.record()
            torch.cuda.synchronize()
            if it >= 2:
                graphed.append(st.elapsed_time(en))
        assert int(og.entry_count.item()) == got
        med = {k: float(np.median(v)) for k, v in times.items()}
        total_ms = sum(med.values())
        det_b, bp_b, dl_b = SURVEY_BYTES[tag]
        alg = n * det_b + 8 * changed + changed * (bp_b + dl_b)
        tex = ks.update_texels.numel() * ks.update_texels.element_size()
        pl = ks.planes[0].numel() * ks.planes[0].element_size()
        pack_bytes = tex + 3 * pl + ks.skip.numel()
        out["kinds"][tag] = {
            "changed": changed, "selected": got, "stage_ms": {k: round(v, 4) for k, v in med.items()},
            "chain_ms": round(total_ms, 4),
            "algorithmic_bytes": alg,
            "achieved_gbs": round(alg / (total_ms / 1e3) / 1e9, 1),
            "frac_of_hbm": round(alg / (total_ms / 1e3) / 1e9 / PEAK, 4),
            "pack_delta_gbs": round(pack_bytes / (med["pack_delta"] / 1e3) / 1e9, 1),
            "pack_delta_frac": round(pack_bytes / (med["pack_delta"] / 1e3) / 1e9 / PEAK, 4),
            "hz_at_chain": round(1e3 / total_ms, 1),
            "graphed_chain_ms": round(float(np.median(graphed)), 4),
        }
        del ks
    return out


def cpu_case(n, p, seed=0):
    """numpy restatement of the reference stages, 1 core, best of 3."""
    from oracle import stream_ops as so

    rng = np.random.default_rng(seed)
    active = np.ones(n, bool)
    res = {}
    for kind in ("color", "visibility"):
        ppr = so.default_probes_per_row(n)
        cur, last, _ = synth(kind, n, ppr, p, rng)
        t = {}

        def best(f):
            b = None
            for _ in range(3):
                t0 = time.perf_counter()
                r = f()
                dt = time.perf_counter() - t0
                b = dt if b is None else min(b, dt)
            return r, b

        ch, t["detect"] = best(lambda: so.detect_changed(cur, last, kind, n, ppr, active))
        sel, t["select"] = best(lambda: so.select_for_client(ch, np.arange(n), active,
                                                             np.full(n, -1), 1))
        cache = so.SlotCache(n, so.block_side(kind) - 2)
        so.build_update_atlas(sel, cache, cur, kind, ppr)  # warm layout
        (tex, _), t["build"] = best(lambda: so.build_update_atlas(sel, cache, cur, kind, ppr))
        planes, t["pack"] = best(lambda: so.pack_texels(tex, kind))
        _, t["delta"] = best(lambda: so.temporal_delta(planes, planes))
        res[kind] = {k: round(1e3 * v, 3) for k, v in t.items()}
        res[kind]["total_ms"] = round(sum(res[kind].values()), 3)
    return {"n": n, "p": p, "cores": 1, "stage_ms": res}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--cpu", action="store_true")
    ap.add_argument("--sizes", default="4096,16384,32768,65536,131072")
    args = ap.parse_args()
    sizes = [int(x) for x in args.sizes.split(",")]
    rows = []
    for n in sizes:
        for p in (1.0, 0.1, 0.01):
            for act in (1.0, 0.75):
                rows.append(gpu_case(n, p, act, args.iters))
                print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
    cpu = [cpu_case(n, p) for n in sizes if n <= 16384 for p in (1.0, 0.01)] if args.cpu else []
    print(json.dumps({"config": "C5 pack/select-only sweep", "gpu": rows, "cpu_reference_port": cpu}))


if __name__ == "__main__":
    main()
