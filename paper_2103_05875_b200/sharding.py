"""Multi-GPU z-slab sharding of the frame pipeline, plus bench helpers.

Probe id = i + nx*(j + ny*k) (volume.py:72-74), so a z-slab is a contiguous
ascending id range: rank r traces, blends and change-detects its slab only
(scene replicated).  The path has two exchanges per texture kind, both over
peer memory by default (distributed.py, csrc/ps_peer.cu): the change bitmap
(16 KB at 131,072 probes), ORed by every rank's detect kernel straight into
every rank's bitmap, so all ranks run the same global selection and slot
assignment (twin-replay determinism, test_packing.py:235-240); and the
selected cores, which each rank's export kernel writes straight into the
encoder rank's (0) update atlas, the single one it packs (the "single
encoder stream" of the north star).  PS_PEER=0 selects the NCCL path
(all-reduce of the bitmaps, send/recv of per-rank payloads).
"""

from __future__ import annotations

import torch

from . import _device as D
from .distributed import slab_range  # noqa: F401  (re-exported)
from .server import ProbeStreamServer


class SlabServer:
    """World size 1: the plain ProbeStreamServer.  World > 1: slab sharding."""

    def __init__(self, volume, scene, rays_per_probe=256, device=None, rank=0, world=1, **kw):
        self.rank, self.world = rank, world
        self.volume = volume
        self.device = torch.device(device) if device is not None else D.device_of()
        if world == 1:
            self.server = ProbeStreamServer(volume, scene, rays_per_probe, device=self.device, **kw)
            self.dist = None
        else:
            from .distributed import DistributedFrame

            self.server = None
            self.dist = DistributedFrame(volume, scene, rays_per_probe, self.device, rank, world, **kw)

    @property
    def impl(self):
        return self.server if self.server is not None else self.dist

    def tick(self, frame, lights=None):
        return self.impl.tick(frame, lights)

    def join(self) -> None:
        """Current stream waits for every stream the last frame used."""
        if hasattr(self.impl, "join"):
            self.impl.join()

    def _out_stream(self, kind):
        if hasattr(self.impl, "output_stream"):
            return self.impl.output_stream(kind)
        return torch.cuda.current_stream(self.device)

    # --- bench helpers ----------------------------------------------------------------

    def _barrier(self) -> None:
        torch.cuda.synchronize(self.device)
        if self.world > 1:
            import torch.distributed as dist

            dist.barrier()
            torch.cuda.synchronize(self.device)

    def run_e2e(self, steps: int, first_frame: int, lights_for):
        """Public-API frames with host I/O: per step the ray table and lights go
        H2D from pinned memory (inside tick) and the index entries, counts and
        SKIP maps come back D2H into pinned memory."""
        impl = self.impl
        outs = impl.tick(first_frame, lights_for(first_frame))  # shapes for the host buffers
        torch.cuda.synchronize(self.device)
        host = []
        for o in outs:
            if o is None:
                host.append(None)
                continue
            host.append((torch.empty_like(o.entries, device="cpu").pin_memory(),
                         torch.empty_like(o.entry_count, device="cpu").pin_memory(),
                         torch.empty_like(o.skip, device="cpu").pin_memory()))
        d2h = sum(h[0].numel() * 8 + 8 + h[2].numel() for h in host if h is not None)
        h2d = impl.h2d_bytes_per_frame()
        stream = torch.cuda.current_stream(self.device)
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        self._barrier()  # every rank done with its setup before any starts the clock
        start.record(stream)
        for k in range(steps):
            f = first_frame + 1 + k
            outs = impl.tick(f, lights_for(f))
            for kind, o, h in zip(("color", "visibility"), outs, host):
                if o is None:
                    continue
                with torch.cuda.stream(self._out_stream(kind)):  # ordered after the chain
                    h[0].copy_(o.entries, non_blocking=True)
                    h[1].copy_(o.entry_count, non_blocking=True)
                    h[2].copy_(o.skip, non_blocking=True)
        self.join()
        end.record(stream)
        torch.cuda.synchronize(self.device)
        return {"ms_per_step": start.elapsed_time(end) / steps, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h}

    def run_e2e_encoded(self, steps: int, first_frame: int, lights_for) -> dict:
        """End to end including §8(f)1/4: every frame is encoded to LPF1 on the
        device and the wire bytes (frames + index buffers) are read back to
        pinned host memory -- what a server sends to its client.  Read-back
        runs one frame behind: after issuing frame f the host waits for frame
        f-1's lengths (its stage chains finish while frame f traces) and queues
        the D2H of its bytes, so the pipeline never drains."""
        impl = self.impl
        if not hasattr(impl, "color") or not hasattr(impl.color, "encode"):
            return {}
        kinds = (impl.color, impl.visibility)
        for ks in kinds:
            ks.encode = True
        try:
            impl.tick(first_frame, lights_for(first_frame))  # buffers + warm
            torch.cuda.synchronize(self.device)
            host = {ks.kind.value: torch.empty(256 << 20, dtype=torch.uint8).pin_memory() for ks in kinds}
            lens = {ks.kind.value: torch.zeros((2, 2), dtype=torch.int64).pin_memory() for ks in kinds}
            d2h = [0]

            def issue_lens(outs, par):
                evs = []
                for ks, o in zip(kinds, outs):
                    st = self._out_stream(ks.kind.value)
                    with torch.cuda.stream(st):
                        lens[ks.kind.value][par, 0:1].copy_(o.frame_len, non_blocking=True)
                        lens[ks.kind.value][par, 1:2].copy_(o.index_len, non_blocking=True)
                        ev = torch.cuda.Event()
                        ev.record(st)
                    evs.append(ev)
                return evs

            def drain(outs, evs, par):
                for ks, o, ev in zip(kinds, outs, evs):
                    ev.synchronize()
                    n, ni = int(lens[ks.kind.value][par, 0]), int(lens[ks.kind.value][par, 1])
                    hb = host[ks.kind.value]
                    with torch.cuda.stream(self._out_stream(ks.kind.value)):
                        hb[:n].copy_(o.frame[:n], non_blocking=True)
                        hb[n:n + ni].copy_(o.index[:ni], non_blocking=True)
                    d2h[0] += n + ni + 16

            stream = torch.cuda.current_stream(self.device)
            start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            self._barrier()
            start.record(stream)
            prev = None
            for k in range(steps):
                f = first_frame + 1 + k
                outs = impl.tick(f, lights_for(f))
                evs = issue_lens(outs, k & 1)
                if prev is not None:
                    drain(*prev)
                prev = (outs, evs, k & 1)
            drain(*prev)
            self.join()
            end.record(stream)
            torch.cuda.synchronize(self.device)
            return {"ms_per_step": start.elapsed_time(end) / steps,
                    "h2d_bytes_per_step": impl.h2d_bytes_per_frame(),
                    "d2h_bytes_per_step": d2h[0] // steps}
        finally:
            for ks in kinds:
                ks.encode = False

    def stage_times(self, frames: int, first_frame: int, lights_for) -> dict:
        """Per-stage device times, measured with the stages serialised on one
        stream (no overlap) so each interval is that stage alone."""
        impl = self.impl
        torch.cuda.synchronize(self.device)
        overlap = getattr(impl, "overlap", False)
        if overlap:
            impl.overlap = False
        impl.enable_stage_timers(True)
        for k in range(frames):
            impl.tick(first_frame + k, lights_for(first_frame + k))
            # one frame at a time: the next frame's early shadow maps (probes.py)
            # would otherwise run beside this frame's stage chains
            torch.cuda.synchronize(self.device)
        t = impl.stage_times_ms()
        impl.enable_stage_timers(False)
        if overlap:
            impl.overlap = True
        return t

    def count_launches(self, frame: int, lights_for):
        from torch.profiler import ProfilerActivity, profile

        impl = self.impl
        torch.cuda.synchronize(self.device)
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            impl.tick(frame, lights_for(frame))
            torch.cuda.synchronize(self.device)
        import re

        names = {}
        total = 0
        for ev in prof.events():
            if ev.device_type != torch.autograd.DeviceType.CUDA:
                continue
            low = ev.name.lower()
            if "memcpy" in low or "memset" in low:
                continue
            key = ev.name.replace("(anonymous namespace)::", "").replace("void ", "")
            key = re.sub(r"<.*", "", key.split("(")[0])
            names[key] = names.get(key, 0) + 1
            if not key.startswith("nccl"):  # NCCL's own kernels are listed, not counted
                total += 1
        return total, names

    def pack_delta_bytes(self) -> dict:
        return self.impl.pack_delta_bytes()

    def pass_times(self, reps: int = 3) -> dict:
        """Probe-ray and blend pass device times of this rank (last measurement:
        it advances the probe state)."""
        torch.cuda.synchronize(self.device)
        return self.impl.updater.pass_times_ms(reps)

    def encode_times(self, reps: int = 3) -> dict:
        """§8(f)1 LPF1 encoding of the last frame's planes (key and P-frame),
        device time per frame and compression ratio; not part of the step."""
        from .codec import encode_frame_device

        impl = self.impl
        if not hasattr(impl, "color") or getattr(impl.color, "planes", None) is None:
            return {}
        torch.cuda.synchronize(self.device)
        out = {}
        for ks in (impl.color, impl.visibility):
            cur, prev = ks.planes[ks._cur], ks.planes[1 - ks._cur]  # newest after _advance
            raw = cur.numel() * cur.element_size()
            for tag, ref in (("key", None), ("p", prev)):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                encode_frame_device(cur, ref, 99, 0)  # warm
                a.record()
                for _ in range(reps):
                    _, ln = encode_frame_device(cur, ref, 99, 0)
                b.record()
                torch.cuda.synchronize(self.device)
                n = int(ln.item())
                out[f"{ks.kind.value}.{tag}"] = {"ms": round(a.elapsed_time(b) / reps, 4),
                                                 "bytes": n, "ratio": round(raw / n, 3)}
        return out
