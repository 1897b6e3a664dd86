"""Server-side frame pipeline: the caller of the hot path.

The reference's server ``on_tick`` (supplement Alg. 1) is
absent from /root/reference; this module plays its role for the
hot path only -- per frame and per texture kind:

  update probes (trace + blend)          probes.ProbeUpdater       stages 1+2
  detect_changed vs last-sent atlas      selection.py:284-323      stage 3
  select_for_client (staleness, budget)  selection.py:413-437      stage 3
  UpdateAtlasLayout.assign               packing.py:283-317        stage 4
  build_update_atlas + commit            packing.py:320-338, SPEC.md:341
  pack_texels + temporal delta / SKIP    packing.py:154, codec.py:207-272

Everything is stream-ordered on one CUDA stream with device-side counts; a
frame launches ~40 kernels and never synchronises with the host.  The
outputs are encoder-ready: packed planes, residual planes against the
previous frame's planes, the SKIP map and the (slot, probe) index entries.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _device as D
from . import _native as N
from .delta import pack_delta, skip_shape
from .packing import UpdateAtlasLayout, widened_width
from .probes import ProbeUpdater
from .selection import detect_changed_device, select_device
from .volume import AtlasKind, ProbeAtlas, ProbeVolume

DEFAULT_GOP = 30  # codec.py:46
# SMs the persistent tracer leaves to the previous frame's stage chains when
# they overlap (high-priority side streams); tunable via PS_RESERVE_SMS.
# Measured at C4, round 2 (N=1 ms/frame, reserve 0 / 2 / 4 / 6 / 8): 5.074 /
# 5.073 / 5.086 / 5.123 / 5.165; the z-slab ranks (distributed.py) keep 4
# (round 1, N=2 reserve 4 / 8: 4.79 / 4.88, N=4: 2.73 / 2.77)
RESERVE_SMS = int(__import__("os").environ.get("PS_RESERVE_SMS", "2"))
DIST_RESERVE_SMS = int(__import__("os").environ.get("PS_RESERVE_SMS", "4"))
# Stream priorities (-1 = high, 0 = default).  One GPU: stages 1-2 run on the
# server's own high-priority stream and the stage chains at default priority,
# so after the trace the blend (and the early shadow maps, probes.py) are
# scheduled ahead of the previous frame's leftover chain kernels (C4 N=1, with
# early shadow maps: 5.050 ms with the chains high, 5.043 with the trace high).
# The z-slab ranks (distributed.py) keep their chains high.  PS_MAIN_PRIORITY=
# "" runs stages 1-2 on the caller's current stream.
_env = __import__("os").environ
CHAIN_PRIORITY = int(_env.get("PS_CHAIN_PRIORITY", "0"))
DIST_CHAIN_PRIORITY = int(_env.get("PS_CHAIN_PRIORITY", "-1"))
_MAIN_PRIORITY = _env.get("PS_MAIN_PRIORITY", "-1")
MAIN_PRIORITY = int(_MAIN_PRIORITY) if _MAIN_PRIORITY != "" else None


@dataclass
class KindOutput:
    planes: torch.Tensor       # (3, h, w) uint16 / uint8, current frame
    residual: torch.Tensor     # (3, h, w) planes - previous planes (mod 2^bits)
    skip: torch.Tensor         # (3, ceil(h/16), ceil(w/16)) uint8
    entries: torch.Tensor      # (slot_count, 2) int64 (slot, probe), first entry_count valid
    entry_count: torch.Tensor  # (1,) int64
    key: bool                  # key frame (no temporal reference)
    frame: torch.Tensor | None = None      # LPF1 wire frame (encode=True), first frame_len bytes
    frame_len: torch.Tensor | None = None  # (1,) int64
    index: torch.Tensor | None = None      # probe index buffer (encode=True), first index_len bytes
    index_len: torch.Tensor | None = None


class KindStream:
    """Per texture kind server state for one client (SPEC.md ClientSession)."""

    def __init__(self, kind: AtlasKind, volume: ProbeVolume, device, slot_count=None,
                 slots_per_row=None, threshold: float = 0.0, gop_length: int = DEFAULT_GOP,
                 budget=None, probes_per_row=None, encode: bool = False, stream_id: int = 0):
        self.kind = kind
        self.encode = encode
        self.stream_id = stream_id
        self.volume = volume
        self.device = device
        n = volume.probe_count
        self.threshold = threshold
        self.budget = budget
        self.gop_length = gop_length
        self.frame_count = 0
        self.last_sent = ProbeAtlas(kind, n, probes_per_row, device=device)
        # never-sent probes are the most stale (selection.py:421-424)
        self.last_sent_seq = torch.full((n,), -1, dtype=torch.int64, device=device)
        self.layout = UpdateAtlasLayout(slot_count or n, kind.core_side, slots_per_row,
                                        probe_count=n, device=device)
        shape = self.layout.texel_shape(kind)
        tdt = torch.uint32 if kind is AtlasKind.COLOR else torch.uint16
        self.update_texels = torch.zeros(shape, dtype=tdt, device=device)
        h, w = shape[0], shape[1]
        pw, pdt = (w, torch.uint16) if kind is AtlasKind.COLOR else (widened_width(w), torch.uint8)
        self.planes = [torch.zeros((3, h, pw), dtype=pdt, device=device) for _ in range(2)]
        self.residual = torch.zeros((3, h, pw), dtype=pdt, device=device)
        self.skip = torch.zeros(skip_shape(h, pw), dtype=torch.uint8, device=device)
        self.bits = torch.empty((n + 31) // 32, dtype=torch.int32, device=device)
        self.sel_ids = torch.empty(n, dtype=torch.int64, device=device)
        self.sel_count = torch.empty(1, dtype=torch.int64, device=device)
        # session-owned scratch and flags: never shared with another session or
        # stream, never reallocated after a CUDA graph captured their pointers
        lib = N.lib()
        self.active = D.active_flags(volume, device)
        self.ws_detect = D.workspace(lib.ps_detect_workspace_bytes(n), device)
        self.ws_select = D.workspace(lib.ps_select_workspace_bytes(n), device)
        self._cur = 0
        self.timers = None  # optional dict of per-stage (start, end) event lists
        # CUDA-graph replay (enable_graphs): {seq, frame_count, key} live on the
        # device and advance inside the graph (ps_frame_advance)
        self.graphs = None
        self.frame_state = torch.zeros(3, dtype=torch.int64, device=device)
        self._state_synced = False
        self._wire = None  # LPF1 frame / index buffers (encode=True), two frame parities

    def _mark(self, name, stage):
        if self.timers is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.timers.setdefault(name, []).append((stage, e))

    def enable_graphs(self, on: bool = True) -> None:
        self.graphs = {} if on else None
        self._state_synced = False

    def _graphable(self) -> bool:
        return (self.graphs is not None and self.frame_count >= 1 and not self.encode
                and self.timers is None)

    def tick(self, rendered: ProbeAtlas, seq: int, pvs_bits=None) -> KindOutput:
        if self._graphable():
            return self._tick_graphed(rendered, seq, pvs_bits)
        self._state_synced = False
        return self._tick_eager(rendered, seq, pvs_bits)

    def _tick_graphed(self, rendered: ProbeAtlas, seq: int, pvs_bits=None) -> KindOutput:
        """Replay this kind's captured chain (one graph per atlas buffer /
        plane parity); identical kernels to the eager chain, with seq and the
        key-frame flag read from ``frame_state`` on the device."""
        if not self._state_synced:
            # state holds the previous frame's values; the graph advances it
            self.frame_state.copy_(torch.tensor([seq - 1, self.frame_count - 1, 0],
                                                dtype=torch.int64))
            self._state_synced = True
        key = (rendered.texels.data_ptr(), self._cur, D.ptr(pvs_bits))
        g = self.graphs.get(key)
        if g is None:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                self._issue(rendered, seq, pvs_bits, graphed=True)
            self.graphs[key] = g
        g.replay()
        return self._advance()

    def _issue(self, rendered: ProbeAtlas, seq: int, pvs_bits, graphed: bool):
        """Stream-ordered stage chain on the current stream; returns (entries,
        count, current planes)."""
        tag = self.kind.value
        seq_dev = key_dev = None
        if graphed:
            N.call("ps_frame_advance", self.frame_state.data_ptr(), self.gop_length,
                   D.stream_ptr(self.device))
            seq_dev = self.frame_state[0:1]
            key_dev = self.frame_state[2:3].view(torch.int32)[:1]
        self._mark(f"{tag}.detect", 0)
        detect_changed_device(rendered, self.last_sent, self.volume, self.threshold,
                              bits=self.bits, with_ids=False, workspace_slot=self.ws_detect,
                              active=self.active)
        self._mark(f"{tag}.detect", 1)
        if self.budget is None and self.layout.slot_count >= self.volume.probe_count:
            # no budget: the selection is the candidate set (changed & pvs &
            # active, detect applied active), so it stays a bitmap and the
            # slot cache assigns straight from it (ps_assign_slots_bits)
            self._mark(f"{tag}.assign", 0)
            entries, count = self.layout.assign_bits_device(self.bits, pvs_bits)
            self._mark(f"{tag}.assign", 1)
        else:
            self._mark(f"{tag}.select", 0)
            select_device(self.bits, pvs_bits, self.volume, self.last_sent_seq, seq, self.budget,
                          out_ids=self.sel_ids, out_count=self.sel_count,
                          workspace_slot=self.ws_select, ordered=False, active=self.active)
            self._mark(f"{tag}.select", 1)
            self._mark(f"{tag}.assign", 0)
            entries, count = self.layout.assign_device(self.sel_ids, self.sel_count)
            self._mark(f"{tag}.assign", 1)
        self._mark(f"{tag}.build", 0)
        N.call("ps_build_update", self.kind.native, rendered.texels.data_ptr(),
               self.volume.probe_count, rendered.probes_per_row, entries.data_ptr(),
               count.data_ptr(), self.layout.slot_count, self.layout.slots_per_row,
               self.update_texels.data_ptr(), self.update_texels.shape[1],
               self.last_sent.texels.data_ptr(), self.last_sent_seq.data_ptr(), int(seq),
               D.ptr(seq_dev), D.stream_ptr(self.device))
        self._mark(f"{tag}.build", 1)
        key = self.frame_count % self.gop_length == 0
        # graphed: the device flag decides key frames per replay
        prev = self.planes[self._cur] if graphed or not key else None
        cur = self.planes[1 - self._cur]
        self._mark(f"{tag}.pack_delta", 0)
        pack_delta(self.update_texels, self.kind, prev, planes_out=cur, residual=self.residual,
                   skip=self.skip, key_dev=key_dev)
        self._mark(f"{tag}.pack_delta", 1)
        return entries, count, cur

    def _advance(self, frame=None, frame_len=None, index=None, index_len=None) -> KindOutput:
        key = self.frame_count % self.gop_length == 0
        cur = self.planes[1 - self._cur]
        self._cur = 1 - self._cur
        self.frame_count += 1
        return KindOutput(cur, self.residual, self.skip, self.layout._entries,
                          self.layout._entry_count, key, frame, frame_len, index, index_len)

    def _tick_eager(self, rendered: ProbeAtlas, seq: int, pvs_bits=None) -> KindOutput:
        tag = self.kind.value
        key = self.frame_count % self.gop_length == 0
        prev = None if key else self.planes[self._cur]
        entries, count, cur = self._issue(rendered, seq, pvs_bits, graphed=False)
        frame = frame_len = index = index_len = None
        if self.encode:  # §8(f)1: LPF1 bitstream, bit-exact with codec.encode_frame
            from .codec import encode_frame_device
            from .index_buffer import encode_index_device

            self._mark(f"{tag}.encode", 0)
            # wire buffers ping-pong by frame parity, so a frame's bytes stay valid
            # while the next frame is encoded (a caller may read them a frame late)
            k = self.frame_count & 1
            if self._wire is None:
                cap = N.lib().ps_encode_frame_capacity(cur.shape[1], cur.shape[2],
                                                      cur.element_size())
                icap = 1 + 20 * max(int(entries.shape[0]), 1)
                self._wire = [(torch.empty(cap, dtype=torch.uint8, device=self.device),
                               torch.zeros(1, dtype=torch.int64, device=self.device),
                               torch.empty(icap, dtype=torch.uint8, device=self.device),
                               torch.zeros(1, dtype=torch.int64, device=self.device))
                              for _ in range(2)]
                lib = N.lib()
                self._ws_encode = D.workspace(lib.ps_encode_workspace_bytes(
                    cur.shape[1], cur.shape[2], cur.element_size()), self.device)
                self._ws_index = D.workspace(
                    lib.ps_index_workspace_bytes(int(entries.shape[0])), self.device)
            fb, fl, ib, il = self._wire[k]
            frame, frame_len = encode_frame_device(cur, prev, self.stream_id, self.frame_count,
                                                   out=fb, frame_len=fl,
                                                   workspace=self._ws_encode)
            index, index_len = encode_index_device(entries, count, out=ib, out_len=il,
                                                   workspace=self._ws_index)  # §8(f)4
            self._mark(f"{tag}.encode", 1)
        return self._advance(frame, frame_len, index, index_len)


class ProbeStreamServer:
    """One client session's hot path: probe update + both texture streams."""

    def __init__(self, volume: ProbeVolume, scene, rays_per_probe: int = 256, device=None,
                 color_threshold: float = 0.0, visibility_threshold: float = 0.0,
                 slot_count=None, budget=None, gop_length: int = DEFAULT_GOP,
                 overlap: bool = True, encode: bool = False, graphs: bool = False,
                 **probe_kwargs):
        self.device = torch.device(device) if device is not None else D.device_of()
        self.volume = volume
        # overlap: the colour and visibility chains run on their own streams,
        # concurrently with each other and with the next frame's trace (which
        # writes the other half of double-buffered atlases)
        self.overlap = overlap
        self.updater = ProbeUpdater(volume, scene, rays_per_probe=rays_per_probe,
                                    device=self.device, atlas_buffers=2 if overlap else 1,
                                    reserve_sms=probe_kwargs.pop("reserve_sms", RESERVE_SMS) if overlap else 0,
                                    **probe_kwargs)
        self.streams = ({"color": torch.cuda.Stream(self.device, priority=CHAIN_PRIORITY),
                         "visibility": torch.cuda.Stream(self.device, priority=CHAIN_PRIORITY)} if overlap else None)
        self._buf_done = [[], []]   # events: stages finished reading atlas buffer k
        self._pending = []          # events of the last frame's stage chains
        ppr = self.updater.color.probes_per_row
        self.color = KindStream(AtlasKind.COLOR, volume, self.device, slot_count,
                                threshold=color_threshold, gop_length=gop_length, budget=budget,
                                probes_per_row=ppr, encode=encode, stream_id=1)
        self.visibility = KindStream(AtlasKind.VISIBILITY, volume, self.device, slot_count,
                                     threshold=visibility_threshold, gop_length=gop_length,
                                     budget=budget, probes_per_row=ppr, encode=encode,
                                     stream_id=2)
        self.main_stream = (torch.cuda.Stream(self.device, priority=MAIN_PRIORITY)
                            if overlap and MAIN_PRIORITY is not None else None)
        self.seq = 0
        self.timers = None
        self.enable_graphs(graphs)

    def enable_graphs(self, on: bool = True) -> None:
        """Replay each frame as three captured CUDA graphs (trace + blend on
        the main stream, one stage chain per kind on its side stream) instead
        of ~130 individual launches; frame 0 always runs eagerly."""
        self.graphs = bool(on)
        for part in (self.updater, self.color, self.visibility):
            part.enable_graphs(on)

    def enable_stage_timers(self, on: bool = True) -> None:
        self.timers = {} if on else None
        self.color.timers = self.timers
        self.visibility.timers = self.timers

    def tick(self, frame: int | None = None, lights=None, pvs_bits=None):
        """One server frame; returns (colour KindOutput, visibility KindOutput).

        With ``overlap`` the outputs are produced on ``self.streams[kind]``;
        call ``join()`` (or wait on those streams) before reading them."""
        frame = self.seq if frame is None else frame
        if self.main_stream is not None:
            caller = torch.cuda.current_stream(self.device)
            self.main_stream.wait_stream(caller)
            with torch.cuda.stream(self.main_stream):
                outs = self._tick(frame, lights, pvs_bits)
            caller.wait_stream(self.main_stream)
            return outs
        return self._tick(frame, lights, pvs_bits)

    def _tick(self, frame, lights, pvs_bits):
        main = torch.cuda.current_stream(self.device)
        timing = self.timers is not None
        if self.overlap:
            buf = self.updater.frames_done % 2
            for ev in self._buf_done[buf]:  # trace may overwrite that atlas half now
                main.wait_event(ev)
        if timing:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.timers.setdefault("trace_blend", []).append((0, e))
        color, vis = self.updater.update(frame, lights)
        if timing:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.timers["trace_blend"].append((1, e))
        if not self.overlap:
            out_c = self.color.tick(color, self.seq, pvs_bits)
            out_v = self.visibility.tick(vis, self.seq, pvs_bits)
            self.seq += 1
            return out_c, out_v
        traced = torch.cuda.Event()
        traced.record(main)
        outs, done = [], []
        for ks, atlas in ((self.color, color), (self.visibility, vis)):
            st = self.streams[ks.kind.value]
            st.wait_event(traced)
            with torch.cuda.stream(st):
                outs.append(ks.tick(atlas, self.seq, pvs_bits))
                ev = torch.cuda.Event()
                ev.record(st)
                done.append(ev)
        self._buf_done[buf] = done
        self._pending = done
        self.seq += 1
        return tuple(outs)

    def join(self) -> None:
        """Make the current stream wait for the last frame's stage chains."""
        main = torch.cuda.current_stream(self.device)
        for ev in self._pending:
            main.wait_event(ev)

    def output_stream(self, kind: str):
        return self.streams[kind] if self.overlap else torch.cuda.current_stream(self.device)

    def h2d_bytes_per_frame(self) -> int:
        u = self.updater
        return u.rays_per_probe * 16 + u.dscene.light_count * 24

    def pack_delta_bytes(self) -> dict:
        """Algorithmic bytes of one pack+delta launch per kind: read the update
        texels and the previous planes, write planes + residual + SKIP map."""
        out = {}
        for ks in (self.color, self.visibility):
            tex = ks.update_texels.numel() * ks.update_texels.element_size()
            pl = ks.planes[0].numel() * ks.planes[0].element_size()
            out[ks.kind.value] = tex + 3 * pl + ks.skip.numel()
        out["total"] = sum(out.values())
        return out

    def stage_times_ms(self) -> dict:
        """Average per-stage device time from the recorded event pairs."""
        out = {}
        for name, evs in (self.timers or {}).items():
            starts = [e for s, e in evs if s == 0]
            ends = [e for s, e in evs if s == 1]
            if starts and ends:
                out[name] = sum(a.elapsed_time(b) for a, b in zip(starts, ends)) / len(ends)
        return out
