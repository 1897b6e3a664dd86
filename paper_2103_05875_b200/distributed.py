"""Slab-sharded frame over N GPUs of one node (one process per GPU).

Per frame, every rank r (z-slab [b_r, e_r), scene replicated):

1. traces + blends its own probes (ProbeUpdater with probe_range);
2. per texture kind, change-detects its slab only;
3. EXCHANGE 1 -- the change bitmap: slabs are disjoint, so the global bitmap
   is the OR of the ranks' bits.  Default (peer memory): the detect kernel
   ORs every changed word straight into each rank's bitmap, mapped with CUDA
   IPC, with system-scope atomics over NVLink -- detection and the all-gather
   are one kernel -- and per-rank release / acquire flags order it with the
   readers.  PS_PEER=0: an int32 NCCL all-reduce(SUM) of the bitmaps;
4. runs the same selection and slot assignment on every rank (replicated,
   deterministic: twin layouts replay identically, test_packing.py:235-240);
5. EXCHANGE 2 -- the selected cores: default, each rank's export kernel
   writes its own probes' cores directly into the encoder rank's update
   atlas at their slots (build and gather in one kernel), commits its blocks
   into last_sent and stamps last_sent_seq for every entry, then raises the
   encoder's flag; PS_PEER=0: a payload per rank, NCCL send/recv to the
   encoder rank and an import pass;
6. the encoder rank waits for every rank's flag and runs pack + temporal
   delta on the single update atlas (the north star's "single encoder
   stream").

The encoder rank's outputs are bit-identical to the single-GPU pipeline's
(tests/test_gpu_dist.py, both exchange paths, eager and CUDA-graph replay).
"""

from __future__ import annotations

import ctypes
import os

import torch
import torch.distributed as dist

from . import _device as D
from . import _native as N
from .delta import pack_delta, skip_shape
from .packing import UpdateAtlasLayout, widened_width
from .probes import ProbeUpdater
from .scene import DeviceScene
from .selection import _threshold_args, detect_changed_device, select_device
from .server import DEFAULT_GOP, DIST_CHAIN_PRIORITY, DIST_RESERVE_SMS, KindOutput
from .volume import AtlasKind, ProbeAtlas


def _peer_timeout_ns() -> int:
    return int(float(os.environ.get("PS_PEER_TIMEOUT_S", "30")) * 1e9)


_PEER_ERR: dict = {}


def peer_error_word(device) -> torch.Tensor:
    """The host-mapped pinned int32 that the bounded peer waits of this
    process report a timeout into (one per device; 0 = healthy)."""
    idx = torch.device(device).index
    w = _PEER_ERR.get(idx)
    if w is None:
        w = _PEER_ERR[idx] = torch.zeros(1, dtype=torch.int32, pin_memory=True)
    return w


def check_peers() -> None:
    """Raise (RuntimeError, PS_ERR_CUDA) if any peer wait of this process gave
    up on a rank that never signalled.  Reads pinned host memory only."""
    for w in _PEER_ERR.values():
        N.call("ps_peer_status", w.data_ptr())


def peer_wait(flags_ptr: int, nflags: int, seq: int, seq_dev_ptr, device, stream) -> None:
    """ps_peer_wait bounded by PS_PEER_TIMEOUT_S (default 30 s)."""
    N.call("ps_peer_wait", flags_ptr, nflags, int(seq), seq_dev_ptr, 1,
           peer_error_word(device).data_ptr(), _peer_timeout_ns(), stream)


def _env_flag(name: str, default: bool) -> bool:
    v = os.environ.get(name)
    return default if v is None else v not in ("0", "false", "no", "")


def _encoder_share() -> float:
    return float(os.environ.get("PS_ENCODER_SHARE", "1.0"))


def slab_range(volume, rank: int, world: int, encoder_share: float | None = None):
    """[begin, end) of rank's z-slab.  encoder_share = 1: whole k-planes,
    equal.  < 1: rank 0 (the encoder, which also packs the whole update
    atlas) gets that fraction of an equal share and the others split the rest,
    cut at rows of nx probes (PS_ENCODER_SHARE)."""
    nx, ny, nz = volume.dims
    plane = nx * ny
    share = _encoder_share() if encoder_share is None else encoder_share
    if world == 1 or share >= 1.0:
        return (nz * rank) // world * plane, (nz * (rank + 1)) // world * plane
    rows = ny * nz
    weights = [share] + [1.0] * (world - 1)
    total = sum(weights)
    cut = lambda r: int(round(rows * sum(weights[:r]) / total))
    return cut(rank) * nx, cut(rank + 1) * nx


def ranges_from_cost(n_units: int, unit: int, world: int, unit_cost) -> list:
    """Contiguous probe ranges of whole units (rows of nx probes) with
    near-equal summed cost; every rank gets at least one unit."""
    cost = [max(float(c), 1e-12) for c in unit_cost]
    total = sum(cost)
    cuts, acc, k = [0], 0.0, 0
    for r in range(1, world):
        target = total * r / world
        while k < n_units and acc + cost[k] / 2 < target and n_units - k > world - r:
            acc += cost[k]
            k += 1
        if k < cuts[-1] + 1:
            acc += sum(cost[k:cuts[-1] + 1])
            k = cuts[-1] + 1
        cuts.append(k)
    cuts.append(n_units)
    return [(cuts[r] * unit, cuts[r + 1] * unit) for r in range(world)]


def balanced_ranges(volume, scene, rays_per_probe, device, rank, world, sub: int = 8,
                    group=None, **probe_kwargs):
    """Cost-balanced slabs: every rank times the trace of ``sub`` pieces of
    its equal z-slab (CUDA events, no shadow pass), the timings are
    all-gathered and every rank cuts the probe rows (nx probes each) at equal
    cumulative cost -- identical ranges on every rank, so the sharded output
    stays bit-identical to one GPU.  Inner slabs of an interior scene cost
    ~9 % more than outer ones, more than a whole z-plane of granularity."""
    nx, ny, nz = volume.dims
    b, e = slab_range(volume, rank, world)
    r0, r1 = b // nx, e // nx
    kw = {k: v for k, v in probe_kwargs.items() if k not in ("shadows", "reserve_sms")}
    upd = ProbeUpdater(volume, scene, rays_per_probe=rays_per_probe, device=device,
                       probe_range=(b, e), shadows="none", **kw)
    upd.update(0)  # warm-up (weights, first-touch)
    nsub = max(1, min(sub, r1 - r0))
    bounds = [r0 + (r1 - r0) * i // nsub for i in range(nsub + 1)]
    local = torch.zeros(sub, dtype=torch.float64, device=device)
    for i in range(nsub):
        upd.probe_begin, upd.probe_end = bounds[i] * nx, bounds[i + 1] * nx
        best = None
        for rep in range(2):
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            upd.update(1 + rep)
            z.record()
            z.synchronize()
            t = a.elapsed_time(z)
            best = t if best is None else min(best, t)
        local[i] = best / max(1, bounds[i + 1] - bounds[i])  # ms per row
    del upd
    allc = torch.zeros(world * sub, dtype=torch.float64, device=device)
    dist.all_gather_into_tensor(allc, local, group=group)
    allc = allc.cpu().tolist()
    row_cost = [0.0] * (ny * nz)
    for r in range(world):
        rb, re_ = slab_range(volume, r, world)
        q0, q1 = rb // nx, re_ // nx
        n = max(1, min(sub, q1 - q0))
        bb = [q0 + (q1 - q0) * i // n for i in range(n + 1)]
        for i in range(n):
            for q in range(bb[i], bb[i + 1]):
                row_cost[q] = allc[r * sub + i]
    return ranges_from_cost(ny * nz, nx, world, row_cost)


def exchange_bitmap(bits: torch.Tensor, group=None) -> None:
    """In place: OR of the ranks' disjoint change bitmaps (all-reduce SUM of
    int32 words; disjoint bits never carry)."""
    dist.all_reduce(bits, op=dist.ReduceOp.SUM, group=group)


def gather_payloads(payload: torch.Tensor, payloads: torch.Tensor | None, rank: int,
                    world: int, encoder: int = 0, group=None) -> None:
    """Send every rank's payload to the encoder rank's ``payloads[r]``.

    The encoder's own payload is expected to already live in
    ``payloads[encoder]`` (it exports in place)."""
    ops = []
    if rank == encoder:
        for r in range(world):
            if r != encoder:
                ops.append(dist.P2POp(dist.irecv, payloads[r], r, group))
    else:
        ops.append(dist.P2POp(dist.isend, payload, encoder, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()


class PeerBuffers:
    """Every rank's copy of some device buffers, mapped into this process with
    CUDA IPC (handles exchanged once with an object all-gather): the device
    pointers the peer-memory kernels read and write over NVLink."""

    def __init__(self, tensors: dict, rank: int, world: int, group=None):
        hb = N.lib().ps_ipc_handle_bytes()
        mine = {}
        for name, t in tensors.items():
            if t is None:
                mine[name] = None
                continue
            h = (ctypes.c_uint8 * hb)()
            off = ctypes.c_int64()
            N.check(N.lib().ps_ipc_export(ctypes.c_void_p(t.data_ptr()), h, ctypes.byref(off)),
                    "ps_ipc_export")
            mine[name] = (bytes(h), off.value)
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        self.ptrs = {name: [] for name in tensors}
        for r in range(world):
            for name, t in tensors.items():
                if r == rank:
                    self.ptrs[name].append(t.data_ptr() if t is not None else 0)
                    continue
                e = allh[r][name]
                if e is None:
                    self.ptrs[name].append(0)
                    continue
                p = ctypes.c_void_p()
                buf = (ctypes.c_uint8 * hb).from_buffer_copy(e[0])
                N.check(N.lib().ps_ipc_open(buf, e[1], ctypes.byref(p)), "ps_ipc_open")
                self.ptrs[name].append(int(p.value))


class DistKindStream:
    def __init__(self, kind: AtlasKind, volume, device, rank, world, ranges, encoder=0,
                 slot_count=None, threshold=0.0, gop_length=DEFAULT_GOP, budget=None,
                 probes_per_row=None, peer: bool = False):
        self.kind, self.volume, self.device = kind, volume, device
        self.rank, self.world, self.encoder = rank, world, encoder
        self.ranges = ranges
        self.begin, self.end = ranges[rank]
        n = volume.probe_count
        self.threshold, self.budget, self.gop_length = threshold, budget, gop_length
        self.frame_count = 0
        self.last_sent = ProbeAtlas(kind, n, probes_per_row, device=device)
        self.last_sent_seq = torch.full((n,), -1, dtype=torch.int64, device=device)
        self.layout = UpdateAtlasLayout(slot_count or n, kind.core_side, probe_count=n,
                                        device=device)
        self.bits = torch.empty((n + 31) // 32, dtype=torch.int32, device=device)
        # session-owned scratch + pinned active flags (see _device.Workspace)
        self.active = D.active_flags(volume, device)
        self.ws_detect = D.workspace(N.lib().ps_detect_workspace_bytes(n), device)
        self.ws_select = D.workspace(N.lib().ps_select_workspace_bytes(n), device)
        self.sel_ids = torch.empty(n, dtype=torch.int64, device=device)
        self.sel_count = torch.empty(1, dtype=torch.int64, device=device)
        core = kind.core_side ** 2
        self.slab_max = max(e - b for b, e in ranges)
        self.is_encoder = rank == encoder
        if self.is_encoder:
            self.payloads = torch.zeros((world, self.slab_max * core), dtype=torch.int32,
                                        device=device)
            self.payload = self.payloads[rank]
            self.rank_begin = torch.tensor([b for b, _ in ranges] + [ranges[-1][1]],
                                           dtype=torch.int64, device=device)
            shape = self.layout.texel_shape(kind)
            tdt = torch.uint32 if kind is AtlasKind.COLOR else torch.uint16
            self.update_texels = torch.zeros(shape, dtype=tdt, device=device)
            h, w = shape[0], shape[1]
            pw, pdt = (w, torch.uint16) if kind is AtlasKind.COLOR else (widened_width(w), torch.uint8)
            self.planes = [torch.zeros((3, h, pw), dtype=pdt, device=device) for _ in range(2)]
            self.residual = torch.zeros((3, h, pw), dtype=pdt, device=device)
            self.skip = torch.zeros(skip_shape(h, pw), dtype=torch.uint8, device=device)
            self._cur = 0
        else:
            self.payloads = None
            self.payload = torch.zeros(self.slab_max * core, dtype=torch.int32, device=device)
        self.timers = None
        self.graphs = None
        self.frame_state = torch.zeros(3, dtype=torch.int64, device=device)
        self._state_synced = False
        self.peer = peer
        if peer:
            self._setup_peer()

    def enable_graphs(self, on: bool = True) -> None:
        self.graphs = {} if on else None
        self._state_synced = False

    def _setup_peer(self) -> None:
        """Peer-memory exchange (no NCCL on the data path): two-parity change
        bitmaps every rank ORs into, per-rank flag slots, and the encoder's
        update atlas every rank exports its cores into."""
        dev, n, world = self.device, self.volume.probe_count, self.world
        words = (n + 31) // 32
        self.bits2 = torch.zeros((2, words), dtype=torch.int32, device=dev)
        self.flags = torch.zeros((2, world), dtype=torch.int64, device=dev)  # bits / export
        pb = PeerBuffers({"bits": self.bits2, "flags": self.flags,
                          "update": self.update_texels if self.is_encoder else None},
                         self.rank, world)
        self._pb = pb
        ptr = lambda xs: torch.tensor(xs, dtype=torch.int64, device=dev)
        self.dst_bits = [ptr([b + k * words * 4 for b in pb.ptrs["bits"]]) for k in range(2)]
        self.sig_bits = ptr([f + self.rank * 8 for f in pb.ptrs["flags"]])
        self.sig_export = ptr([pb.ptrs["flags"][self.encoder] + (world + self.rank) * 8])
        self.enc_update = pb.ptrs["update"][self.encoder]
        self.enc_update_stride = int(self.layout.texel_shape(self.kind)[1])

    def _issue_peer(self, rendered: ProbeAtlas, seq: int, pvs_bits, graphed: bool):
        """detect + bitmap all-gather in one kernel (peer atomics) -> flags ->
        selection -> assign -> export straight into the encoder's update atlas
        -> flag -> (encoder) pack + delta.  Kernels only: one CUDA graph."""
        tag, dev, world = self.kind.value, self.device, self.world
        st = D.stream_ptr(dev)
        seq_dev = self.frame_state[0:1] if graphed else None
        key_dev = self.frame_state[2:3].view(torch.int32)[:1] if graphed else None
        if graphed:
            N.call("ps_frame_advance", self.frame_state.data_ptr(), self.gop_length, st)
        k = self.frame_count & 1
        vol, src = self.volume, rendered
        thr, is64 = _threshold_args(self.threshold)
        self._mark(f"{tag}.detect", 0)
        N.call("ps_detect_changed_bcast", self.kind.native, src.texels.data_ptr(),
               self.last_sent.texels.data_ptr(), vol.probe_count, src.probes_per_row,
               src.block_rows, self.begin, self.end, self.active.data_ptr(), thr, is64,
               self.dst_bits[k].data_ptr(), world, st)
        self._mark(f"{tag}.detect", 1)
        self._mark(f"{tag}.exchange_bits", 0)
        N.call("ps_peer_signal", self.sig_bits.data_ptr(), world, int(seq), D.ptr(seq_dev), 1, st)
        peer_wait(self.flags.data_ptr(), world, seq, D.ptr(seq_dev), dev, st)
        self._mark(f"{tag}.exchange_bits", 1)
        entries, count = self._select_assign(self.bits2[k], pvs_bits, seq)
        self.bits2[k].zero_()  # ready for frame + 2 (peers write it only after our next flag)
        self._mark(f"{tag}.export", 0)
        N.call("ps_export_tiles_peer", self.kind.native, src.texels.data_ptr(), vol.probe_count,
               src.probes_per_row, entries.data_ptr(), count.data_ptr(), self.layout.slot_count,
               self.begin, self.end, self.layout.slots_per_row, self.enc_update,
               self.enc_update_stride, self.last_sent.texels.data_ptr(),
               self.last_sent_seq.data_ptr(), int(seq), D.ptr(seq_dev), st)
        self._mark(f"{tag}.export", 1)
        self._mark(f"{tag}.gather", 0)
        N.call("ps_peer_signal", self.sig_export.data_ptr(), 1, int(seq), D.ptr(seq_dev), 1, st)
        if self.is_encoder:
            peer_wait(self.flags[1].data_ptr(), world, seq, D.ptr(seq_dev), dev, st)
        self._mark(f"{tag}.gather", 1)
        if self.is_encoder:
            key = self.frame_count % self.gop_length == 0
            prev = self.planes[self._cur] if graphed or not key else None
            cur = self.planes[1 - self._cur]
            self._mark(f"{tag}.pack_delta", 0)
            pack_delta(self.update_texels, self.kind, prev, planes_out=cur,
                       residual=self.residual, skip=self.skip, key_dev=key_dev)
            self._mark(f"{tag}.pack_delta", 1)

    def _select_assign(self, bits, pvs_bits, seq: int):
        """Global selection + slot assignment, replicated on every rank.
        Without a budget the selection is the candidate bitmap itself and the
        slot cache assigns straight from it (ps_assign_slots_bits)."""
        tag = self.kind.value
        if self.budget is None and self.layout.slot_count >= self.volume.probe_count:
            self._mark(f"{tag}.assign", 0)
            out = self.layout.assign_bits_device(bits, pvs_bits)
            self._mark(f"{tag}.assign", 1)
            return out
        self._mark(f"{tag}.select", 0)
        select_device(bits, pvs_bits, self.volume, self.last_sent_seq, seq, self.budget,
                      out_ids=self.sel_ids, out_count=self.sel_count,
                      workspace_slot=self.ws_select, ordered=False, active=self.active)
        self._mark(f"{tag}.select", 1)
        self._mark(f"{tag}.assign", 0)
        out = self.layout.assign_device(self.sel_ids, self.sel_count)
        self._mark(f"{tag}.assign", 1)
        return out

    def _tick_peer(self, rendered: ProbeAtlas, seq: int, pvs_bits=None):
        graphed = self.graphs is not None and self.frame_count >= 1 and self.timers is None
        if not graphed:
            self._state_synced = False
            self._issue_peer(rendered, seq, pvs_bits, graphed=False)
            return self._finish()
        if not self._state_synced:
            self.frame_state.copy_(torch.tensor([seq - 1, self.frame_count - 1, 0],
                                                dtype=torch.int64))
            self._state_synced = True
        key = ("peer", rendered.texels.data_ptr(), getattr(self, "_cur", 0), self.frame_count & 1,
               D.ptr(pvs_bits))
        g = self.graphs.get(key)
        if g is None:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                self._issue_peer(rendered, seq, pvs_bits, graphed=True)
            self.graphs[key] = g
        g.replay()
        return self._finish()

    def _mark(self, name, stage):
        if self.timers is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.timers.setdefault(name, []).append((stage, e))

    def tick(self, rendered: ProbeAtlas, seq: int, pvs_bits=None):
        if self.peer:
            return self._tick_peer(rendered, seq, pvs_bits)
        graphed = self.graphs is not None and self.frame_count >= 1 and self.timers is None
        if not graphed:
            self._state_synced = False
        elif not self._state_synced:
            # state holds the previous frame's values; segment A advances it
            self.frame_state.copy_(torch.tensor([seq - 1, self.frame_count - 1, 0],
                                                dtype=torch.int64))
            self._state_synced = True
        return self._issue(rendered, seq, pvs_bits, graphed)

    def _segment(self, name: str, key: tuple, fn, graphed: bool) -> None:
        """Run ``fn`` eagerly, or replay its captured graph.  The NCCL
        exchanges stay outside the graphs (issued eagerly between segments),
        so a frame is 3 graph launches + 2 collectives per kind."""
        if not graphed:
            fn()
            return
        k = (name,) + key
        g = self.graphs.get(k)
        if g is None:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                fn()
            self.graphs[k] = g
        g.replay()

    def _finish(self):
        key = self.frame_count % self.gop_length == 0
        self.frame_count += 1
        if not self.is_encoder:
            return None
        cur = self.planes[1 - self._cur]
        self._cur = 1 - self._cur
        return KindOutput(cur, self.residual, self.skip, self.layout._entries,
                          self.layout._entry_count, key)

    def _issue(self, rendered: ProbeAtlas, seq: int, pvs_bits, graphed: bool):
        tag = self.kind.value
        dev = self.device
        seq_dev = self.frame_state[0:1] if graphed else None
        key_dev = self.frame_state[2:3].view(torch.int32)[:1] if graphed else None
        gkey = (rendered.texels.data_ptr(), getattr(self, "_cur", 0), D.ptr(pvs_bits))

        def seg_detect():
            if graphed:
                N.call("ps_frame_advance", self.frame_state.data_ptr(), self.gop_length,
                       D.stream_ptr(dev))
            self._mark(f"{tag}.detect", 0)
            detect_changed_device(rendered, self.last_sent, self.volume, self.threshold,
                                  bits=self.bits, with_ids=False, workspace_slot=self.ws_detect,
                                  probe_range=(self.begin, self.end), active=self.active)
            self._mark(f"{tag}.detect", 1)

        def seg_select_export():
            entries, count = self._select_assign(self.bits, pvs_bits, seq)
            self._mark(f"{tag}.export", 0)
            N.call("ps_export_tiles", self.kind.native, rendered.texels.data_ptr(),
                   self.volume.probe_count, rendered.probes_per_row, entries.data_ptr(),
                   count.data_ptr(), self.layout.slot_count, self.begin, self.end,
                   self.payload.data_ptr(), self.last_sent.texels.data_ptr(),
                   self.last_sent_seq.data_ptr(), int(seq), D.ptr(seq_dev), D.stream_ptr(dev))
            self._mark(f"{tag}.export", 1)

        def seg_import_pack():
            entries, count = self.layout._entries, self.layout._entry_count
            self._mark(f"{tag}.import", 0)
            N.call("ps_import_tiles", self.kind.native, self.payloads.data_ptr(), self.slab_max,
                   self.rank_begin.data_ptr(), self.world, entries.data_ptr(), count.data_ptr(),
                   self.layout.slot_count, self.layout.slots_per_row,
                   self.update_texels.data_ptr(), self.update_texels.shape[1],
                   D.stream_ptr(dev))
            self._mark(f"{tag}.import", 1)
            key = self.frame_count % self.gop_length == 0
            # graphed: the device flag decides key frames per replay
            prev = self.planes[self._cur] if graphed or not key else None
            cur = self.planes[1 - self._cur]
            self._mark(f"{tag}.pack_delta", 0)
            pack_delta(self.update_texels, self.kind, prev, planes_out=cur,
                       residual=self.residual, skip=self.skip, key_dev=key_dev)
            self._mark(f"{tag}.pack_delta", 1)

        self._segment("detect", gkey, seg_detect, graphed)
        self._mark(f"{tag}.exchange_bits", 0)
        exchange_bitmap(self.bits)
        self._mark(f"{tag}.exchange_bits", 1)
        self._segment("select", gkey, seg_select_export, graphed)
        self._mark(f"{tag}.gather", 0)
        gather_payloads(self.payload, self.payloads, self.rank, self.world, self.encoder)
        self._mark(f"{tag}.gather", 1)
        if self.is_encoder:
            self._segment("pack", gkey, seg_import_pack, graphed)
        return self._finish()


class DistributedFrame:
    """One client session's hot path sharded over the process group."""

    def __init__(self, volume, scene, rays_per_probe, device, rank, world, encoder=None,
                 color_threshold=0.0, visibility_threshold=0.0, slot_count=None, budget=None,
                 gop_length=DEFAULT_GOP, overlap: bool = True, graphs: bool = False,
                 balance: bool = _env_flag("PS_BALANCE", False),
                 shard_shadows: bool = _env_flag("PS_SHADOW_SHARD", False),
                 peer: bool = _env_flag("PS_PEER", True), **probe_kwargs):
        self.volume, self.device, self.rank, self.world = volume, device, rank, world
        # peer (default; PS_PEER=0 for NCCL): the change-bitmap all-gather is fused
        # into the detect kernel (system atomics into every rank's mapped bitmap)
        # and the core gather into the export kernel (stores into the encoder's
        # mapped update atlas), ordered by release / acquire flags: no NCCL on the
        # data path and one CUDA graph per kind (N=4 C4: 2.67 -> 2.34 ms/frame).
        # balance / shard_shadows (off by default, PS_BALANCE / PS_SHADOW_SHARD):
        # measured at N=4 on C4 both lose -- the per-frame shadow all-gather couples
        # the ranks' traces (a fast rank can no longer run a frame ahead), and cost
        # balancing hands the encoder rank, which also imports and packs the whole
        # update, more probes -- 2.99 / 2.91 ms vs 2.80 ms per frame
        if not isinstance(scene, DeviceScene):
            scene = scene.device(device)  # one BVH build, shared with the calibration
        if balance and world > 1:
            self.ranges = balanced_ranges(volume, scene, rays_per_probe, device, rank, world,
                                          **probe_kwargs)
        else:
            self.ranges = [slab_range(volume, r, world) for r in range(world)]
        # overlap: both kind chains (with their NCCL exchanges) run on side
        # streams concurrently with the next frame's trace, as on one GPU
        self.overlap = overlap
        self.updater = ProbeUpdater(volume, scene, rays_per_probe=rays_per_probe, device=device,
                                    probe_range=self.ranges[rank],
                                    atlas_buffers=2 if overlap else 1,
                                    reserve_sms=probe_kwargs.pop("reserve_sms", DIST_RESERVE_SMS) if overlap else 0, **probe_kwargs)
        # shadow maps: each rank traces 1/world of the texels; peer mode stores
        # them into every rank's maps directly, NCCL mode all-gathers them
        if shard_shadows:
            if peer:
                self.updater.set_shadow_peers(rank, world)
            else:
                self.updater.shadow_split = (rank, world, None)
        self.streams = {"color": torch.cuda.Stream(device, priority=DIST_CHAIN_PRIORITY),
                        "visibility": torch.cuda.Stream(device, priority=DIST_CHAIN_PRIORITY)}
        self._buf_done = [[], []]
        self._pending = []
        ppr = self.updater.color.probes_per_row
        # encoder ranks per kind: colour and visibility are separate encoder
        # streams, so at N = 2 they are packed on different ranks (colour on
        # rank 0, visibility on rank 1): the encoder-serial pack of the whole
        # update atlas, which the other ranks never do, is split over two ranks
        # (C4: 2.614 vs 2.632 ms).  From N = 4 the peer export traffic into
        # two encoder ranks costs more than it saves and both kinds stay on
        # rank 0 (1.488 vs 1.515 ms; profiles/dist_r2/head3).  encoder=r puts
        # both on rank r; PS_SPLIT_ENCODERS=0 / 1 forces one / two ranks.
        if encoder is None:
            split = _env_flag("PS_SPLIT_ENCODERS", world == 2) and world > 1
            encoder = (0, 1 if split else 0)
        elif isinstance(encoder, int):
            encoder = (encoder, encoder)
        self.encoders = tuple(int(e) for e in encoder)
        kw = dict(slot_count=slot_count, gop_length=gop_length, budget=budget,
                  probes_per_row=ppr, peer=peer)
        self.color = DistKindStream(AtlasKind.COLOR, volume, device, rank, world, self.ranges,
                                    encoder=self.encoders[0], threshold=color_threshold, **kw)
        self.visibility = DistKindStream(AtlasKind.VISIBILITY, volume, device, rank, world,
                                         self.ranges, encoder=self.encoders[1],
                                         threshold=visibility_threshold, **kw)
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

    def enable_stage_timers(self, on=True):
        self.timers = {} if on else None
        self.color.timers = self.timers
        self.visibility.timers = self.timers

    def tick(self, frame=None, lights=None, pvs_bits=None):
        frame = self.seq if frame is None else frame
        check_peers()
        main = torch.cuda.current_stream(self.device)
        if self.overlap:
            buf = self.updater.frames_done % 2
            for ev in self._buf_done[buf]:
                main.wait_event(ev)
        if self.timers is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.timers.setdefault("trace_blend", []).append((0, e))
        color, vis = self.updater.update(frame, lights)
        if self.timers is not None:
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
        # same program order on every rank: colour's collectives, then visibility's
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
        main = torch.cuda.current_stream(self.device)
        for ev in self._pending:
            main.wait_event(ev)
        check_peers()

    def output_stream(self, kind: str):
        return self.streams[kind] if self.overlap else torch.cuda.current_stream(self.device)

    def h2d_bytes_per_frame(self) -> int:
        u = self.updater
        return u.rays_per_probe * 16 + u.dscene.light_count * 24

    def pack_delta_bytes(self) -> dict:
        out = {}
        for ks in (self.color, self.visibility):
            if not ks.is_encoder:
                continue
            tex = ks.update_texels.numel() * ks.update_texels.element_size()
            pl = ks.planes[0].numel() * ks.planes[0].element_size()
            out[ks.kind.value] = tex + 3 * pl + ks.skip.numel()
        out["total"] = sum(out.values())
        return out

    def stage_times_ms(self) -> dict:
        out = {}
        for name, evs in (self.timers or {}).items():
            starts = [e for s, e in evs if s == 0]
            ends = [e for s, e in evs if s == 1]
            if starts and ends:
                out[name] = sum(a.elapsed_time(b) for a, b in zip(starts, ends)) / len(ends)
        return out
