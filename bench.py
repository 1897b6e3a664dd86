#!/usr/bin/env python
"""Benchmark of the server-side probe hot path (BASELINE.json north_star).

A step is one full-volume server frame at config 4 (64x32x64 probes, 256 rays
per probe, the ~270k-triangle interior hall): trace + DDGI blend, then for
colour and visibility: change detection, budgeted selection, slot
assignment, update-atlas build + commit, plane packing + temporal delta.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun: probes shard by z-slab, value is
the whole-job probe updates/s, timed as the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "probe updates/s & Grays/s at 1/2/4/8 B200; packed-atlas GB/s vs HBM roofline"
CONFIGS = {
    # name: (dims, rays, scene)
    "c4": ((64, 32, 64), 256, "hall"),
    "c2": ((32, 16, 32), 256, "hall"),
    "c1": ((8, 8, 8), 64, "cornell"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled through NVML every
    ~5 ms while the timed region runs (falls back to nvidia-smi)."""

    REASONS = {
        "hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
        "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
        "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
        "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
        "hw_power_brake": "nvmlClocksEventReasonHwPowerBrakeSlowdown",
    }

    def __init__(self, index: int, period_s: float = 0.005):
        self.index = index
        self.period = period_s
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._thread = None
        self._nvml = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            visible = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(visible.split(",")[self.index]) if visible else self.index
            h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self._nvml = (pynvml, h)
        except Exception:
            self._nvml = None
            return self

        def loop():
            pynvml, h = self._nvml
            while not self._stop.is_set():
                try:
                    mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    reasons = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((mhz, reasons))
                except Exception:
                    pass
                time.sleep(self.period)

        self._thread = threading.Thread(target=loop, daemon=True)
        self._thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread is not None:
            self._thread.join(timeout=2)

    def summary(self):
        import statistics

        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["no NVML samples"]}
        pynvml = self._nvml[0]
        reasons = set()
        for _, bits in self.samples:
            for name, attr in self.REASONS.items():
                if bits & getattr(pynvml, attr, 0):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(m for m, _ in self.samples),
                "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons),
                "samples": len(self.samples), "source": "NVML"}


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_summary_path() -> Path:
    """The newest committed ncu summary (profiles/ncu_summary_r*.json, else
    the round-1 profiles/ncu_summary.json)."""
    rounds = sorted((ROOT / "profiles").glob("ncu_summary_r*.json"))
    return rounds[-1] if rounds else ROOT / "profiles" / "ncu_summary.json"


def profile_metric(prefix: str, key: str):
    """A fraction (pct / 100) for the first kernel starting with `prefix` in the
    committed ncu summary, or None."""
    p = ncu_summary_path()
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text()).get("kernels", {})
        for k, v in d.items():
            if k.startswith(prefix) and key in v:
                return round(float(v[key]) / 100.0, 4)
    except Exception:
        return None
    return None


def trace_issue_profile():
    """Warp instructions per C4 trace launch and the capture they come from
    (profiles/trace_accounting_*.json, newest round first), or None."""
    for p in sorted((ROOT / "profiles").glob("trace_accounting_r*.json"), reverse=True):
        try:
            d = json.loads(p.read_text())
            return {"warp_inst_per_launch": d["totals"]["warp_inst"],
                    "thread_inst_per_ray": d["per_ray"]["thread_inst"],
                    "simt_efficiency": d["simt_efficiency"], "source": f"profiles/{p.name}",
                    "kernel": d["kernel"]}
        except Exception:
            continue
    return None


def profile_traffic(prefix: str):
    """DRAM bytes (read + write) per launch, summed over the kernels whose name
    starts with `prefix` (one launch per texture kind), from the committed
    ncu summary (profiles/ncu_summary_r*.json); None if absent."""
    p = ncu_summary_path()
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text()).get("kernels", {})
        vals = [v["dram_bytes_per_launch"] for k, v in d.items()
                if k.startswith(prefix) and "dram_bytes_per_launch" in v]
        return round(sum(vals)) if vals else None
    except Exception:
        return None


# --------------------------------------------------------------------------------------------


def trace_roofline(trace_ms, rays_total, world, clocks) -> dict:
    """The trace is issue-bound (no HBM / tensor roofline): its bound is the
    SM issue rate, 148 SMs x 4 schedulers x 1 warp instruction per clock.
    achieved = the warp instructions one launch executes (ncu capture of the
    same kernel, profiles/trace_accounting_*.json; divided by the ranks for a
    slab) / the live CUDA-event time of the launch."""
    out = {"kernel": "trace_kernel (probe rays, this rank's slab; CUDA events, pass alone)",
           "ms": round(trace_ms, 4),
           "rays_per_s": round(rays_total / world / (trace_ms / 1e3), 1),
           "bound": "issue"}
    prof = trace_issue_profile()
    mhz = (clocks.summary() or {}).get("sm_mhz") or 1965
    if prof:
        import torch

        sms = torch.cuda.get_device_properties(0).multi_processor_count
        peak = sms * 4 * mhz * 1e6  # warp instructions / s
        achieved = prof["warp_inst_per_launch"] / world / (trace_ms / 1e3)
        out.update({"achieved": round(achieved / 1e9, 1), "peak": round(peak / 1e9, 1),
                    "unit": "G warp-inst/s", "frac": round(achieved / peak, 4),
                    "warp_inst_per_launch": int(prof["warp_inst_per_launch"] / world),
                    "thread_inst_per_ray": prof["thread_inst_per_ray"],
                    "simt_efficiency": prof["simt_efficiency"],
                    "profile": prof["source"], "profiled_kernel": prof["kernel"]})
    return out


def build_scene(name):
    from paper_2103_05875_b200 import scene as S

    return S.interior_hall() if name == "hall" else S.cornell_box()


def make_config(args, sc, vol, world) -> dict:
    """The workload description, identical in both arms (ours / reference)."""
    dims, rays, _ = CONFIGS[args.config]
    return {
        "workload": f"config 4: {dims[0]}x{dims[1]}x{dims[2]} probe grid, {rays} rays/probe, "
                    f"~{sc.triangle_count // 1000}k-triangle interior hall, full-volume update "
                    "+ change detection + selection + slot assign + build + pack + temporal "
                    "delta, colour + visibility" if args.config == "c4" else
                    f"{args.config}: {dims} probes, {rays} rays/probe",
        "probes": vol.probe_count, "rays_per_probe": rays, "triangles": sc.triangle_count,
        "lights": len(sc.lights), "shadows": args.shadows,
        "l2": "per-frame working set (atlases, float state, planes) > 126 MB L2; no flush",
        "n_gpus_requested": world,
    }


def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist

    from paper_2103_05875_b200 import scene as S
    from paper_2103_05875_b200.sharding import SlabServer

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    dims, rays, scene_name = CONFIGS[args.config]
    sc = build_scene(scene_name)
    vol = S.volume_for(sc, dims)
    n = vol.probe_count
    server = SlabServer(vol, sc, rays_per_probe=rays, device=dev, rank=rank, world=world,
                        irradiance_scale=4.0 if scene_name == "hall" else 2.0,
                        shadows=args.shadows, graphs=not args.eager)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def frame_lights(f):
        return S.moving_light(sc, f).lights

    for f in range(args.warmup):
        server.tick(f, frame_lights(f))
    barrier()
    # ---- timed region: K full frames, inputs resident (scene, state), outputs on device
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    outs = (None, None)
    with ClockSampler(local) as clocks:
        barrier()
        start.record(stream)
        for k in range(args.steps):
            f = args.warmup + k
            outs = server.tick(f, frame_lights(f))
        server.join()  # the last frame's colour / visibility chains run on side streams
        end.record(stream)
        barrier()
    ms = start.elapsed_time(end) / args.steps
    # probes selected (= entries written) in the last timed frame, per kind:
    # the full-volume update means every probe, every frame
    selected = {k: (int(o.entry_count.item()) if o is not None else -1)
                for k, o in zip(("color", "visibility"), outs)}
    if world > 1:  # each kind's outputs live on its encoder rank
        t = torch.tensor([selected["color"], selected["visibility"]], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        selected = {"color": int(t[0]), "visibility": int(t[1])}
    ms_max = ms
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())

    # ---- end-to-end through the public API with host buffers -------------------------
    e2e = server.run_e2e(args.steps, args.warmup + args.steps, frame_lights)
    e2e_ms = e2e["ms_per_step"]
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
        # host I/O of the whole job: every rank's H2D, each encoder rank's D2H
        b = torch.tensor([e2e["h2d_bytes_per_step"], e2e["d2h_bytes_per_step"]], device=dev,
                         dtype=torch.int64)
        dist.all_reduce(b, op=dist.ReduceOp.SUM)
        e2e["h2d_bytes_per_step"], e2e["d2h_bytes_per_step"] = int(b[0]), int(b[1])

    e2e_enc = server.run_e2e_encoded(args.steps, args.warmup + 2 * args.steps + 40,
                                     frame_lights) if world == 1 else {}

    # ---- per-stage device times + launch count (untimed instrumented frames) ---------
    base = args.warmup + 2 * args.steps + 1
    stages = server.stage_times(3, base, frame_lights)
    rank_trace = [stages.get("trace_blend", 0.0)]
    if world > 1:
        t = torch.tensor([rank_trace[0]], device=dev, dtype=torch.float64)
        allt = torch.zeros(world, device=dev, dtype=torch.float64)
        dist.all_gather_into_tensor(allt, t)
        rank_trace = [round(v, 4) for v in allt.cpu().tolist()]
    slabs = getattr(server.impl, "ranges", None)
    launches_per_step, kernel_names = server.count_launches(base + 3, frame_lights)
    encode = server.encode_times() if world == 1 else {}
    passes = server.pass_times()  # last: re-running the blend advances the probe state

    peer_ranks = None
    if world > 1:
        pb = getattr(getattr(server.impl, "color", None), "_pb", None)
        if pb is not None:  # peers whose buffers this rank mapped with CUDA IPC
            peer_ranks = sum(1 for r, p in enumerate(pb.ptrs["flags"]) if r != rank and p)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    rays_total = n * rays
    # tcgen05 blend flops issued per frame: per probe and k-step of 8 rays, two
    # depth tiles (128 x 2P... per probe 128 texels x 2 moments x 8 rays x 2 flops)
    # and one colour tile (128 x 3 channels x 8) -- each issued twice (hi, lo)
    blend_flops = n * (rays // 8) * 2 * 8 * (3 * 2 * 128 * 2 + 2 * 128 * 3)
    # blend HBM bytes per probe: ray records read (16 B / ray), float state
    # read + written (64 x 3 irradiance + 256 x 2 moments, fp32), colour atlas
    # block (10 x 10 u32) and visibility block (18 x 18 half2) written
    blend_bytes = n * (16 * rays + 2 * 4 * (64 * 3 + 256 * 2) + 4 * 100 + 4 * 324)
    value = n / (ms_max / 1e3)
    peak, peak_kind = load_peaks()
    # roofline of the HBM-bound pack kernel (pack + temporal delta over the update atlas)
    pk = server.pack_delta_bytes()
    pack_ms = stages.get("color.pack_delta", 0) + stages.get("visibility.pack_delta", 0)
    achieved = pk["total"] / (pack_ms / 1e3) / 1e9 if pack_ms > 0 else None
    traffic = profile_traffic("pack_delta_kernel")
    trace_ms = stages.get("trace_blend", None)
    out = {
        "metric": METRIC,
        "value": round(value, 1),
        "unit": "probe updates/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_max, 4),
        "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None,
        "dtype": "f32+u32",
        "data": "synthetic",
        "config": make_config(args, sc, vol, world),
        "parallelism": f"z-slab x{world}",
        "run": {
            "slabs": ([[int(b), int(e)] for b, e in slabs] if slabs and world > 1 else None),
            "rank_trace_blend_ms": rank_trace if world > 1 else None,
            "launch": "eager" if args.eager else (
                "CUDA graphs (shadow maps on a side stream overlapping the previous blend; "
                "trace; blend; one chain per kind)"
                if getattr(getattr(server.impl, "updater", None), "_early", False)
                else "CUDA graphs (trace+blend, one chain per kind)"),
            "reserved_sms": getattr(getattr(server.impl, "updater", None), "reserve_sms", None),
            "exchange": (("peer memory (CUDA IPC over NVLink)"
                          if getattr(getattr(server.impl, "color", None), "peer", False)
                          else "NCCL") if world > 1 else None),
            "peer_ranks_mapped": peer_ranks,
            "encoder_ranks": (dict(zip(("color", "visibility"), server.impl.encoders))
                              if world > 1 else None),
        },
        "selected_last_frame": selected,
        "grays_per_s": round(rays_total / (ms_max / 1e3) / 1e9, 4),
        "frame_hz": round(1e3 / ms_max, 2),
        "stages_ms": {k: round(v, 4) for k, v in stages.items()},
        "passes_ms": {k: round(v, 4) for k, v in passes.items()},
        "packed_atlas_gbs": round(achieved, 1) if achieved else None,
        "roofline": {
            "bound": "hbm",
            "kernel": "pack_delta_kernel (colour + visibility)" if world == 1 else
                      "pack_delta_kernel (the kinds rank 0 encodes: colour)",
            "achieved": round(achieved, 1) if achieved else None,
            "peak": peak,
            "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind}, burst copy)",
            "unit": "GB/s",
            "frac": round(achieved / peak, 4) if achieved else None,
            "traffic": traffic,
            "algorithmic_bytes_per_launch": pk,
        },
        "roofline_trace": trace_roofline(passes["trace"], rays_total, world, clocks),
        "roofline_blend": {
            "bound": "tensor",
            "kernel": "blend_tc_kernel (tcgen05.mma kind::tf32, this rank's slab)",
            "ms": round(passes["blend"], 4),
            "achieved": round(blend_flops / world / (passes["blend"] / 1e3) / 1e12, 2),
            "peak": 1100.0,
            "unit": "TFLOP/s",
            "frac": round(blend_flops / world / (passes["blend"] / 1e3) / 1e12 / 1100.0, 4),
            "flops_per_launch": blend_flops // world,
            "hbm": {"algorithmic_bytes_per_launch": blend_bytes // world,
                    "achieved_gbs": round(blend_bytes / world / (passes["blend"] / 1e3) / 1e9, 1),
                    "peak": peak,
                    "frac": round(blend_bytes / world / (passes["blend"] / 1e3) / 1e9 / peak, 4),
                    "traffic": profile_traffic("tc::blend_tc_kernel"),
                    "note": "HBM is the blend's binding roofline (ray records + state "
                            "read-modify-write + atlas blocks)"},
            "note": "tf32 MMA flops issued (3xTF32, fp32-accurate): 3 MMAs (W_hi*B_hi + "
                    "W_hi*B_lo + W_lo*B_hi) per 128-texel depth tile, 2 for the colour tile "
                    "(W_hi rows 0-63, W_lo rows 64-127); peak = B200 dense tf32 "
                    "(B200_PROFILING.md); the useful fp32 work is 47 GFLOP/frame at C4",
        },
        "clocks": clocks.summary(),
        "e2e": {"value": round(n / (e2e_ms / 1e3), 1), "unit": "probe updates/s",
                "ms_per_step": round(e2e_ms, 4),
                "h2d_bytes_per_step": e2e["h2d_bytes_per_step"],
                "d2h_bytes_per_step": e2e["d2h_bytes_per_step"],
                "path": "ProbeStreamServer.tick via the C ABI; per-frame ray table + lights "
                        "H2D from pinned host memory, index entries + counts + SKIP maps D2H"},
        "encode_lpf1": {"note": "§8(f)1 GPU LPF1 encoder (bit-exact with codec.encode_frame) on "
                                "this frame's planes; not inside the step", **encode},
        "e2e_encoded": ({"value": round(n / (e2e_enc["ms_per_step"] / 1e3), 1),
                         "unit": "probe updates/s", **{k: (round(v, 4) if isinstance(v, float) else v)
                                                        for k, v in e2e_enc.items()},
                         "path": "as e2e, plus GPU LPF1 encoding (§8(f)1) + index buffer (§8(f)4) "
                                 "and D2H of the wire bytes each frame"} if e2e_enc else None),
        "gpu_launches": launches_per_step * args.steps,
        "gpu_launches_per_step": launches_per_step,
        "kernels": kernel_names,
    }
    if world == 1:
        # the reference-facing drop-in (numpy in / numpy out), not in the step
        out["dropin_numpy"] = dropin_numpy(dims)
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(sc, vol, rays, args.cpu_sample, args.shadows)
        parts = out["cpu_baseline"]["detail"].get("stages_parts_s", {})
        for kind in ("color", "visibility"):
            if kind in parts and kind in out["dropin_numpy"]:
                ref_ms = 1e3 * sum(v for k, v in parts[kind].items() if k != "delta")
                out["dropin_numpy"][kind]["reference_ms"] = round(ref_ms, 1)
                out["dropin_numpy"][kind]["speedup"] = round(
                    ref_ms / out["dropin_numpy"][kind]["ms"], 1)
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _reference_package():
    """The reference ``probestream`` from $PROBESTREAM_REF or baseline/_ref
    (the offline install that travels to the GPU box), or None."""
    import importlib

    for c in (os.environ.get("PROBESTREAM_REF"), str(ROOT / "baseline" / "_ref")):
        if c and (Path(c) / "probestream" / "__init__.py").exists():
            if c not in sys.path:
                sys.path.insert(0, c)
            try:
                mod = importlib.import_module("probestream")
                importlib.import_module("probestream.volume")
                return mod
            except Exception:
                return None
    return None


def dropin_numpy(dims, reps: int = 3) -> dict:
    """The INTEGRATION.md §1 swap as a reference caller sees it: numpy atlases
    in the reference's own ProbeVolume / ProbeAtlas objects (baseline/_ref;
    this package's mirrors when absent) through this package's
    detect_changed -> select_for_client -> build_update_atlas -> pack_texels,
    every probe changed, at the bench volume.  Wall time per kind (best of
    ``reps``), host <-> device staging of the numpy arrays included."""
    import numpy as np
    import torch

    from paper_2103_05875_b200 import packing, selection
    from paper_2103_05875_b200 import volume as V_ours

    ref = _reference_package()
    V = ref.volume if ref is not None else V_ours
    n = dims[0] * dims[1] * dims[2]
    vol = V.ProbeVolume(tuple(dims))
    rng = np.random.default_rng(0)
    out = {"objects": "reference probestream (baseline/_ref)" if ref is not None
           else "package mirrors (reference not importable)", "probes": n}
    for K in (V.AtlasKind.COLOR, V.AtlasKind.VISIBILITY):
        a = V.ProbeAtlas(K, n)
        dt = a.texels.dtype
        cur = rng.integers(0, 2**16, size=a.texels.shape, dtype=dt)
        rendered, last = V.ProbeAtlas(K, n, a.probes_per_row, cur), V.ProbeAtlas(
            K, n, a.probes_per_row, cur ^ dt.type(1))
        best = None
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            changed = selection.detect_changed(rendered, last, vol)
            sel = selection.select_for_client(changed, changed, vol, np.zeros(n, np.int64), 1)
            layout = packing.UpdateAtlasLayout(n, K.core_side)
            upd, entries = packing.build_update_atlas(sel, layout, rendered)
            planes = packing.pack_texels(upd, K)
            t = time.perf_counter() - t0
            best = t if best is None else min(best, t)
        assert len(entries) == n and isinstance(planes.data, np.ndarray)
        out[K.value] = {"ms": round(best * 1e3, 2), "selected": len(sel)}
    return out


def cpu_baseline(sc, vol, rays, sample, shadows="map"):
    """One sampled step of the reference's CPU path (oracle/cpu_frame.py)."""
    from oracle import cpu_frame

    cpu_frame.warm_up(sc)
    r = cpu_frame.time_frame(sc, vol, rays, sample_probes=sample, shadows=shadows)
    return {
        "value": round(r["probe_updates_per_s"], 4),
        "unit": "probe updates/s",
        "cores": r["threads"],
        "kind": "port",
        "sampled": True,
        "sample": sample_text(r, rays),
        "wall_s": round(r["wall_s"], 3),
        "detail": {k: (round(v, 6) if isinstance(v, float) else v) for k, v in r.items()},
    }


def sample_text(r, rays):
    return (f"{r['sample_probes']} probes x {rays} rays traced by the oracle's C restatement of "
            f"the reference brute-force raycast (float64, OpenMP on {r['threads']} threads) + numpy "
            f"DDGI blend; {r['map_sample_texels']} shadow-map texels by the same query; stages 3-4 "
            f"on {r['stage_probes']} probes by the {r['stages_impl']} functions (detect_changed, "
            f"select_for_client, build_update_atlas, pack_texels; temporal delta by the numpy "
            f"port). value = probes / (probes x measured per-probe cost of each part + measured "
            f"per-texel shadow-map cost x map texels)")


def run_reference(args, rank, world, local):
    """The reference's CPU path on the host cores (see oracle/cpu_frame.py):
    every step is a measured, bounded sample of the frame; ms_per_step is the
    wall time those steps took, value the per-probe rate they measured."""
    if rank != 0:
        return
    from paper_2103_05875_b200 import scene as S
    from oracle import cpu_frame

    dims, rays, scene_name = CONFIGS[args.config]
    sc = build_scene(scene_name)
    vol = S.volume_for(sc, dims)
    cpu_frame.warm_up(sc)
    for w in range(min(args.warmup, 1)):
        cpu_frame.time_frame(sc, vol, rays, sample_probes=1, frame=w, shadows=args.shadows,
                             stage_probes=dims[0] * dims[1], map_sample=64)
    steps = []
    w0 = time.perf_counter()
    for k in range(args.steps):
        steps.append(cpu_frame.time_frame(sc, vol, rays, sample_probes=args.cpu_sample, frame=k,
                                          rng_seed=k, shadows=args.shadows))
    wall = time.perf_counter() - w0
    per_probe = sum(1.0 / r["probe_updates_per_s"] for r in steps) / len(steps)
    value = 1.0 / per_probe
    r0 = steps[0]
    out = {
        "metric": METRIC, "value": round(value, 4), "unit": "probe updates/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(wall / args.steps * 1e3, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64+u32", "data": "synthetic",
        "config": make_config(args, sc, vol, world),
        "parallelism": f"host CPU, {os.cpu_count()} threads (rank 0 only)",
        "sampled": True,
        "note": "ms_per_step is the measured wall time of each sampled step; value is the "
                "whole-volume rate the step's measured per-probe / per-texel costs give "
                "(projected frame time per step in detail.frame_s)",
        "grays_per_s": round(vol.probe_count * rays * value / vol.probe_count / 1e9, 12),
        "selected_last_frame": r0["selected"],
        "detail": {"frame_s": [round(r["frame_s"], 1) for r in steps],
                   "wall_s": [round(r["wall_s"], 3) for r in steps],
                   "trace_blend_s_per_probe": [round(r["trace_blend_s_per_probe"], 5) for r in steps],
                   "stages_s": [round(r["stages_s"], 3) for r in steps],
                   "stages_parts_s": r0["stages_parts_s"],
                   "shadow_map_frame_s": [round(r["shadow_map_frame_s"], 1) for r in steps]},
        "cpu_baseline": {"value": round(value, 4), "unit": "probe updates/s",
                         "cores": os.cpu_count(), "kind": "port", "sampled": True,
                         "sample": sample_text(r0, rays)},
        "e2e": {"value": round(value, 4), "unit": "probe updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    # keep rank 0's stdout to the single JSON line: NCCL's debug output
    # (version banner, communicator lines at NCCL_DEBUG=INFO) goes to stderr
    if not os.environ.get("NCCL_DEBUG_FILE"):
        os.environ["NCCL_DEBUG_FILE"] = "/dev/stderr"
    # NCCL_DEBUG=VERSION prints its banner to stdout whatever NCCL_DEBUG_FILE
    # says: log the version to stderr instead (INFO / TRACE lines go to the file)
    if os.environ.get("NCCL_DEBUG", "").upper() == "VERSION":
        os.environ["NCCL_DEBUG"] = "WARN"
        try:
            import torch

            log("NCCL version", ".".join(map(str, torch.cuda.nccl.version())))
        except Exception:
            pass
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--cpu-sample", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shadows", default="map", choices=["map", "rays", "none"])
    ap.add_argument("--eager", action="store_true",
                    help="issue every kernel from the host instead of replaying CUDA graphs")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (timing rules)")
        args.warmup = 3
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world, local)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
