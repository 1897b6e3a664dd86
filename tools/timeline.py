#!/usr/bin/env python
"""Kernel timeline of the sharded frame (torch profiler, CUDA activity) plus the
host issue time per tick; one JSON per rank in gpurun_out/.  Launch with
    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/timeline.py [--config c4]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--frames", type=int, default=6)
    ap.add_argument("--eager", action="store_true")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    from torch.profiler import ProfilerActivity, profile

    import bench
    from paper_2103_05875_b200 import scene as S
    from paper_2103_05875_b200.sharding import SlabServer

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    dims, rays, name = bench.CONFIGS[args.config]
    sc = bench.build_scene(name)
    vol = S.volume_for(sc, dims)
    srv = SlabServer(vol, sc, rays_per_probe=rays, device=dev, rank=rank, world=world,
                     irradiance_scale=4.0, graphs=not args.eager)
    for f in range(4):
        srv.tick(f, S.moving_light(sc, f).lights)
    srv.join()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    host = []
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for k in range(args.frames):
            t0 = time.perf_counter()
            srv.tick(4 + k, S.moving_light(sc, 4 + k).lights)
            host.append(time.perf_counter() - t0)
        srv.join()
        torch.cuda.synchronize()
    evs = []
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            evs.append({"name": e.name[:80], "start_us": e.time_range.start,
                        "dur_us": e.time_range.end - e.time_range.start,
                        "stream": getattr(e, "device_resource_id", None)})
    evs.sort(key=lambda x: x["start_us"])
    out = Path("gpurun_out") / f"timeline_n{world}_r{rank}{'_eager' if args.eager else ''}.json"
    out.parent.mkdir(exist_ok=True)
    json.dump({"host_ms_per_tick": [1e3 * h for h in host], "kernels": evs}, open(out, "w"))
    if rank == 0:
        print(f"host issue ms/tick: {[round(1e3 * h, 3) for h in host]}")
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
