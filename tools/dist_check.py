#!/usr/bin/env python
"""Multi-GPU parity: run the slab-sharded frame on every rank and, on rank 0,
the single-GPU pipeline for the same frames; the encoder rank's outputs must
be bit-identical.  Launch with
    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/dist_check.py [--config c1]
"""

import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--frames", type=int, default=3)
    ap.add_argument("--graphs", action="store_true", help="sharded side replays CUDA graphs")
    ap.add_argument("--gop", type=int, default=30)
    ap.add_argument("--nccl", action="store_true", help="NCCL exchanges instead of peer memory")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import bench
    from paper_2103_05875_b200 import scene as S
    from paper_2103_05875_b200.distributed import DistributedFrame
    from paper_2103_05875_b200.server import ProbeStreamServer

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    dims, rays, scene_name = bench.CONFIGS[args.config]
    sc = bench.build_scene(scene_name)
    vol = S.volume_for(sc, dims)
    kw = dict(irradiance_scale=2.0, shadows="map", shadow_map_size=128, gop_length=args.gop)
    frame = DistributedFrame(vol, sc, rays, dev, rank, world, graphs=args.graphs, peer=not args.nccl,
                             **kw)
    # each kind is checked on its encoder rank (colour on rank 0, visibility on
    # rank 1 by default), against a single-GPU server on that rank
    enc = frame.encoders
    single = ProbeStreamServer(vol, sc, rays, device=dev, **kw) if rank in enc else None
    ok = True
    for f in range(args.frames):
        lights = S.moving_light(sc, f).lights
        outs = frame.tick(f, lights)
        if single is not None:
            ref = single.tick(f, lights)
            torch.cuda.synchronize()
            for name, a, b, e in zip(("color", "visibility"), outs, ref, enc):
                if e != rank:
                    assert a is None, "outputs on a rank that does not encode the kind"
                    continue
                n = int(b.entry_count.item())
                same = (int(a.entry_count.item()) == n
                        and torch.equal(a.entries[:n], b.entries[:n])
                        and torch.equal(a.planes.view(torch.uint8), b.planes.view(torch.uint8))
                        and torch.equal(a.skip, b.skip)
                        and (b.key or torch.equal(a.residual.view(torch.uint8),
                                                  b.residual.view(torch.uint8))))
                print(f"frame {f} {name} (rank {rank}): entries {n} bit-identical={same}",
                      flush=True)
                ok &= same
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("DIST OK" if flag.item() else "DIST MISMATCH", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if flag.item() else 1)


if __name__ == "__main__":
    main()
