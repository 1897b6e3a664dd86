#!/usr/bin/env python
"""Compare the probe-ray records of one frame between two tracer variants
(tuning only): run once with --save under variant A, then with --compare
under variant B (PS_TRACE_VARIANT).  Prints how many rays differ in hit
distance / radiance and the largest differences."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--save")
    ap.add_argument("--compare")
    ap.add_argument("--frame", type=int, default=2)
    args = ap.parse_args()
    import os

    import torch

    import bench
    from paper_2103_05875_b200 import scene as S
    from paper_2103_05875_b200.probes import ProbeUpdater

    dims, rays, name = bench.CONFIGS[args.config]
    sc = bench.build_scene(name)
    vol = S.volume_for(sc, dims)
    upd = ProbeUpdater(vol, sc.device(), rays_per_probe=rays, shadows="map")
    upd.update(args.frame, S.moving_light(sc, args.frame).lights)
    torch.cuda.synchronize()
    rec = upd.records
    if args.save:
        torch.save(rec.cpu(), args.save)
        print(json.dumps({"saved": args.save, "rays": rec.shape[0]}))
        return
    ref = torch.load(args.compare).to(rec.device)
    diff = (rec != ref).any(dim=1)
    n = int(diff.sum())
    out = {"variant": os.environ.get("PS_TRACE_VARIANT", "default"), "rays": rec.shape[0],
           "differing_rays": n, "frac": n / rec.shape[0]}
    if n:
        dd = (rec[:, 3] - ref[:, 3]).abs()
        out["max_depth_diff"] = float(dd.max())
        out["max_rgb_diff"] = float((rec[:, :3] - ref[:, :3]).abs().max())
        out["depth_diff_gt_1e-3"] = int((dd > 1e-3).sum())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
