#!/usr/bin/env python
"""Time the GPU LPF1 encoder on C4-sized update atlases (key + P frames)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    from paper_2103_05875_b200.codec import encode_frame_device

    rng = np.random.default_rng(0)
    res = {}
    for name, shape, dt, hi in (("color", (3, 2896, 2904), torch.int16, 1024),
                                ("visibility", (3, 5792, 7744), torch.uint8, 256)):
        base = torch.randint(0, hi, shape, device="cuda", dtype=torch.int32)
        cur = base.to(torch.uint8) if dt == torch.uint8 else base.to(torch.int16).view(torch.uint16)
        prev = cur.clone()
        flat = prev.view(-1) if dt == torch.uint8 else prev.view(torch.int16).view(-1)
        flat[::97] ^= 1
        for tag, ref in (("key", None), ("p", prev)):
            encode_frame_device(cur, ref, 1, 0)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(3):
                out, ln = encode_frame_device(cur, ref, 1, 0)
            b.record()
            torch.cuda.synchronize()
            res[f"{name}.{tag}"] = {"ms": round(a.elapsed_time(b) / 3, 3), "bytes": int(ln.item())}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
