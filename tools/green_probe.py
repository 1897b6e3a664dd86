#!/usr/bin/env python
"""Feasibility probe (tuning only): can runtime-API kernels (torch, libprobestream)
run on a stream of a CUDA green context confined to K SMs?"""
import json
import sys
import time

import torch
from cuda.bindings import driver as d


def check(r):
    err = r[0] if isinstance(r, tuple) else r
    if err != d.CUresult.CUDA_SUCCESS:
        raise RuntimeError(str(err))
    return r[1:] if isinstance(r, tuple) and len(r) > 2 else (r[1] if isinstance(r, tuple) and len(r) == 2 else None)


def green_stream(k):
    torch.cuda.init()
    torch.zeros(1, device="cuda")
    check(d.cuInit(0))
    dev = check(d.cuDeviceGet(0))
    res = check(d.cuDeviceGetDevResource(dev, d.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))
    print("total SMs", res.sm.smCount)
    groups, nb, rem = d.cuDevSmResourceSplitByCount(1, res, 0, k)[1:]
    print("group SMs", groups[0].sm.smCount, "remaining", rem.sm.smCount)
    desc = check(d.cuDevResourceGenerateDesc([groups[0]], 1))
    g = check(d.cuGreenCtxCreate(desc, dev, d.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM))
    st = check(d.cuGreenCtxStreamCreate(g, d.CUstream_flags.CU_STREAM_NON_BLOCKING, 0))
    return g, st


def bench(stream, a, b, reps=20):
    with torch.cuda.stream(stream):
        for _ in range(3):
            a @ b
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            a @ b
        e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    g, st = green_stream(k)
    ext = torch.cuda.ExternalStream(int(st))
    a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    t_full = bench(torch.cuda.current_stream(), a, b)
    t_green = bench(ext, a, b)
    x = torch.empty(1 << 28, dtype=torch.float32, device="cuda")
    def copy_ms(s):
        with torch.cuda.stream(s):
            y = x.clone()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); y.copy_(x); e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)
    c_full, c_green = copy_ms(torch.cuda.current_stream()), copy_ms(ext)
    print(json.dumps({"k": k, "gemm_full_ms": t_full, "gemm_green_ms": t_green,
                      "copy_full_ms": c_full, "copy_green_ms": c_green,
                      "copy_green_gbs": 2 * x.numel() * 4 / c_green / 1e6}))
    # graph capture on the green stream
    try:
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.stream(ext):
            with torch.cuda.graph(gr, stream=ext):
                y = a @ b
        torch.cuda.synchronize()
        with torch.cuda.stream(ext):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); gr.replay(); e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"graph_on_green_ms": e0.elapsed_time(e1)}))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); gr.replay(); e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"graph_green_captured_replayed_on_default_ms": e0.elapsed_time(e1)}))
    except Exception as ex:  # noqa: BLE001
        print("graph failed:", ex)


if __name__ == "__main__":
    main()
