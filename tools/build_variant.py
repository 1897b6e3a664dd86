#!/usr/bin/env python
"""Tuning builds: relink libprobestream with one source recompiled under extra
nvcc flags, as a separate library selected at run time with PROBESTREAM_LIB.

    python tools/build_variant.py NAME SOURCE.cu -D... [-D...]
    PROBESTREAM_LIB=paper_2103_05875_b200/libprobestream_NAME.so python tools/trace_bench.py
"""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2103_05875_b200 import build_native as B  # noqa: E402


def main():
    name, src, flags = sys.argv[1], sys.argv[2], sys.argv[3:]
    B.build()
    objs = sorted(B.BUILD.glob("*.o"))
    out_dir = B.BUILD / f"variant_{name}"
    out_dir.mkdir(exist_ok=True)
    srcp = B.CSRC / src
    obj = out_dir / (srcp.name + ".o")
    cmd = [B._nvcc(), *B.ARCH, *B.NVCC_FLAGS, *flags, f"-I{B.INCLUDE}", f"-I{B.CSRC}", "-c",
           str(srcp), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode:
        sys.exit(res.stderr[-3000:])
    objs = [obj if o.name == srcp.name + ".o" else o for o in objs]
    lib = B.PKG / f"libprobestream_{name}.so"
    res = subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-o", str(lib), *map(str, objs)],
                         capture_output=True, text=True)
    if res.returncode:
        sys.exit(res.stderr[-3000:])
    print(lib)


if __name__ == "__main__":
    main()
