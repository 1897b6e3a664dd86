// Guard-band source index shared by the blend kernels.
#pragma once

namespace ps {

// guard band rule (packing.py:180-196): block (r, c) -> core index
__device__ __forceinline__ int guard_source(int r, int c, int side) {
    const int n = side - 2;
    const bool top = r == 0, bot = r == side - 1, left = c == 0, right = c == side - 1;
    int rr = r, cc = c;
    if ((top || bot) && (left || right)) {
        rr = top ? n : 1;
        cc = left ? n : 1;
    } else if (top || bot) {
        rr = top ? 1 : n;
        cc = side - 1 - c;
    } else if (left || right) {
        rr = side - 1 - r;
        cc = left ? 1 : n;
    }
    return (rr - 1) * n + (cc - 1);
}

}  // namespace ps
