// Shared helpers for the probestream CUDA library (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>

#include "probestream.h"

#ifndef __CUDA_ARCH__
#else
#if __CUDA_ARCH__ < 1000
#error "probestream kernels target sm_100a only"
#endif
#endif

namespace ps {

// error carrying a status code; converted to (status, thread-local message)
// at the C boundary by PS_ABI_BEGIN/END.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string &msg);

[[noreturn]] inline void fail(int code, const std::string &msg) { throw Error(code, msg); }

inline void check_cuda(cudaError_t e, const char *what) {
    if (e != cudaSuccess) {
        fail(PS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    }
}

inline void check_launch(const char *what) { check_cuda(cudaGetLastError(), what); }

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

inline int sm_count() {
    static int cached = 0;
    if (!cached) {
        int dev = 0;
        check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
        check_cuda(cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev),
                   "cudaDeviceGetAttribute");
    }
    return cached;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// carve aligned sub-buffers out of a caller workspace
struct Carver {
    char *base;
    size_t cap, off = 0;
    Carver(void *b, size_t c) : base(static_cast<char *>(b)), cap(c) {}
    template <class T>
    T *take(size_t n) {
        off = (off + 255) & ~size_t(255);
        T *p = reinterpret_cast<T *>(base ? base + off : nullptr);
        off += n * sizeof(T);
        return p;
    }
    void check() const {
        if (off > cap) fail(PS_ERR_WORKSPACE, "workspace too small");
    }
};


#ifdef __CUDACC__
// Division by a run-time constant d >= 1 for dividends n < 2^31 as a
// multiply-high, an add and a shift (Granlund-Montgomery): s = ceil(log2 d),
// m = floor(2^32 (2^s - d) / d) + 1, n / d = (umulhi(n, m) + n) >> s.  Set up
// once per thread; replaces the ~15-instruction reciprocal sequence (or the
// 64-bit software division) of every per-ray / per-entry index split.
struct FastDiv {
    uint32_t d, m, s;
    __device__ __forceinline__ explicit FastDiv(uint32_t d_) : d(d_) {
        s = 0;
        while ((1ull << s) < d) ++s;
        m = uint32_t((((1ull << s) - d) << 32) / d + 1);
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        return (__umulhi(n, m) + n) >> s;
    }
};

// (row, column) origin of block `id` in a grid of `per_row` blocks of `side`
// texels: ids and grids are < 2^31, so one 32-bit division instead of a
// 64-bit software divide and modulo
__device__ __forceinline__ void block_origin(int64_t id, int64_t per_row, int side, int64_t &y,
                                             int64_t &x) {
    const uint32_t i = uint32_t(id), n = uint32_t(per_row), r = i / n;
    y = int64_t(r) * side;
    x = int64_t(i - r * n) * side;
}

// One warp moves probe block (y0, x0) -- SIDE x SIDE words of a rendered
// atlas, row stride src_w -- handing each interior (core) word to `core(r, c,
// v)` and, if last_sent is set, committing the whole block there.  Every load
// of the block is issued before the first store (the source is read-only for
// the kernel), so a warp keeps SIDE^2 / 32 loads in flight instead of one.
template <int SIDE, class CoreStore>
__device__ __forceinline__ void warp_copy_block(const uint32_t *__restrict__ src, int64_t src_w,
                                                int64_t y0, int64_t x0, int lane,
                                                uint32_t *last_sent, CoreStore core) {
    constexpr int WORDS = SIDE * SIDE, CORE = SIDE - 2, N = (WORDS + 31) / 32;
    // one 64-bit block base, 32-bit offsets inside the block (a block spans
    // SIDE rows, far below 2^31 words): fewer live 64-bit addresses
    const int w32 = int(src_w);
    const uint32_t *__restrict__ sb = src + y0 * src_w + x0;
    uint32_t v[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
        const int k = lane + 32 * j;
        if (k < WORDS) v[j] = __ldg(sb + (k / SIDE) * w32 + k % SIDE);
    }
#pragma unroll
    for (int j = 0; j < N; ++j) {
        const int k = lane + 32 * j;
        if (k < WORDS) {
            const int r = k / SIDE, c = k % SIDE;
            if (r >= 1 && r <= CORE && c >= 1 && c <= CORE) core(r - 1, c - 1, v[j]);
            if (last_sent) last_sent[(y0 * src_w + x0) + (r * w32 + c)] = v[j];
        }
    }
}
#endif

}  // namespace ps

#define PS_ABI_BEGIN try {
#define PS_ABI_END                                  \
    return PS_OK;                                   \
    }                                               \
    catch (const ps::Error &e) {                    \
        ps::set_last_error(e.what());               \
        return e.code;                              \
    }                                               \
    catch (const std::exception &e) {               \
        ps::set_last_error(e.what());               \
        return PS_ERR_CUDA;                         \
    }
