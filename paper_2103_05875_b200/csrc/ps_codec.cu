// §8(f) row 1: bit-exact LPF1 frame encoding on the GPU (codec.py:76-201,
// 207-292, 335-366; varint.py:16-84).
//
// The reference encodes 16x16 blocks one by one in Python (2.5 s / 12.8 s per
// colour / visibility I-frame at 32x16x32).  Here every block is one warp:
//
//   size pass   SKIP test against the reference block (P-frames); otherwise
//               the raw byte stream and, when a predictor exists (reference
//               block, or the left neighbour in a key frame), the zig-zag
//               LEB128 residual stream are built in shared memory and their
//               zero-run-length encodings are sized with warp scans; DELTA
//               wins only if strictly shorter (ties go to RAW, codec.py:283).
//   scan        exclusive prefix sum of the block sizes (payload offsets).
//   emit pass   the chosen stream is rebuilt and written at its offset:
//               mode byte, LEB128 length, tokens -- literal bytes land at
//               offsets given by per-segment prefix sums, so stores from a
//               warp are contiguous.
//   container   LPF1 header (<4sBIIHHBBI), then CRC32 of header+payload in
//               4 KB chunks combined with GF(2) polynomial shifts (the zlib
//               crc32_combine algorithm), appended little-endian.
//
// Entropy tokens (codec.py:76-103): a maximal zero run of >= 2 bytes becomes
// uvarint(len << 1 | 1); every other stretch is a literal segment
// uvarint(len << 1) + bytes.  A zero byte belongs to such a run iff a
// neighbouring byte is also zero.
#include <cub/device/device_scan.cuh>
#include <cstdlib>
#include <cuda_runtime.h>

#include "ps_common.cuh"

namespace ps {
namespace {

constexpr int WARPS = 4;           // warps (blocks) per CTA
constexpr int MAXS = 768;          // max stream bytes per block (256 x 3-byte varints)
constexpr int HDR = 23;            // LPF1 header bytes
constexpr uint32_t CRC_POLY = 0xEDB88320u;
constexpr int CRC_CHUNK = 4096;

struct WarpScratch {
    uint8_t s[MAXS];               // stream bytes
    uint8_t e[MAXS];               // zero byte inside a run of >= 2
    uint16_t seg[MAXS];            // segment index of each byte
    uint16_t start[MAXS + 1];      // segment start positions (+ sentinel n)
    uint16_t off[MAXS + 1];        // segment output offsets
};

__device__ __forceinline__ int vlen(uint32_t v) { return v < 128u ? 1 : (v < 16384u ? 2 : (v < 2097152u ? 3 : 4)); }

__device__ __forceinline__ int put_varint(uint8_t *dst, uint32_t v) {
    int k = 0;
    while (true) {
        const uint32_t b = v & 0x7Fu;
        v >>= 7;
        if (v) {
            dst[k++] = uint8_t(b | 0x80u);
        } else {
            dst[k++] = uint8_t(b);
            return k;
        }
    }
}

// warp-wide exclusive scan of v with a running carry; returns exclusive prefix
__device__ __forceinline__ uint32_t warp_excl(uint32_t v, uint32_t &carry, int lane) {
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    const uint32_t ex = carry + inc - v;
    carry += __shfl_sync(0xffffffffu, inc, 31);
    return ex;
}

// Zero-run-length encoding of ws.s[0..n) by one warp.  Returns the encoded
// length; writes the tokens to `out` when it is non-null.
__device__ int warp_entropy(WarpScratch &ws, int n, uint8_t *out, int lane) {
    if (n == 0) return 0;
    // pass 1: run-eligible zeros, segment starts and indices
    uint32_t kcarry = 0;
    int e_last = 0;  // e of the previous tile's last byte
    for (int t0 = 0; t0 < n; t0 += 32) {
        const int i = t0 + lane;
        const bool valid = i < n;
        const bool z = valid && ws.s[i] == 0;
        const bool zp = valid && i > 0 && ws.s[i - 1] == 0;
        const bool zn = valid && i + 1 < n && ws.s[i + 1] == 0;
        const int e = (z && (zp || zn)) ? 1 : 0;
        int ep = __shfl_up_sync(0xffffffffu, e, 1);
        if (lane == 0) ep = e_last;
        const bool st = valid && (i == 0 || e != ep);
        const unsigned m = __ballot_sync(0xffffffffu, st);
        const unsigned lt = (1u << lane) - 1u;
        if (valid) {
            ws.e[i] = uint8_t(e);
            ws.seg[i] = uint16_t(kcarry + __popc(m & (lt | (1u << lane))) - 1);
            if (st) ws.start[kcarry + __popc(m & lt)] = uint16_t(i);
        }
        kcarry += __popc(m);
        e_last = __shfl_sync(0xffffffffu, e, 31);
    }
    const int K = int(kcarry);
    if (lane == 0) ws.start[K] = uint16_t(n);
    __syncwarp();
    // pass 2: segment sizes and output offsets
    uint32_t ocarry = 0;
    for (int k0 = 0; k0 < K; k0 += 32) {
        const int k = k0 + lane;
        uint32_t sz = 0;
        if (k < K) {
            const uint32_t L = uint32_t(ws.start[k + 1] - ws.start[k]);
            sz = ws.e[ws.start[k]] ? uint32_t(vlen((L << 1) | 1u)) : uint32_t(vlen(L << 1)) + L;
        }
        const uint32_t ex = warp_excl(sz, ocarry, lane);
        if (k < K) ws.off[k] = uint16_t(ex);
    }
    const int total = int(ocarry);
    if (!out) return total;
    __syncwarp();
    // pass 3: token headers
    for (int k = lane; k < K; k += 32) {
        const uint32_t L = uint32_t(ws.start[k + 1] - ws.start[k]);
        const bool zr = ws.e[ws.start[k]] != 0;
        put_varint(out + ws.off[k], zr ? ((L << 1) | 1u) : (L << 1));
    }
    // pass 4: literal bytes
    for (int i = lane; i < n; i += 32) {
        if (ws.e[i]) continue;
        const int k = ws.seg[i];
        const uint32_t L = uint32_t(ws.start[k + 1] - ws.start[k]);
        out[ws.off[k] + vlen(L << 1) + (i - ws.start[k])] = ws.s[i];
    }
    return total;
}

struct EncArgs {
    const uint8_t *cur;
    const uint8_t *ref;  // null: key frame
    int eb;              // element bytes (2 colour, 1 visibility)
    int h, w, nby, nbx;
    int64_t nblocks;
    uint32_t *sizes;     // bytes of each block in the payload
    uint32_t *lens;      // entropy payload length (non-SKIP)
    uint8_t *modes;
    const uint64_t *offsets;
    uint8_t *out;        // frame buffer (header at 0, payload at HDR)
};

__device__ __forceinline__ uint32_t load_elem(const uint8_t *plane, int w, int y, int x, int eb) {
    const int64_t idx = int64_t(y) * w + x;
    return eb == 2 ? uint32_t(reinterpret_cast<const uint16_t *>(plane)[idx]) : uint32_t(plane[idx]);
}

// builds the RAW (mode 2) or residual (mode 1) stream of block b into ws.s
__device__ int build_stream(const EncArgs &a, WarpScratch &ws, int mode, int pl, int y0, int x0,
                            int bh, int bw, bool intra, int lane) {
    const int64_t psz = int64_t(a.h) * a.w * a.eb;
    const uint8_t *cur = a.cur + pl * psz;
    const int m = bh * bw;
    if (mode == 2) {
        for (int j = lane; j < m; j += 32) {
            const uint32_t v = load_elem(cur, a.w, y0 + j / bw, x0 + j % bw, a.eb);
            ws.s[j * a.eb] = uint8_t(v);
            if (a.eb == 2) ws.s[j * 2 + 1] = uint8_t(v >> 8);
        }
        __syncwarp();
        return m * a.eb;
    }
    const uint8_t *pred = intra ? cur : a.ref + pl * psz;
    const int px = intra ? x0 - 16 : x0;
    uint32_t carry = 0;
    for (int j0 = 0; j0 < m; j0 += 32) {
        const int j = j0 + lane;
        uint32_t z = 0;
        int c = 0;
        if (j < m) {
            const int y = y0 + j / bw, xo = j % bw;
            const uint32_t cv = load_elem(cur, a.w, y, x0 + xo, a.eb);
            const uint32_t pv = load_elem(pred, a.w, y, px + xo, a.eb);
            int32_t r;
            if (a.eb == 2) r = int32_t(int16_t(uint16_t(cv - pv)));
            else r = int32_t(int8_t(uint8_t(cv - pv)));
            z = (uint32_t(r) << 1) ^ uint32_t(r >> 31);  // zig-zag
            c = vlen(z);
        }
        const uint32_t pos = warp_excl(uint32_t(c), carry, lane);
        if (j < m) put_varint(ws.s + pos, z);
    }
    __syncwarp();
    return int(carry);
}

__device__ __forceinline__ void block_coords(const EncArgs &a, int64_t b, int &pl, int &y0, int &x0,
                                             int &bh, int &bw) {
    const int64_t per = int64_t(a.nby) * a.nbx;
    pl = int(b / per);
    const int64_t r = b - pl * per;
    const int by = int(r / a.nbx), bx = int(r - int64_t(by) * a.nbx);
    y0 = by * 16;
    x0 = bx * 16;
    bh = min(16, a.h - y0);
    bw = min(16, a.w - x0);
}

__global__ void __launch_bounds__(WARPS * 32) encode_size_kernel(EncArgs a) {
    __shared__ WarpScratch scratch[WARPS];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    WarpScratch &ws = scratch[wid];
    for (int64_t b = int64_t(blockIdx.x) * WARPS + wid; b < a.nblocks; b += int64_t(gridDim.x) * WARPS) {
        int pl, y0, x0, bh, bw;
        block_coords(a, b, pl, y0, x0, bh, bw);
        const int64_t psz = int64_t(a.h) * a.w * a.eb;
        bool has_pred = false, intra = false;
        if (a.ref) {
            // SKIP iff bit-identical to the reference block (codec.py:264-272)
            bool diff = false;
            for (int j = lane; j < bh * bw; j += 32) {
                const int y = y0 + j / bw, x = x0 + j % bw;
                diff |= load_elem(a.cur + pl * psz, a.w, y, x, a.eb) !=
                        load_elem(a.ref + pl * psz, a.w, y, x, a.eb);
            }
            if (!__any_sync(0xffffffffu, diff)) {
                if (lane == 0) {
                    a.sizes[b] = 1;
                    a.modes[b] = 0;
                    a.lens[b] = 0;
                }
                continue;
            }
            has_pred = true;
        } else if (x0 >= 16) {
            has_pred = intra = true;
        }
        int n = build_stream(a, ws, 2, pl, y0, x0, bh, bw, intra, lane);
        const int raw_len = warp_entropy(ws, n, nullptr, lane);
        __syncwarp();
        int mode = 2, len = raw_len;
        if (has_pred) {
            n = build_stream(a, ws, 1, pl, y0, x0, bh, bw, intra, lane);
            const int delta_len = warp_entropy(ws, n, nullptr, lane);
            __syncwarp();
            if (delta_len < raw_len) {
                mode = 1;
                len = delta_len;
            }
        }
        if (lane == 0) {
            a.sizes[b] = uint32_t(1 + vlen(uint32_t(len)) + len);
            a.modes[b] = uint8_t(mode);
            a.lens[b] = uint32_t(len);
        }
    }
}

// ---- size pass, one thread per block --------------------------------------------------
// The entropy size of a stream only needs its zero-run structure: a maximal
// run of >= 2 zero bytes costs vlen(2L+1) bytes, every literal stretch of L
// bytes vlen(2L) + L, and vlen(2L[+1]) = 1 + (L >= 64) for the <= 768-byte
// streams of a block.  So a thread streams its block's RAW bytes and its
// residual varint bytes through two small state machines (no scratch, no
// warp collectives): 32 neighbouring blocks per warp, coalesced row loads.
struct Sizer {
    int run = 0, lit = 0, size = 0;
    __device__ __forceinline__ void push(uint32_t byte) {
        if (byte == 0) {
            ++run;
            return;
        }
        if (run >= 2) {
            if (lit) size += 1 + (lit >= 64) + lit;
            size += 1 + (run >= 64);
            lit = 0;
        } else {
            lit += run;
        }
        ++lit;
        run = 0;
    }
    __device__ __forceinline__ int finish() {
        if (run >= 2) {
            if (lit) size += 1 + (lit >= 64) + lit;
            size += 1 + (run >= 64);
        } else if (lit + run) {
            size += 1 + (lit + run >= 64) + lit + run;
        }
        return size;
    }
};

__device__ __forceinline__ void push_varint(Sizer &z, uint32_t v) {
    while (v >= 128u) {
        z.push((v & 0x7Fu) | 0x80u);
        v >>= 7;
    }
    z.push(v);
}

__global__ void __launch_bounds__(128) encode_size_thread_kernel(EncArgs a) {
    const int64_t psz = int64_t(a.h) * a.w * a.eb;
    for (int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < a.nblocks;
         b += int64_t(gridDim.x) * blockDim.x) {
        int pl, y0, x0, bh, bw;
        block_coords(a, b, pl, y0, x0, bh, bw);
        const uint8_t *cur = a.cur + pl * psz;
        const bool p_frame = a.ref != nullptr;
        const bool intra = !p_frame && x0 >= 16;
        const uint8_t *pred = p_frame ? a.ref + pl * psz : cur;
        const int px = intra ? x0 - 16 : x0;
        Sizer raw, del;
        bool diff = false;
        for (int y = y0; y < y0 + bh; ++y) {
            for (int x = 0; x < bw; ++x) {
                const uint32_t cv = load_elem(cur, a.w, y, x0 + x, a.eb);
                raw.push(cv & 0xFFu);
                if (a.eb == 2) raw.push(cv >> 8);
                if (p_frame || intra) {
                    const uint32_t pv = load_elem(pred, a.w, y, px + x, a.eb);
                    diff |= cv != pv;
                    int32_t r;
                    if (a.eb == 2) r = int32_t(int16_t(uint16_t(cv - pv)));
                    else r = int32_t(int8_t(uint8_t(cv - pv)));
                    push_varint(del, (uint32_t(r) << 1) ^ uint32_t(r >> 31));
                }
            }
        }
        if (p_frame && !diff) {  // SKIP iff bit-identical to the reference block
            a.sizes[b] = 1;
            a.modes[b] = 0;
            a.lens[b] = 0;
            continue;
        }
        int mode = 2, len = raw.finish();
        if (p_frame || intra) {
            const int dl = del.finish();
            if (dl < len) {  // strictly shorter, ties go to RAW (codec.py:283)
                mode = 1;
                len = dl;
            }
        }
        a.sizes[b] = uint32_t(1 + vlen(uint32_t(len)) + len);
        a.modes[b] = uint8_t(mode);
        a.lens[b] = uint32_t(len);
    }
}

// ---- emit pass, one thread per block, staged per warp ----------------------------------
// Each thread writes its block (mode, uvarint(len), tokens) into the warp's
// shared staging at its offset relative to the warp's first block -- the 32
// blocks of a warp are consecutive in the payload -- and the warp then copies
// the staged bytes out with coalesced stores.  Literal headers are reserved as
// one byte and widened (the segment shifted by one) when the literal reaches
// 64 bytes, the only case whose uvarint(2L) needs two bytes.
constexpr int EMIT_WARPS = 4;
constexpr int BLOCK_OUT_MAX = 776;  // 1 mode + 2 length + 770 tokens, rounded up

struct Emitter {
    uint8_t *o;
    int pos = 0, run = 0, lit = 0, hdr = 0;
    __device__ __forceinline__ void lit_byte(uint32_t v) {
        if (lit == 0) hdr = pos++;
        o[pos++] = uint8_t(v);
        ++lit;
    }
    __device__ __forceinline__ void close_lit() {
        if (!lit) return;
        if (lit >= 64) {  // two-byte header: shift the literal bytes up by one
            for (int i = pos - 1; i > hdr; --i) o[i + 1] = o[i];
            ++pos;
            put_varint(o + hdr, uint32_t(lit) << 1);
        } else {
            o[hdr] = uint8_t(lit << 1);
        }
        lit = 0;
    }
    __device__ __forceinline__ void close_run() {
        close_lit();
        pos += put_varint(o + pos, (uint32_t(run) << 1) | 1u);
    }
    __device__ __forceinline__ void push(uint32_t byte) {
        if (byte == 0) {
            ++run;
            return;
        }
        if (run >= 2) close_run();
        else if (run == 1) lit_byte(0);
        lit_byte(byte);
        run = 0;
    }
    __device__ __forceinline__ void finish() {
        if (run >= 2) close_run();
        else if (run == 1) lit_byte(0);
        close_lit();
    }
};

__device__ __forceinline__ void emit_varint(Emitter &e, uint32_t v) {
    while (v >= 128u) {
        e.push((v & 0x7Fu) | 0x80u);
        v >>= 7;
    }
    e.push(v);
}

__global__ void __launch_bounds__(EMIT_WARPS * 32) encode_emit_thread_kernel(EncArgs a) {
    extern __shared__ uint8_t stage_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint8_t *stage = stage_raw + wid * (32 * BLOCK_OUT_MAX);
    const int64_t psz = int64_t(a.h) * a.w * a.eb;
    const int64_t nwarps = (a.nblocks + 31) / 32;
    for (int64_t wb = int64_t(blockIdx.x) * EMIT_WARPS + wid; wb < nwarps;
         wb += int64_t(gridDim.x) * EMIT_WARPS) {
        const int64_t b0 = wb * 32;
        const int64_t b = b0 + lane;
        const uint64_t base = a.offsets[b0];
        const int64_t last = (b0 + 32 < a.nblocks ? b0 + 32 : a.nblocks) - 1;
        const uint64_t total = a.offsets[last] + a.sizes[last] - base;
        if (b < a.nblocks) {
            Emitter e;
            e.o = stage + (a.offsets[b] - base);
            const int mode = a.modes[b];
            e.o[0] = uint8_t(mode);
            if (mode != 0) {
                e.pos = 1 + put_varint(e.o + 1, a.lens[b]);
                e.o += e.pos;  // tokens start here
                e.pos = 0;
                int pl, y0, x0, bh, bw;
                block_coords(a, b, pl, y0, x0, bh, bw);
                const uint8_t *cur = a.cur + pl * psz;
                const bool intra = a.ref == nullptr;
                const uint8_t *pred = intra ? cur : a.ref + pl * psz;
                const int px = intra ? x0 - 16 : x0;
                for (int y = y0; y < y0 + bh; ++y)
                    for (int x = 0; x < bw; ++x) {
                        const uint32_t cv = load_elem(cur, a.w, y, x0 + x, a.eb);
                        if (mode == 2) {
                            e.push(cv & 0xFFu);
                            if (a.eb == 2) e.push(cv >> 8);
                        } else {
                            const uint32_t pv = load_elem(pred, a.w, y, px + x, a.eb);
                            int32_t r;
                            if (a.eb == 2) r = int32_t(int16_t(uint16_t(cv - pv)));
                            else r = int32_t(int8_t(uint8_t(cv - pv)));
                            emit_varint(e, (uint32_t(r) << 1) ^ uint32_t(r >> 31));
                        }
                    }
                e.finish();
            }
        }
        __syncwarp();
        uint8_t *dst = a.out + HDR + base;
        for (uint64_t i = lane; i < total; i += 32) dst[i] = stage[i];
        __syncwarp();
    }
}

__global__ void __launch_bounds__(WARPS * 32) encode_emit_kernel(EncArgs a) {
    __shared__ WarpScratch scratch[WARPS];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    WarpScratch &ws = scratch[wid];
    for (int64_t b = int64_t(blockIdx.x) * WARPS + wid; b < a.nblocks; b += int64_t(gridDim.x) * WARPS) {
        uint8_t *dst = a.out + HDR + a.offsets[b];
        const int mode = a.modes[b];
        if (mode == 0) {
            if (lane == 0) dst[0] = 0;
            continue;
        }
        int pl, y0, x0, bh, bw;
        block_coords(a, b, pl, y0, x0, bh, bw);
        const bool intra = a.ref == nullptr;
        const int n = build_stream(a, ws, mode, pl, y0, x0, bh, bw, intra, lane);
        const uint32_t len = a.lens[b];
        int hl = 1;
        if (lane == 0) dst[0] = uint8_t(mode);
        hl += vlen(len);
        if (lane == 0) put_varint(dst + 1, len);
        warp_entropy(ws, n, dst + hl, lane);
        __syncwarp();
    }
}

// ---- container + CRC32 ----------------------------------------------------------------

__device__ __forceinline__ uint32_t multmodp(uint32_t a, uint32_t b) {
    if (a == 0) return 0;  // the loop below needs a set bit to terminate
    uint32_t m = 1u << 31, p = 0;
    while (true) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = (b & 1) ? (b >> 1) ^ CRC_POLY : b >> 1;
    }
    return p;
}

// X8[k] = x^(8 * 2^k) mod P (reflected, zlib's representation), k < 48
__constant__ uint32_t c_X8[48] = {
    0x00800000u, 0x00008000u, 0xedb88320u, 0xb1e6b092u, 0xa06a2517u, 0xed627daeu, 0x88d14467u, 0xd7bbfe6au, 0xec447f11u, 0x8e7ea170u, 0x6427800eu, 0x4d47bae0u, 0x09fe548fu, 0x83852d0fu, 0x30362f1au, 0x7b5a9cc3u, 0x31fec169u, 0x9fec022au, 0x6c8dedc4u, 0x15d6874du, 0x5fde7a4eu, 0xbad90e37u, 0x2e4e5eefu, 0x4eaba214u, 0xa8a472c0u, 0x429a969eu, 0x148d302au, 0xc40ba6d0u, 0xc4e22c3cu, 0x40000000u, 0x20000000u, 0x08000000u, 0x00800000u, 0x00008000u, 0xedb88320u, 0xb1e6b092u, 0xa06a2517u, 0xed627daeu, 0x88d14467u, 0xd7bbfe6au, 0xec447f11u, 0x8e7ea170u, 0x6427800eu, 0x4d47bae0u, 0x09fe548fu, 0x83852d0fu, 0x30362f1au, 0x7b5a9cc3u};

// x^(8n) mod P
__device__ __forceinline__ uint32_t x8n(uint64_t n) {
    uint32_t p = 1u << 31;
    for (int k = 0; n; ++k, n >>= 1)
        if (n & 1) p = multmodp(c_X8[k], p);
    return p;
}

__global__ void header_kernel(uint8_t *out, const uint64_t *offsets, const uint32_t *sizes,
                              int64_t nblocks, int key, uint32_t stream_id, uint32_t seq, int w,
                              int h, int bits, uint64_t *frame_len) {
    const uint64_t payload = offsets[nblocks - 1] + sizes[nblocks - 1];
    uint8_t hdr[HDR] = {'L', 'P', 'F', '1'};
    hdr[4] = uint8_t(key ? 1 : 0);
    for (int k = 0; k < 4; ++k) {
        hdr[5 + k] = uint8_t(stream_id >> (8 * k));
        hdr[9 + k] = uint8_t(seq >> (8 * k));
        hdr[19 + k] = uint8_t(uint32_t(payload) >> (8 * k));
    }
    hdr[13] = uint8_t(w);
    hdr[14] = uint8_t(w >> 8);
    hdr[15] = uint8_t(h);
    hdr[16] = uint8_t(h >> 8);
    hdr[17] = 3;
    hdr[18] = uint8_t(bits);
    for (int k = 0; k < HDR; ++k) out[k] = hdr[k];
    *frame_len = HDR + payload + 4;
}

// CRC32 of 4 KB chunks, one thread per chunk: 16-byte loads, slicing-by-16
// (16 independent table lookups per word; only the final XOR is serial)
__global__ void __launch_bounds__(128) crc_chunk_kernel(const uint8_t *data, const uint64_t *frame_len,
                                                       uint32_t *crcs, int64_t max_chunks) {
    __shared__ uint32_t T[16][256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = uint32_t(i);
        for (int k = 0; k < 8; ++k) c = (c & 1) ? CRC_POLY ^ (c >> 1) : c >> 1;
        T[0][i] = c;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = T[0][i];
        for (int k = 1; k < 16; ++k) {
            c = (c >> 8) ^ T[0][c & 0xFFu];
            T[k][i] = c;
        }
    }
    __syncthreads();
    const uint64_t len = *frame_len - 4;  // CRC covers header + payload
    const int64_t chunks = int64_t((len + CRC_CHUNK - 1) / CRC_CHUNK);
    for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < chunks && c < max_chunks;
         c += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t b0 = uint64_t(c) * CRC_CHUNK;
        const uint64_t b1 = b0 + CRC_CHUNK < len ? b0 + CRC_CHUNK : len;
        uint32_t crc = 0xFFFFFFFFu;
        uint64_t i = b0;
        const uint4 *v = reinterpret_cast<const uint4 *>(data + b0);  // chunk starts are 16-B aligned
        for (; i + 16 <= b1; i += 16, ++v) {
            const uint4 q = __ldg(v);
            const uint32_t w0 = q.x ^ crc;
            crc = T[15][w0 & 0xFFu] ^ T[14][(w0 >> 8) & 0xFFu] ^ T[13][(w0 >> 16) & 0xFFu] ^
                  T[12][w0 >> 24] ^ T[11][q.y & 0xFFu] ^ T[10][(q.y >> 8) & 0xFFu] ^
                  T[9][(q.y >> 16) & 0xFFu] ^ T[8][q.y >> 24] ^ T[7][q.z & 0xFFu] ^
                  T[6][(q.z >> 8) & 0xFFu] ^ T[5][(q.z >> 16) & 0xFFu] ^ T[4][q.z >> 24] ^
                  T[3][q.w & 0xFFu] ^ T[2][(q.w >> 8) & 0xFFu] ^ T[1][(q.w >> 16) & 0xFFu] ^
                  T[0][q.w >> 24];
        }
        for (; i < b1; ++i) crc = T[0][(crc ^ data[i]) & 0xFFu] ^ (crc >> 8);
        crcs[c] = crc ^ 0xFFFFFFFFu;
    }
}

// crc(whole) = XOR_c crc(chunk c) * x^(8 * bytes after chunk c): every chunk
// is shifted independently (the product is associative), XOR-reduced per
// block and folded into one word with atomicXor
__global__ void __launch_bounds__(256) crc_shift_kernel(const uint64_t *frame_len,
                                                        const uint32_t *crcs, int64_t max_chunks,
                                                        uint32_t *acc) {
    const uint64_t len = *frame_len - 4;
    const int64_t chunks = int64_t((len + CRC_CHUNK - 1) / CRC_CHUNK);
    uint32_t v = 0;
    for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < chunks && c < max_chunks;
         c += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t end = uint64_t(c + 1) * CRC_CHUNK < len ? uint64_t(c + 1) * CRC_CHUNK : len;
        v ^= multmodp(x8n(len - end), crcs[c]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) v ^= __shfl_xor_sync(0xffffffffu, v, o);
    __shared__ uint32_t part[8];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t r = 0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) r ^= part[w];
        if (r) atomicXor(acc, r);
    }
}

__global__ void crc_store_kernel(uint8_t *out, const uint64_t *frame_len, const uint32_t *acc) {
    const uint64_t len = *frame_len - 4;
    for (int k = 0; k < 4; ++k) out[len + k] = uint8_t(*acc >> (8 * k));
}

struct EncWs {
    uint32_t *sizes, *lens, *crcs, *crc_acc;
    uint8_t *modes;
    uint64_t *offsets, *frame_len;
    void *scan_tmp;
    size_t scan_bytes;
    int64_t max_chunks;
    size_t total;
};

EncWs carve_enc(void *ws, size_t bytes, int64_t nblocks, int64_t capacity) {
    Carver c(ws, bytes);
    EncWs w;
    w.sizes = c.take<uint32_t>(size_t(nblocks));
    w.lens = c.take<uint32_t>(size_t(nblocks));
    w.modes = c.take<uint8_t>(size_t(nblocks));
    w.offsets = c.take<uint64_t>(size_t(nblocks));
    w.frame_len = c.take<uint64_t>(1);
    w.max_chunks = ceil_div(capacity, CRC_CHUNK);
    w.crcs = c.take<uint32_t>(size_t(w.max_chunks));
    w.crc_acc = c.take<uint32_t>(1);
    w.scan_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, w.scan_bytes, (const uint32_t *)nullptr,
                                  (uint64_t *)nullptr, int(nblocks));
    w.scan_tmp = c.take<char>(w.scan_bytes);
    c.take<char>(1);
    w.total = c.off;
    if (ws) c.check();
    return w;
}

int64_t frame_capacity(int64_t h, int64_t w, int eb) {
    const int64_t nb = 3 * ceil_div(h, 16) * ceil_div(w, 16);
    return HDR + 4 + nb * (1 + 3 + 2 * 256 * eb + 8);
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" {

int64_t ps_encode_frame_capacity(int64_t h, int64_t w, int elem_bytes) {
    return frame_capacity(h, w, elem_bytes);
}

size_t ps_encode_workspace_bytes(int64_t h, int64_t w, int elem_bytes) {
    const int64_t nb = std::max<int64_t>(3 * ceil_div(h, 16) * ceil_div(w, 16), 1);
    return carve_enc(nullptr, 0, nb, frame_capacity(h, w, elem_bytes)).total + 256;
}

int ps_encode_frame(int elem_bytes, const void *planes, const void *reference, int64_t h,
                    int64_t w, uint32_t stream_id, uint32_t frame_seq, uint8_t *out,
                    int64_t out_capacity, int64_t *frame_len, void *workspace,
                    size_t workspace_bytes, void *stream) {
    PS_ABI_BEGIN
    if (elem_bytes != 1 && elem_bytes != 2) fail(PS_ERR_VALUE, "element bytes must be 1 or 2");
    if (h < 1 || w < 1 || h > 65535 || w > 65535) fail(PS_ERR_VALUE, "plane dims must be in [1, 65535]");
    if (out_capacity < frame_capacity(h, w, elem_bytes)) fail(PS_ERR_VALUE, "output buffer too small");
    const int64_t nb = 3 * ceil_div(h, 16) * ceil_div(w, 16);
    if (workspace_bytes < ps_encode_workspace_bytes(h, w, elem_bytes))
        fail(PS_ERR_WORKSPACE, "encode workspace too small");
    EncWs ws = carve_enc(workspace, workspace_bytes, nb, frame_capacity(h, w, elem_bytes));
    auto s = as_stream(stream);
    EncArgs a;
    a.cur = static_cast<const uint8_t *>(planes);
    a.ref = static_cast<const uint8_t *>(reference);
    a.eb = elem_bytes;
    a.h = int(h);
    a.w = int(w);
    a.nby = int(ceil_div(h, 16));
    a.nbx = int(ceil_div(w, 16));
    a.nblocks = nb;
    a.sizes = ws.sizes;
    a.lens = ws.lens;
    a.modes = ws.modes;
    a.offsets = ws.offsets;
    a.out = out;
    const unsigned grid = unsigned(std::min<int64_t>(ceil_div(nb, WARPS), int64_t(sm_count()) * 64));
    static const bool warp_size_pass = [] {
        const char *e = getenv("PS_ENCODE_SIZE");  // "warp": the warp-per-block passes
        return e && e[0] == 'w';
    }();
    if (warp_size_pass) {
        encode_size_kernel<<<grid, WARPS * 32, 0, s>>>(a);
        check_launch("encode_size_kernel");
    } else {
        const unsigned tgrid = unsigned(std::min<int64_t>(ceil_div(nb, 128), int64_t(sm_count()) * 16));
        encode_size_thread_kernel<<<tgrid, 128, 0, s>>>(a);
        check_launch("encode_size_thread_kernel");
    }
    size_t tmp = ws.scan_bytes;
    check_cuda(cub::DeviceScan::ExclusiveSum(ws.scan_tmp, tmp, ws.sizes, ws.offsets, int(nb), s),
               "cub ExclusiveSum");
    // emit: the staged thread-per-block pass wins for 1-byte elements (visibility
    // 1.46 -> 1.38 ms key, P 1.59 -> 1.31 ms at C4); with 2-byte elements the
    // 776-byte staging per block caps occupancy and the warp pass stays ahead
    // (colour key 0.54 vs 0.63 ms)
    if (warp_size_pass || elem_bytes == 2) {
        encode_emit_kernel<<<grid, WARPS * 32, 0, s>>>(a);
        check_launch("encode_emit_kernel");
    } else {
        static bool attr = false;
        const int smem = EMIT_WARPS * 32 * BLOCK_OUT_MAX;
        if (!attr) {
            check_cuda(cudaFuncSetAttribute(encode_emit_thread_kernel,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
                       "cudaFuncSetAttribute(emit)");
            attr = true;
        }
        const int64_t nw = ceil_div(nb, 32);
        const unsigned egrid = unsigned(std::min<int64_t>(ceil_div(nw, EMIT_WARPS), int64_t(sm_count()) * 8));
        encode_emit_thread_kernel<<<egrid, EMIT_WARPS * 32, smem, s>>>(a);
        check_launch("encode_emit_thread_kernel");
    }
    header_kernel<<<1, 1, 0, s>>>(out, ws.offsets, ws.sizes, nb, reference == nullptr, stream_id,
                                   frame_seq, int(w), int(h), elem_bytes * 8, ws.frame_len);
    check_launch("header_kernel");
    const unsigned cgrid = unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(ws.max_chunks, 128), 4096)));
    crc_chunk_kernel<<<cgrid, 128, 0, s>>>(out, ws.frame_len, ws.crcs, ws.max_chunks);
    check_launch("crc_chunk_kernel");
    check_cuda(cudaMemsetAsync(ws.crc_acc, 0, sizeof(uint32_t), s), "memset crc");
    const unsigned sgrid = unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(ws.max_chunks, 256), 1024)));
    crc_shift_kernel<<<sgrid, 256, 0, s>>>(ws.frame_len, ws.crcs, ws.max_chunks, ws.crc_acc);
    check_launch("crc_shift_kernel");
    crc_store_kernel<<<1, 1, 0, s>>>(out, ws.frame_len, ws.crc_acc);
    check_launch("crc_store_kernel");
    check_cuda(cudaMemcpyAsync(frame_len, ws.frame_len, sizeof(int64_t), cudaMemcpyDeviceToDevice, s),
               "copy frame length");
    PS_ABI_END
}

}  // extern "C"
