// §8(f) row 3: client side on the GPU -- LPF1 frame decoding (codec.py:106-124,
// 218-236, 295-329, 369-395) and the update-atlas apply with guard-band
// reconstruction (packing.py:341-350, 180-196).  Used as the end-to-end
// verifier of the server path: client atlas == server last-sent atlas.
//
// The payload has no block index, so one thread walks the block headers to
// find every block's offset (SKIP = 1 byte, else mode + LEB128 length +
// payload).  Blocks of a P-frame are then decoded independently (one warp
// per block); key-frame blocks predict from their reconstructed left
// neighbour, so a warp decodes a whole block row left to right.
#include <cuda_runtime.h>

#include "ps_common.cuh"

namespace ps {
namespace {

constexpr int HDR = 23;
constexpr int MAXS = 768;
constexpr uint32_t DEC_ERR_CORRUPT = 1u;   // CorruptFrameError
constexpr uint32_t DEC_ERR_ENTROPY = 2u;   // EntropyDecodeError / malformed stream

struct DecArgs {
    const uint8_t *payload;  // frame + HDR
    uint64_t payload_len;
    const uint8_t *ref;      // previous planes (P-frame) or null (key)
    uint8_t *out;            // decoded planes
    int eb, h, w, nby, nbx;
    int64_t nblocks;
    uint64_t *offsets;
    uint32_t *status;
};

__device__ __forceinline__ bool read_varint(const uint8_t *p, uint64_t len, uint64_t &pos,
                                            uint64_t &value) {
    value = 0;
    int shift = 0;
    while (true) {
        if (pos >= len) return false;
        const uint8_t b = p[pos++];
        value |= uint64_t(b & 0x7F) << shift;
        if (!(b & 0x80)) return true;
        shift += 7;
        if (shift > 63) return false;
    }
}

// single thread: offsets of every block (codec.py:295-316)
__global__ void walk_kernel(DecArgs a) {
    uint64_t pos = 0;
    const bool key = a.ref == nullptr;
    for (int64_t b = 0; b < a.nblocks; ++b) {
        if (pos >= a.payload_len) {
            atomicOr(a.status, DEC_ERR_CORRUPT);  // payload ends mid-plane
            return;
        }
        a.offsets[b] = pos;
        const uint8_t mode = __ldg(a.payload + pos);
        pos += 1;
        if (mode == 0) {
            if (key) {
                atomicOr(a.status, DEC_ERR_CORRUPT);  // SKIP block in a key frame
                return;
            }
            continue;
        }
        if (mode > 2) {
            atomicOr(a.status, DEC_ERR_CORRUPT);  // unknown block mode
            return;
        }
        uint64_t len;
        if (!read_varint(a.payload, a.payload_len, pos, len) || pos + len > a.payload_len) {
            atomicOr(a.status, DEC_ERR_CORRUPT);
            return;
        }
        pos += len;
    }
    if (pos != a.payload_len) atomicOr(a.status, DEC_ERR_CORRUPT);  // trailing bytes
}

__device__ __forceinline__ void block_geom(const DecArgs &a, int64_t b, int &pl, int &y0, int &x0,
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

__device__ __forceinline__ uint32_t get_el(const uint8_t *plane, int w, int y, int x, int eb) {
    const int64_t i = int64_t(y) * w + x;
    return eb == 2 ? uint32_t(reinterpret_cast<const uint16_t *>(plane)[i]) : uint32_t(plane[i]);
}
__device__ __forceinline__ void put_el(uint8_t *plane, int w, int y, int x, int eb, uint32_t v) {
    const int64_t i = int64_t(y) * w + x;
    if (eb == 2)
        reinterpret_cast<uint16_t *>(plane)[i] = uint16_t(v);
    else
        plane[i] = uint8_t(v);
}

// decodes one block (warp); lane 0 expands the token stream into smem
__device__ void decode_block(const DecArgs &a, int64_t b, uint8_t *s, uint32_t *vals, int lane) {
    int pl, y0, x0, bh, bw;
    block_geom(a, b, pl, y0, x0, bh, bw);
    const int64_t psz = int64_t(a.h) * a.w * a.eb;
    uint8_t *dst = a.out + pl * psz;
    const int m = bh * bw;
    uint64_t pos = a.offsets[b];
    const uint8_t mode = a.payload[pos++];
    if (mode == 1 && a.ref == nullptr && x0 < 16) {  // DELTA block without a reference
        if (lane == 0) atomicOr(a.status, DEC_ERR_CORRUPT);
        return;
    }
    if (mode == 0) {  // SKIP: copy the reference block
        const uint8_t *ref = a.ref + pl * psz;
        for (int j = lane; j < m; j += 32) {
            const int y = y0 + j / bw, x = x0 + j % bw;
            put_el(dst, a.w, y, x, a.eb, get_el(ref, a.w, y, x, a.eb));
        }
        return;
    }
    // entropy decode (codec.py:106-124) + value parse, by lane 0
    int ok = 1, n = 0;
    if (lane == 0) {
        uint64_t len;
        read_varint(a.payload, a.payload_len, pos, len);
        const uint64_t end = pos + len;
        while (pos < end && ok) {
            uint64_t hdr;
            if (!read_varint(a.payload, end, pos, hdr)) { ok = 0; break; }
            const uint64_t run = hdr >> 1;
            if (n + run > MAXS) { ok = 0; break; }
            if (hdr & 1) {
                for (uint64_t k = 0; k < run; ++k) s[n++] = 0;
            } else {
                if (run == 0 || pos + run > end) { ok = 0; break; }
                for (uint64_t k = 0; k < run; ++k) s[n++] = a.payload[pos++];
            }
        }
        if (ok) {
            if (mode == 2) {  // RAW: little-endian elements (codec.py:231-236)
                if (n != m * a.eb) ok = 0;
                for (int j = 0; ok && j < m; ++j)
                    vals[j] = a.eb == 2 ? uint32_t(s[2 * j]) | (uint32_t(s[2 * j + 1]) << 8) : s[j];
            } else {  // DELTA: m zig-zag LEB128 residuals, nothing left over (codec.py:218-224)
                uint64_t p = 0;
                for (int j = 0; ok && j < m; ++j) {
                    uint64_t z;
                    if (!read_varint(s, uint64_t(n), p, z)) { ok = 0; break; }
                    const int64_t r = int64_t(z >> 1) ^ -int64_t(z & 1);
                    vals[j] = uint32_t(r);
                }
                if (ok && p != uint64_t(n)) ok = 0;
            }
        }
    }
    ok = __shfl_sync(0xffffffffu, ok, 0);
    __syncwarp();
    if (!ok) {
        if (lane == 0) atomicOr(a.status, DEC_ERR_ENTROPY);
        return;
    }
    const uint32_t mask = a.eb == 2 ? 0xFFFFu : 0xFFu;
    if (mode == 2) {
        for (int j = lane; j < m; j += 32) put_el(dst, a.w, y0 + j / bw, x0 + j % bw, a.eb, vals[j]);
    } else {
        const bool key = a.ref == nullptr;
        const uint8_t *pred = key ? dst : a.ref + pl * psz;
        const int px = key ? x0 - 16 : x0;
        for (int j = lane; j < m; j += 32) {
            const int y = y0 + j / bw, xo = j % bw;
            const uint32_t v = (get_el(pred, a.w, y, px + xo, a.eb) + vals[j]) & mask;
            put_el(dst, a.w, y, x0 + xo, a.eb, v);
        }
    }
}

constexpr int DWARPS = 4;

__global__ void __launch_bounds__(DWARPS * 32) decode_p_kernel(DecArgs a) {
    __shared__ uint8_t s[DWARPS][MAXS];
    __shared__ uint32_t vals[DWARPS][256];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t b = int64_t(blockIdx.x) * DWARPS + wid; b < a.nblocks; b += int64_t(gridDim.x) * DWARPS)
        decode_block(a, b, s[wid], vals[wid], lane);
}

// key frames: a warp decodes a block row left to right (intra prediction)
__global__ void __launch_bounds__(DWARPS * 32) decode_key_kernel(DecArgs a) {
    __shared__ uint8_t s[DWARPS][MAXS];
    __shared__ uint32_t vals[DWARPS][256];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t rows = a.nblocks / a.nbx;
    for (int64_t r = int64_t(blockIdx.x) * DWARPS + wid; r < rows; r += int64_t(gridDim.x) * DWARPS)
        for (int bx = 0; bx < a.nbx; ++bx) {
            decode_block(a, r * a.nbx + bx, s[wid], vals[wid], lane);
            __syncwarp();
            __threadfence_block();
        }
}

// client apply (packing.py:341-350): slot core -> probe block + guard band
template <int SIDE>
__global__ void __launch_bounds__(256)
    apply_kernel(const uint32_t *upd, int64_t upd_w, int64_t slots_per_row, const int64_t *entries,
                 const int64_t *entry_count, uint32_t *atlas, int64_t atlas_w, int64_t ppr) {
    constexpr int CORE = SIDE - 2;
    const int64_t count = *entry_count;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t e = warp; e < count; e += nwarps) {
        const int64_t slot = entries[2 * e], p = entries[2 * e + 1];
        int64_t sy, sx;
        block_origin(slot, slots_per_row, CORE, sy, sx);
        int64_t y0, x0;
        block_origin(p, ppr, SIDE, y0, x0);
        for (int k = lane; k < SIDE * SIDE; k += 32) {
            const int r = k / SIDE, c = k % SIDE;
            const int n = CORE;
            const bool top = r == 0, bot = r == SIDE - 1, left = c == 0, right = c == SIDE - 1;
            int rr = r, cc = c;
            if ((top || bot) && (left || right)) {
                rr = top ? n : 1;
                cc = left ? n : 1;
            } else if (top || bot) {
                rr = top ? 1 : n;
                cc = SIDE - 1 - c;
            } else if (left || right) {
                rr = SIDE - 1 - r;
                cc = left ? 1 : n;
            }
            atlas[(y0 + r) * atlas_w + x0 + c] = upd[(sy + rr - 1) * upd_w + sx + cc - 1];
        }
    }
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" {

size_t ps_decode_workspace_bytes(int64_t h, int64_t w) {
    return size_t(3 * ceil_div(h, 16) * ceil_div(w, 16)) * 8 + 256;
}

int ps_decode_frame(int elem_bytes, const uint8_t *frame, int64_t payload_len,
                    const void *reference, int64_t h, int64_t w, void *planes_out,
                    uint32_t *status_dev, void *workspace, size_t workspace_bytes, void *stream) {
    PS_ABI_BEGIN
    if (elem_bytes != 1 && elem_bytes != 2) fail(PS_ERR_VALUE, "element bytes must be 1 or 2");
    if (h < 1 || w < 1) fail(PS_ERR_VALUE, "plane dims must be >= 1");
    if (workspace_bytes < ps_decode_workspace_bytes(h, w)) fail(PS_ERR_WORKSPACE, "decode workspace");
    auto s = as_stream(stream);
    DecArgs a;
    a.payload = frame + HDR;
    a.payload_len = uint64_t(payload_len);
    a.ref = static_cast<const uint8_t *>(reference);
    a.out = static_cast<uint8_t *>(planes_out);
    a.eb = elem_bytes;
    a.h = int(h);
    a.w = int(w);
    a.nby = int(ceil_div(h, 16));
    a.nbx = int(ceil_div(w, 16));
    a.nblocks = 3 * int64_t(a.nby) * a.nbx;
    a.offsets = static_cast<uint64_t *>(workspace);
    a.status = status_dev;
    walk_kernel<<<1, 1, 0, s>>>(a);
    check_launch("walk_kernel");
    if (reference) {
        const unsigned grid = unsigned(std::min<int64_t>(ceil_div(a.nblocks, DWARPS), int64_t(sm_count()) * 32));
        decode_p_kernel<<<grid, DWARPS * 32, 0, s>>>(a);
    } else {
        const int64_t rows = a.nblocks / a.nbx;
        decode_key_kernel<<<unsigned(std::max<int64_t>(1, ceil_div(rows, DWARPS))), DWARPS * 32, 0, s>>>(a);
    }
    check_launch("decode_kernel");
    PS_ABI_END
}

int ps_apply_entries(int kind, const void *update_texels, int64_t update_row_stride,
                     int64_t slots_per_row, const int64_t *entries, const int64_t *entry_count,
                     int64_t max_entries, void *atlas, int64_t probes_per_row, void *stream) {
    PS_ABI_BEGIN
    if (kind != PS_KIND_COLOR && kind != PS_KIND_VISIBILITY) fail(PS_ERR_VALUE, "bad kind");
    if (max_entries <= 0) return PS_OK;
    auto s = as_stream(stream);
    const unsigned blocks = unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(max_entries, 8), 4096)));
    if (kind == PS_KIND_COLOR)
        apply_kernel<10><<<blocks, 256, 0, s>>>(static_cast<const uint32_t *>(update_texels),
                                                update_row_stride, slots_per_row, entries,
                                                entry_count, static_cast<uint32_t *>(atlas),
                                                probes_per_row * 10, probes_per_row);
    else
        apply_kernel<18><<<blocks, 256, 0, s>>>(static_cast<const uint32_t *>(update_texels),
                                                update_row_stride, slots_per_row, entries,
                                                entry_count, static_cast<uint32_t *>(atlas),
                                                probes_per_row * 18, probes_per_row);
    check_launch("apply_kernel");
    PS_ABI_END
}

}  // extern "C"
