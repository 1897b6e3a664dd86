// Stage (4): lossless plane packing + temporal delta (+ SKIP map), sm_100a.
//
// One kernel family covers pack_color (packing.py:73-89), pack_visibility
// (packing.py:112-133) and the codec's temporal residual / SKIP rule
// (codec.py:207-215, :250-272).  The unit of work is a 16-element row
// segment of a plane, which is exactly one row of one 16x16 codec block:
//   colour     : 16 texels (64 B)      -> 16 uint16 per plane
//   visibility : 12 texels (48 B)      -> 16 uint8 per plane  (48 stream bytes)
// so the SKIP decision of a block is an OR over the 16 threads that own its
// rows, and every byte is read once and written once (HBM-bound).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <algorithm>
#include <mutex>
#include <string>

#include "ps_common.cuh"

namespace ps {

static thread_local std::string g_last_error;
void set_last_error(const std::string &msg) { g_last_error = msg; }

namespace {

constexpr int SEG = 16;     // elements per plane per thread == codec block side
constexpr int TILE_X = 16;  // segments (codec blocks) per CTA in x
constexpr int TILE_Y = 16;  // rows per CTA == codec block side

__device__ __forceinline__ uint32_t bfe10(uint32_t t, int e) { return (t >> (10 * e)) & 0x3FFu; }

// Visibility: 3 texel words (R | G << 16, little endian) -> 4 plane bytes per
// plane.  Stream per texel is [R.hi, R.lo, G.hi, G.lo]; byte k of the 12-byte
// stream goes to plane k % 3, element k / 3.
__device__ __forceinline__ void vis_group(uint32_t t0, uint32_t t1, uint32_t t2, uint32_t &y,
                                          uint32_t &u, uint32_t &v) {
    // stream bytes: s0=t0.b1 s1=t0.b0 s2=t0.b3 s3=t0.b2 s4=t1.b1 s5=t1.b0
    //               s6=t1.b3 s7=t1.b2 s8=t2.b1 s9=t2.b0 s10=t2.b3 s11=t2.b2
    // Y = s0 s3 s6 s9 ; U = s1 s4 s7 s10 ; V = s2 s5 s8 s11
    // __byte_perm(x, y, sel): result byte i = byte sel_i of {y:x} (x: 0..3, y: 4..7)
    y = __byte_perm(__byte_perm(t0, t1, 0x0721), t2, 0x4210);  // t0.b1 t0.b2 t1.b3 t2.b0
    u = __byte_perm(__byte_perm(t0, t1, 0x0650), t2, 0x7210);  // t0.b0 t1.b1 t1.b2 t2.b3
    v = __byte_perm(__byte_perm(t0, t1, 0x0043), t2, 0x6510);  // t0.b3 t1.b0 t2.b1 t2.b2
}

struct PackArgs {
    const uint8_t *texels;  // colour u32 / visibility u16x2 texel rows
    int64_t h, w;           // texel rows / texels per row
    int64_t row_stride_b;   // texel row stride in bytes
    int64_t pw;             // plane width in elements
    int64_t nseg;           // segments (16-element blocks) per row
    uint8_t *cur;           // planes (3, h, pw)
    const uint8_t *prev;    // previous planes or nullptr
    uint8_t *residual;      // may be nullptr
    uint8_t *skip;          // (3, ceil(h/16), nseg) or nullptr
    int vec_in;             // texel rows 16-byte aligned
    int vec_out;            // plane rows 16-byte aligned
    const int32_t *key_dev; // optional device flag: non-zero = key frame (ignore prev)
};

// Loads the 16-element segment `seg` of row `r` for all three planes into
// `out` as 32-bit words (colour: 8 words of 2 x u16; visibility: 4 words of
// 4 x u8).  Elements beyond the plane width are zero.
template <int KIND>
__device__ __forceinline__ void load_segment(const PackArgs &a, int64_t r, int64_t seg,
                                             uint32_t out[3][8]) {
    const uint8_t *row = a.texels + r * a.row_stride_b;
    if (KIND == PS_KIND_COLOR) {
        const int64_t x0 = seg * SEG;
        uint32_t t[16];
        if (a.vec_in && x0 + 16 <= a.w) {
            const uint4 *p = reinterpret_cast<const uint4 *>(row + x0 * 4);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                uint4 q = __ldg(p + i);
                t[4 * i] = q.x;
                t[4 * i + 1] = q.y;
                t[4 * i + 2] = q.z;
                t[4 * i + 3] = q.w;
            }
        } else {
            const uint32_t *p = reinterpret_cast<const uint32_t *>(row);
#pragma unroll
            for (int i = 0; i < 16; ++i) t[i] = (x0 + i < a.w) ? __ldg(p + x0 + i) : 0u;
        }
#pragma unroll
        for (int e = 0; e < 3; ++e)
#pragma unroll
            for (int i = 0; i < 8; ++i)
                out[e][i] = bfe10(t[2 * i], e) | (bfe10(t[2 * i + 1], e) << 16);
    } else {
        const int64_t t0 = seg * 12;  // first texel of the 48-byte stream window
        uint32_t t[12];
        if (a.vec_in && t0 + 12 <= a.w) {
            const uint4 *p = reinterpret_cast<const uint4 *>(row + t0 * 4);
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                uint4 q = __ldg(p + i);
                t[4 * i] = q.x;
                t[4 * i + 1] = q.y;
                t[4 * i + 2] = q.z;
                t[4 * i + 3] = q.w;
            }
        } else {
            const uint32_t *p = reinterpret_cast<const uint32_t *>(row);
#pragma unroll
            for (int i = 0; i < 12; ++i) t[i] = (t0 + i < a.w) ? __ldg(p + t0 + i) : 0u;
        }
#pragma unroll
        for (int g = 0; g < 4; ++g) vis_group(t[3 * g], t[3 * g + 1], t[3 * g + 2], out[0][g],
                                              out[1][g], out[2][g]);
#pragma unroll
        for (int e = 0; e < 3; ++e)
#pragma unroll
            for (int i = 4; i < 8; ++i) out[e][i] = 0u;
    }
}

template <int KIND>
__device__ __forceinline__ void load_plane_words(const uint8_t *base, int64_t x0_b,
                                                 int64_t valid_b, bool vec, uint32_t w[8]) {
    constexpr int NB = (KIND == PS_KIND_COLOR) ? 32 : 16;  // bytes per segment
    const uint8_t *p = base + x0_b;
    if (vec && valid_b >= NB) {
        const uint4 *q = reinterpret_cast<const uint4 *>(p);
#pragma unroll
        for (int i = 0; i < NB / 16; ++i) {
            uint4 v = __ldg(q + i);
            w[4 * i] = v.x;
            w[4 * i + 1] = v.y;
            w[4 * i + 2] = v.z;
            w[4 * i + 3] = v.w;
        }
#pragma unroll
        for (int i = NB / 4; i < 8; ++i) w[i] = 0u;
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            uint32_t v = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                int64_t b = 4 * i + k;
                if (b < NB && b < valid_b) v |= uint32_t(p[b]) << (8 * k);
            }
            w[i] = v;
        }
    }
}

template <int KIND>
__device__ __forceinline__ void store_plane_words(uint8_t *base, int64_t x0_b, int64_t valid_b,
                                                  bool vec, const uint32_t w[8]) {
    constexpr int NB = (KIND == PS_KIND_COLOR) ? 32 : 16;
    uint8_t *p = base + x0_b;
    if (vec && valid_b >= NB) {
        uint4 *q = reinterpret_cast<uint4 *>(p);
#pragma unroll
        for (int i = 0; i < NB / 16; ++i)
            q[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                int64_t b = 4 * i + k;
                if (b < NB && b < valid_b) p[b] = uint8_t(w[i] >> (8 * k));
            }
    }
}

template <int KIND>
__global__ void __launch_bounds__(TILE_X *TILE_Y)
    pack_delta_kernel(PackArgs a) {
    if (a.key_dev && *a.key_dev) a.prev = nullptr;  // key frame decided on the device
    constexpr int EB = (KIND == PS_KIND_COLOR) ? 2 : 1;  // element bytes
    constexpr int NB = SEG * EB;                         // bytes per plane segment
    __shared__ uint32_t dirty[3][TILE_X];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t seg = int64_t(blockIdx.x) * TILE_X + tx;
    const int64_t by = blockIdx.y;
    const int64_t r = by * TILE_Y + ty;
    if (ty == 0)
        for (int e = 0; e < 3; ++e) dirty[e][tx] = 0u;
    __syncthreads();
    if (seg < a.nseg && r < a.h) {
        // colour keeps the 16 texel words and extracts one plane at a time (the
        // three planes at once held ~120 registers); visibility's byte shuffles
        // produce all planes together
        uint32_t cur[3][8];
        uint32_t tex[16];
        if (KIND == PS_KIND_COLOR) {
            const int64_t x0 = seg * SEG;
            const uint8_t *row = a.texels + r * a.row_stride_b;
            if (a.vec_in && x0 + 16 <= a.w) {
                const uint4 *p = reinterpret_cast<const uint4 *>(row + x0 * 4);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint4 q = __ldg(p + i);
                    tex[4 * i] = q.x;
                    tex[4 * i + 1] = q.y;
                    tex[4 * i + 2] = q.z;
                    tex[4 * i + 3] = q.w;
                }
            } else {
                const uint32_t *p = reinterpret_cast<const uint32_t *>(row);
#pragma unroll
                for (int i = 0; i < 16; ++i) tex[i] = (x0 + i < a.w) ? __ldg(p + x0 + i) : 0u;
            }
        } else {
            load_segment<KIND>(a, r, seg, cur);
        }
        const int64_t x0_b = seg * NB;
        const int64_t valid_b = (a.pw - seg * SEG) * EB;
        const int64_t plane_b = a.h * a.pw * EB;
        const int64_t row_b = r * a.pw * EB;
#pragma unroll
        for (int e = 0; e < 3; ++e) {
            if (KIND == PS_KIND_COLOR) {
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    cur[e][i] = bfe10(tex[2 * i], e) | (bfe10(tex[2 * i + 1], e) << 16);
            }
            uint8_t *dst = a.cur + e * plane_b + row_b;
            if (a.prev) {
                uint32_t pv[8];
                load_plane_words<KIND>(a.prev + e * plane_b + row_b, x0_b, valid_b, a.vec_out,
                                       pv);
                uint32_t any = 0, res[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    any |= cur[e][i] ^ pv[i];
                    res[i] = (KIND == PS_KIND_COLOR) ? __vsub2(cur[e][i], pv[i])
                                                     : __vsub4(cur[e][i], pv[i]);
                }
                if (a.residual)
                    store_plane_words<KIND>(a.residual + e * plane_b + row_b, x0_b, valid_b,
                                            a.vec_out, res);
                if (any) atomicOr(&dirty[e][tx], 1u);
            }
            store_plane_words<KIND>(dst, x0_b, valid_b, a.vec_out, cur[e]);
        }
    }
    __syncthreads();
    if (a.skip && ty < 3 && seg < a.nseg) {
        const int64_t nby = (a.h + TILE_Y - 1) / TILE_Y;
        uint8_t s = a.prev ? uint8_t(dirty[ty][tx] == 0u) : uint8_t(0);
        a.skip[(int64_t(ty) * nby + by) * a.nseg + seg] = s;
    }
}

// Visibility planes whose rows are not 16-byte aligned (plane width
// ceil(4w/3) % 16 != 0, e.g. a 4,096-texel update atlas): same work as
// pack_delta_kernel, but the 16-byte plane segments are funnel-shifted onto
// the aligned 16-byte words of the row.  Thread j writes the aligned word that
// holds its segment's tail and the next segment's head (taken from lane j+1
// with a 16-wide shuffle); only the first / last thread of a tile row and the
// row ends fall back to byte stores.  Previous planes are read as the two
// aligned words around each segment.
__device__ __forceinline__ void funnel16(const uint32_t lo[4], const uint32_t hi[4], int s,
                                         uint32_t out[4]) {
    // bytes [s, s + 16) of lo || hi, 0 <= s <= 16
    const uint32_t c[9] = {lo[0], lo[1], lo[2], lo[3], hi[0], hi[1], hi[2], hi[3], 0u};
    const int q = s >> 2, r = (s & 3) * 8;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        uint32_t a0 = c[i], a1 = c[i + 1];
#pragma unroll
        for (int k = 1; k <= 4; ++k) {
            a0 = q == k ? c[i + k] : a0;
            a1 = q == k ? c[i + k + 1 < 9 ? i + k + 1 : 8] : a1;
        }
        out[i] = r ? __funnelshift_r(a0, a1, r) : a0;
    }
}

// bytes [lo, hi) of the 16-byte value x to the 16-byte aligned address base,
// as a few naturally aligned 8 / 4 / 2 / 1-byte stores
__device__ __forceinline__ void store_range(uint8_t *base, const uint32_t x[4], int lo, int hi) {
    while (lo < hi) {
        const int q = lo >> 2;
        const uint32_t wq = q == 0 ? x[0] : q == 1 ? x[1] : q == 2 ? x[2] : x[3];
        if ((lo & 7) == 0 && lo + 8 <= hi) {
            *reinterpret_cast<uint2 *>(base + lo) = make_uint2(wq, q == 0 ? x[1] : x[3]);
            lo += 8;
        } else if ((lo & 3) == 0 && lo + 4 <= hi) {
            *reinterpret_cast<uint32_t *>(base + lo) = wq;
            lo += 4;
        } else if ((lo & 1) == 0 && lo + 2 <= hi) {
            *reinterpret_cast<uint16_t *>(base + lo) = uint16_t(wq >> (8 * (lo & 3)));
            lo += 2;
        } else {
            base[lo] = uint8_t(wq >> (8 * (lo & 3)));
            lo += 1;
        }
    }
}

// one 16-byte segment at row offset x0_b of the row starting at `row` (any
// alignment); valid_b = row bytes from the segment start on.  Every lane of
// the 16-wide group calls this (inactive lanes with valid_b <= 0).
__device__ __forceinline__ void store_seg_unaligned(uint8_t *row, int64_t x0_b, int64_t valid_b,
                                                    int tx, const uint32_t w[4]) {
    const int m = int(reinterpret_cast<uintptr_t>(row) & 15u);  // x0_b is a multiple of 16
    uint32_t nxt[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) nxt[i] = __shfl_down_sync(0xffffffffu, w[i], 1, 16);
    if (valid_b <= 0) return;
    uint8_t *seg = row + x0_b;
    if (m == 0) {
        if (valid_b >= 16)
            *reinterpret_cast<uint4 *>(seg) = make_uint4(w[0], w[1], w[2], w[3]);
        else
            store_range(seg, w, 0, int(valid_b));
        return;
    }
    const uint32_t zero[4] = {0u, 0u, 0u, 0u};
    // head: segment bytes [0, 16 - m) = word j bytes [m, 16), written by the previous
    // lane unless this is the tile row's first lane
    if (tx == 0) {
        uint32_t x[4];
        funnel16(zero, w, 16 - m, x);
        store_range(seg - m, x, m, m + int(valid_b < 16 - m ? valid_b : 16 - m));
    }
    if (valid_b <= 16 - m) return;  // the segment ends inside word j
    // word j + 1: our tail (m bytes) then the next segment's head (16 - m bytes)
    uint8_t *word = seg + (16 - m);  // 16-byte aligned
    const int64_t in_row = valid_b - (16 - m);  // row bytes from `word` on (ours + later)
    uint32_t x[4];
    funnel16(w, nxt, 16 - m, x);
    if (tx < 15 && in_row >= 16) {
        *reinterpret_cast<uint4 *>(word) = make_uint4(x[0], x[1], x[2], x[3]);
        return;
    }
    const int64_t lim = tx < 15 ? 16 : m;  // the last lane only owns its own tail
    store_range(word, x, 0, int(in_row < lim ? in_row : lim));
}

__global__ void __launch_bounds__(TILE_X *TILE_Y)
    pack_delta_vis_unaligned_kernel(PackArgs a) {
    if (a.key_dev && *a.key_dev) a.prev = nullptr;
    __shared__ uint32_t dirty[3][TILE_X];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t seg = int64_t(blockIdx.x) * TILE_X + tx;
    const int64_t by = blockIdx.y;
    const int64_t r = by * TILE_Y + ty;
    if (ty == 0)
        for (int e = 0; e < 3; ++e) dirty[e][tx] = 0u;
    __syncthreads();
    const bool active = seg < a.nseg && r < a.h;
    uint32_t cur[3][8];
    if (active) {
        load_segment<PS_KIND_VISIBILITY>(a, r, seg, cur);
    } else {
#pragma unroll
        for (int e = 0; e < 3; ++e)
#pragma unroll
            for (int i = 0; i < 8; ++i) cur[e][i] = 0u;
    }
    const int64_t x0_b = seg * SEG;
    const int64_t valid_b = active ? a.pw - seg * SEG : 0;
    const int64_t plane_b = a.h * a.pw;
    const int64_t row_b = (r < a.h ? r : 0) * a.pw;
#pragma unroll
    for (int e = 0; e < 3; ++e) {
        if (a.prev) {
            uint32_t pv[4] = {0u, 0u, 0u, 0u};
            if (active) {
                const uint8_t *p = a.prev + e * plane_b + row_b + x0_b;
                const int m = int(reinterpret_cast<uintptr_t>(p) & 15u);
                const uint8_t *al = p - m;
                const int64_t left = (a.prev + 3 * plane_b) - al;  // bytes to the buffer end
                if (left >= 32) {
                    const uint4 l0 = __ldg(reinterpret_cast<const uint4 *>(al));
                    const uint4 l1 = __ldg(reinterpret_cast<const uint4 *>(al) + 1);
                    const uint32_t lo[4] = {l0.x, l0.y, l0.z, l0.w}, hi[4] = {l1.x, l1.y, l1.z, l1.w};
                    funnel16(lo, hi, m, pv);
                } else {
                    for (int b = 0; b < 16 && b < valid_b; ++b)
                        pv[b >> 2] |= uint32_t(p[b]) << (8 * (b & 3));
                }
                if (valid_b < 16) {  // bytes past the row end count as zero, as in the cur planes
                    for (int b = int(valid_b); b < 16; ++b) pv[b >> 2] &= ~(0xFFu << (8 * (b & 3)));
                }
            }
            uint32_t any = 0, res[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                any |= cur[e][i] ^ pv[i];
                res[i] = __vsub4(cur[e][i], pv[i]);
            }
            if (a.residual)
                store_seg_unaligned(a.residual + e * plane_b + row_b, x0_b, valid_b, tx, res);
            if (active && any) atomicOr(&dirty[e][tx], 1u);
        }
        store_seg_unaligned(a.cur + e * plane_b + row_b, x0_b, valid_b, tx, cur[e]);
    }
    __syncthreads();
    if (a.skip && ty < 3 && seg < a.nseg) {
        const int64_t nby = (a.h + TILE_Y - 1) / TILE_Y;
        uint8_t sk = a.prev ? uint8_t(dirty[ty][tx] == 0u) : uint8_t(0);
        a.skip[(int64_t(ty) * nby + by) * a.nseg + seg] = sk;
    }
}

// Visibility planes with misaligned rows, as a flat byte array per plane: a
// thread owns one 16-byte-aligned word of every plane (the same flat offset
// in all three), so every plane / residual store and previous-plane load is
// one aligned 16-byte access -- no funnel shifts, no partial stores.  Needs
// planes whose size h * pw is a multiple of 16 (update atlases: h is a
// multiple of 16) at least 16 bytes wide.  A word covers plane columns
// [x0, x0 + 16) of one row, or the tail of row r and the head of row r + 1.
//
// The word's stream window: plane column x needs stream byte 3x + e, i.e.
// texel (3x + e) >> 2, byte ((3x + e) & 3) ^ 1 of the little-endian texel
// word (stream order R.hi R.lo G.hi G.lo).  With c = 3 * x0 mod 16 the 16
// texels from (3 * x0 - c) / 4 (one aligned 64-byte window) hold every stream
// byte of the word, and c is the same for every word of a row, so the byte
// gather is a compile-time PRMT pattern chosen by a row-uniform switch on c.
template <int C, int E, int J>
__device__ __forceinline__ uint32_t vis_word(const uint32_t (&t)[16]) {
    // output bytes i = 4J + p, p = 0..3 <- stream byte k = C + 3i + E, i.e. byte
    // (k & 3) ^ 1 of texel k >> 2; the four bytes span up to four texels
    // ta..ta+3, gathered by up to three permutes: (t[ta], t[ta+1]), then the
    // result with t[ta+2], then with t[ta+3]
    constexpr auto tex = [](int p) { return (C + 3 * (4 * J + p) + E) >> 2; };
    constexpr auto byt = [](int p) { return ((C + 3 * (4 * J + p) + E) & 3) ^ 1; };
    constexpr int ta = tex(0);
    constexpr auto sel1 = [](int p) { return tex(p) - tex(0) < 2 ? (tex(p) - tex(0)) * 4 + byt(p) : 0; };
    constexpr auto sel2 = [](int p) { return tex(p) - tex(0) == 2 ? 4 + byt(p) : p; };
    constexpr auto sel3 = [](int p) { return tex(p) - tex(0) == 3 ? 4 + byt(p) : p; };
    constexpr uint32_t s1 = sel1(0) | (sel1(1) << 4) | (sel1(2) << 8) | (sel1(3) << 12);
    constexpr uint32_t s2 = sel2(0) | (sel2(1) << 4) | (sel2(2) << 8) | (sel2(3) << 12);
    constexpr uint32_t s3 = sel3(0) | (sel3(1) << 4) | (sel3(2) << 8) | (sel3(3) << 12);
    uint32_t v = __byte_perm(t[ta], t[ta + 1 < 16 ? ta + 1 : 15], s1);
    if constexpr (tex(3) - ta >= 2) v = __byte_perm(v, t[ta + 2 < 16 ? ta + 2 : 15], s2);
    if constexpr (tex(3) - ta >= 3) v = __byte_perm(v, t[ta + 3 < 16 ? ta + 3 : 15], s3);
    return v;
}

template <int C>
__device__ __forceinline__ void vis_words(const uint32_t (&t)[16], uint32_t (&o)[3][4]) {
#define PS_VW(E, J) o[E][J] = vis_word<C, E, J>(t);
    PS_VW(0, 0) PS_VW(0, 1) PS_VW(0, 2) PS_VW(0, 3)
    PS_VW(1, 0) PS_VW(1, 1) PS_VW(1, 2) PS_VW(1, 3)
    PS_VW(2, 0) PS_VW(2, 1) PS_VW(2, 2) PS_VW(2, 3)
#undef PS_VW
}

// the 16 plane bytes (3 planes) of row r, columns [x0, x0 + 16); x0 may be
// negative (the head of a straddling word), texels outside the row read as 0
__device__ __forceinline__ void vis_segment(const PackArgs &a, int r, int x0,
                                            uint32_t (&o)[3][4]) {
    const int s0 = 3 * x0;
    const int c = s0 & 15;         // 3 * x0 mod 16, also for negative x0
    const int t0 = (s0 - c) >> 2;  // multiple of 4 texels (16 bytes)
    const uint8_t *row = a.texels + int64_t(r) * a.row_stride_b;
    uint32_t t[16];
    if (t0 >= 0 && t0 + 16 <= int(a.w)) {  // rows are 16-byte aligned (vec_in)
        const uint4 *p = reinterpret_cast<const uint4 *>(row + 4 * t0);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint4 q = __ldg(p + i);
            t[4 * i] = q.x;
            t[4 * i + 1] = q.y;
            t[4 * i + 2] = q.z;
            t[4 * i + 3] = q.w;
        }
    } else {
        const uint32_t *p = reinterpret_cast<const uint32_t *>(row);
#pragma unroll
        for (int i = 0; i < 16; ++i)
            t[i] = (t0 + i >= 0 && t0 + i < int(a.w)) ? __ldg(p + t0 + i) : 0u;
    }
    switch (c) {
#define PS_VC(C) case C: vis_words<C>(t, o); break;
        PS_VC(0) PS_VC(1) PS_VC(2) PS_VC(3) PS_VC(4) PS_VC(5) PS_VC(6) PS_VC(7)
        PS_VC(8) PS_VC(9) PS_VC(10) PS_VC(11) PS_VC(12) PS_VC(13) PS_VC(14)
        default: vis_words<15>(t, o);
#undef PS_VC
    }
}

// bytes [lo, hi) of a 16-byte word as a 4 x 32-bit lane mask
__device__ __forceinline__ uint32_t byte_mask_word(int j, int lo, int hi) {
    uint32_t m = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) m |= (4 * j + b >= lo && 4 * j + b < hi) ? (0xFFu << (8 * b)) : 0u;
    return m;
}

__global__ void __launch_bounds__(256) pack_delta_vis_flat_kernel(PackArgs a) {
    const bool key = a.key_dev && *a.key_dev;
    const uint8_t *prev = key ? nullptr : a.prev;
    // 32-bit offsets: the launcher routes planes of >= 2^31 bytes elsewhere
    const uint32_t pw = uint32_t(a.pw), h = uint32_t(a.h);
    const uint32_t T = h * pw;  // bytes per plane, multiple of 16
    const uint32_t nwords = T / 16;
    const uint32_t nby = (h + TILE_Y - 1) / TILE_Y, nseg = uint32_t(a.nseg);
    for (uint32_t W = blockIdx.x * blockDim.x + threadIdx.x; W < nwords;
         W += gridDim.x * blockDim.x) {
        const uint32_t f0 = 16 * W;
        const uint32_t r = f0 / pw, x0 = f0 - r * pw;
        const int n1 = int(pw - x0 < 16 ? pw - x0 : 16);  // bytes in row r
        uint32_t o[3][4];
        vis_segment(a, int(r), int(x0), o);
        if (n1 < 16) {  // the word runs into row r + 1: its columns [0, 16 - n1)
            uint32_t o2[3][4];
            vis_segment(a, int(r) + 1, -n1, o2);  // byte i <- column i - n1
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t m = byte_mask_word(j, 0, n1);
#pragma unroll
                for (int e = 0; e < 3; ++e) o[e][j] = (o[e][j] & m) | (o2[e][j] & ~m);
            }
        }
#pragma unroll
        for (int e = 0; e < 3; ++e) {
            const size_t off = size_t(e) * T + f0;
            *reinterpret_cast<uint4 *>(a.cur + off) = make_uint4(o[e][0], o[e][1], o[e][2], o[e][3]);
            if (!a.skip && !a.residual) continue;
            uint32_t d[4] = {o[e][0], o[e][1], o[e][2], o[e][3]};
            if (prev) {
                const uint4 pv = __ldg(reinterpret_cast<const uint4 *>(prev + off));
                const uint32_t pw4[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) d[j] = o[e][j] ^ pw4[j];
                if (a.residual)
                    *reinterpret_cast<uint4 *>(a.residual + off) =
                        make_uint4(__vsub4(o[e][0], pw4[0]), __vsub4(o[e][1], pw4[1]),
                                   __vsub4(o[e][2], pw4[2]), __vsub4(o[e][3], pw4[3]));
            } else if (a.residual) {
                *reinterpret_cast<uint4 *>(a.residual + off) =
                    make_uint4(o[e][0], o[e][1], o[e][2], o[e][3]);
            }
            if (!a.skip) continue;
            // SKIP (preset to 1): a changed byte clears its codec block; key frames
            // clear every block the word touches.  Bytes [lo, hi) of the word are
            // row rr, columns xa + (b - lo); they meet at most two blocks.
            auto clear = [&](uint32_t rr, uint32_t xa, int lo, int hi) {
                const uint32_t bxa = xa >> 4, bxb = (xa + uint32_t(hi - lo) - 1) >> 4;
                uint8_t *sk = a.skip + (size_t(e) * nby + (rr >> 4)) * nseg;
                for (uint32_t bx = bxa; bx <= bxb; ++bx) {
                    const int blo = lo + int(bx * 16 > xa ? bx * 16 - xa : 0);
                    const int bhi = lo + int((bx + 1) * 16 - xa < uint32_t(hi - lo)
                                                 ? (bx + 1) * 16 - xa : uint32_t(hi - lo));
                    bool dirty = !prev;
#pragma unroll
                    for (int j = 0; j < 4; ++j) dirty |= (d[j] & byte_mask_word(j, blo, bhi)) != 0u;
                    if (dirty) sk[bx] = 0;
                }
            };
            clear(r, x0, 0, n1);
            if (n1 < 16) clear(r + 1, 0, n1, 16);
        }
    }
}

// The flat-word kernel with one thread-block cluster per 16-row band (a
// codec block row): a band's bytes [16 by pw, 16 (by + 1) pw) of each plane
// are pw whole 16-byte words, so the band's SKIP row can be reduced on chip:
// the BAND_CL CTAs of the cluster split the band's words and OR dirty bits
// (per plane and block column) into the leader CTA's shared memory over
// DSMEM; the leader writes the SKIP row once -- no SKIP memset launch and no
// racing byte stores.  Needs h % 16 == 0 (update atlases).
constexpr int BAND_CL = 4;
constexpr int BAND_THREADS = 256;

__global__ void __launch_bounds__(BAND_THREADS) pack_delta_vis_band_kernel(PackArgs a) {
    namespace cg = cooperative_groups;
    extern __shared__ uint32_t s_dirty[];  // [3][ceil(nseg / 32)], used in the leader
    cg::cluster_group cl = cg::this_cluster();
    const uint32_t rank = cl.block_rank();
    const bool key = a.key_dev && *a.key_dev;
    const uint8_t *prev = key ? nullptr : a.prev;
    const uint32_t pw = uint32_t(a.pw), h = uint32_t(a.h);
    const uint32_t T = h * pw;
    const uint32_t nseg = uint32_t(a.nseg), nsw = (nseg + 31) / 32;
    const uint32_t by = blockIdx.x / BAND_CL;
    const bool track = a.skip && prev;
    if (rank == 0 && track)
        for (uint32_t i = threadIdx.x; i < 3 * nsw; i += blockDim.x) s_dirty[i] = 0u;
    cl.sync();
    uint32_t *dirty = cl.map_shared_rank(s_dirty, 0);
    const uint32_t q = (pw + BAND_CL - 1) / BAND_CL;
    const uint32_t w_end = by * pw + min(pw, (rank + 1) * q);
    for (uint32_t W = by * pw + rank * q + threadIdx.x; W < w_end; W += blockDim.x) {
        const uint32_t f0 = 16 * W;
        const uint32_t r = f0 / pw, x0 = f0 - r * pw;
        const int n1 = int(pw - x0 < 16 ? pw - x0 : 16);  // bytes in row r
        // previous planes first: their loads overlap the texel gather
        const bool need_prev = prev && (a.residual || track);
        uint4 pv[3];
#pragma unroll
        for (int e = 0; e < 3; ++e)
            pv[e] = need_prev ? __ldg(reinterpret_cast<const uint4 *>(prev + size_t(e) * T + f0))
                              : make_uint4(0u, 0u, 0u, 0u);
        uint32_t o[3][4];
        vis_segment(a, int(r), int(x0), o);
        if (n1 < 16) {  // the word runs into row r + 1 (same band)
            uint32_t o2[3][4];
            vis_segment(a, int(r) + 1, -n1, o2);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t m = byte_mask_word(j, 0, n1);
#pragma unroll
                for (int e = 0; e < 3; ++e) o[e][j] = (o[e][j] & m) | (o2[e][j] & ~m);
            }
        }
#pragma unroll
        for (int e = 0; e < 3; ++e) {
            const size_t off = size_t(e) * T + f0;
            *reinterpret_cast<uint4 *>(a.cur + off) = make_uint4(o[e][0], o[e][1], o[e][2], o[e][3]);
            if (!prev) {
                if (a.residual)
                    *reinterpret_cast<uint4 *>(a.residual + off) =
                        make_uint4(o[e][0], o[e][1], o[e][2], o[e][3]);
                continue;
            }
            if (!need_prev) continue;
            const uint32_t pw4[4] = {pv[e].x, pv[e].y, pv[e].z, pv[e].w};
            if (a.residual)
                *reinterpret_cast<uint4 *>(a.residual + off) =
                    make_uint4(__vsub4(o[e][0], pw4[0]), __vsub4(o[e][1], pw4[1]),
                               __vsub4(o[e][2], pw4[2]), __vsub4(o[e][3], pw4[3]));
            if (!track) continue;
            uint32_t d[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) d[j] = o[e][j] ^ pw4[j];
            if ((d[0] | d[1] | d[2] | d[3]) == 0u) continue;
            // bytes [lo, hi) of the word: columns xa + (b - lo) of one row
            auto mark = [&](uint32_t xa, int lo, int hi) {
                const uint32_t bxa = xa >> 4, bxb = (xa + uint32_t(hi - lo) - 1) >> 4;
                for (uint32_t bx = bxa; bx <= bxb; ++bx) {
                    const int blo = lo + int(bx * 16 > xa ? bx * 16 - xa : 0);
                    const int bhi = lo + int((bx + 1) * 16 - xa < uint32_t(hi - lo)
                                                 ? (bx + 1) * 16 - xa : uint32_t(hi - lo));
                    bool dv = false;
#pragma unroll
                    for (int j = 0; j < 4; ++j) dv |= (d[j] & byte_mask_word(j, blo, bhi)) != 0u;
                    if (dv) atomicOr(dirty + e * nsw + (bx >> 5), 1u << (bx & 31));
                }
            };
            mark(x0, 0, n1);
            if (n1 < 16) mark(0, n1, 16);
        }
    }
    cl.sync();  // every CTA's dirty bits have landed in the leader
    if (rank != 0 || !a.skip) return;
    // SKIP row `by` of every plane: 1 = block identical to the previous frame
    const uint32_t nby = h / 16;
    for (uint32_t i = threadIdx.x; i < 3 * nseg; i += blockDim.x) {
        const uint32_t e = i / nseg, bx = i - e * nseg;
        const uint8_t sk = track ? uint8_t(((s_dirty[e * nsw + (bx >> 5)] >> (bx & 31)) & 1u) == 0u)
                                 : uint8_t(0);
        a.skip[(size_t(e) * nby + by) * nseg + bx] = sk;
    }
}

// Generic temporal delta over already-packed planes (elements of 1 or 2 B).
template <int EB>
__global__ void __launch_bounds__(TILE_X *TILE_Y)
    delta_kernel(const uint8_t *cur, const uint8_t *prev, int64_t h, int64_t w, int64_t nseg,
                 uint8_t *residual, uint8_t *skip) {
    __shared__ uint32_t dirty[TILE_X];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t seg = int64_t(blockIdx.x) * TILE_X + tx;
    const int64_t by = blockIdx.y;
    const int e = blockIdx.z;
    const int64_t r = by * TILE_Y + ty;
    if (ty == 0) dirty[tx] = 0u;
    __syncthreads();
    if (seg < nseg && r < h && prev) {
        const int64_t base = (int64_t(e) * h + r) * w;
        uint32_t any = 0;
        for (int i = 0; i < SEG; ++i) {
            const int64_t x = seg * SEG + i;
            if (x >= w) break;
            if (EB == 2) {
                uint16_t c = reinterpret_cast<const uint16_t *>(cur)[base + x];
                uint16_t p = reinterpret_cast<const uint16_t *>(prev)[base + x];
                any |= uint32_t(c ^ p);
                if (residual) reinterpret_cast<uint16_t *>(residual)[base + x] = uint16_t(c - p);
            } else {
                uint8_t c = cur[base + x], p = prev[base + x];
                any |= uint32_t(c ^ p);
                if (residual) residual[base + x] = uint8_t(c - p);
            }
        }
        if (any) atomicOr(&dirty[tx], 1u);
    }
    __syncthreads();
    if (skip && ty == 0 && seg < nseg) {
        const int64_t nby = (h + TILE_Y - 1) / TILE_Y;
        skip[(int64_t(e) * nby + by) * nseg + seg] = prev ? uint8_t(dirty[tx] == 0u) : 0;
    }
}

__global__ void unpack_color_kernel(const uint16_t *planes, int64_t n, uint32_t *texels) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        texels[i] = uint32_t(planes[i]) | (uint32_t(planes[n + i]) << 10) |
                    (uint32_t(planes[2 * n + i]) << 20);
    }
}

__global__ void unpack_vis_kernel(const uint8_t *planes, int64_t h, int64_t w, int64_t pw,
                                  uint16_t *texels) {
    const int64_t total = h * w;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = i / w, x = i % w;
        uint8_t s[4];
        for (int k = 0; k < 4; ++k) {
            const int64_t b = 4 * x + k;
            s[k] = planes[((b % 3) * h + r) * pw + b / 3];
        }
        texels[2 * i] = uint16_t((s[0] << 8) | s[1]);
        texels[2 * i + 1] = uint16_t((s[2] << 8) | s[3]);
    }
}

inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int launch_pack_delta(int kind, const void *texels, int64_t h, int64_t w, int64_t row_stride,
                      void *planes_cur, const void *planes_prev, void *residual,
                      uint8_t *skip, cudaStream_t stream, const int32_t *key_dev = nullptr) {
    if (h < 0 || w < 0) fail(PS_ERR_VALUE, "negative texel region shape");
    if (row_stride < w) fail(PS_ERR_VALUE, "row stride smaller than width");
    if (kind != PS_KIND_COLOR && kind != PS_KIND_VISIBILITY) fail(PS_ERR_VALUE, "bad kind");
    PackArgs a;
    a.texels = static_cast<const uint8_t *>(texels);
    a.h = h;
    a.w = w;
    a.row_stride_b = row_stride * 4;
    a.pw = (kind == PS_KIND_COLOR) ? w : (4 * w + 2) / 3;
    a.nseg = ceil_div(a.pw, SEG);
    a.cur = static_cast<uint8_t *>(planes_cur);
    a.prev = static_cast<const uint8_t *>(planes_prev);
    a.residual = static_cast<uint8_t *>(residual);
    a.skip = skip;
    a.key_dev = key_dev;
    a.vec_in = aligned16(texels) && (a.row_stride_b % 16 == 0);
    const int eb = (kind == PS_KIND_COLOR) ? 2 : 1;
    a.vec_out = aligned16(planes_cur) && (!planes_prev || aligned16(planes_prev)) &&
                (!residual || aligned16(residual)) && ((a.pw * eb) % 16 == 0);
    if (h == 0 || a.pw == 0) return PS_OK;
    dim3 block(TILE_X, TILE_Y);
    dim3 grid(unsigned(ceil_div(a.nseg, TILE_X)), unsigned(ceil_div(h, TILE_Y)));
    if (grid.y > 65535u) fail(PS_ERR_VALUE, "plane too tall");
    const bool rows_misaligned = kind == PS_KIND_VISIBILITY && !a.vec_out && a.vec_in &&
                                 aligned16(planes_cur) && (!planes_prev || aligned16(planes_prev)) &&
                                 (!residual || aligned16(residual));
    static const bool funnel = getenv("PS_PACK_FUNNEL") != nullptr;  // tuning: old path
    const bool flat = rows_misaligned && !funnel && (h * a.pw) % 16 == 0 && a.pw >= 16 && a.vec_in &&
                      3 * h * a.pw < (int64_t(1) << 31);
    // one cluster per 16-row band (SKIP reduced on chip) when the bands are
    // whole; PS_PACK_FLAT selects the grid-stride flat kernel (tuning)
    static const bool flat_only = getenv("PS_PACK_FLAT") != nullptr;
    const bool band = !flat_only && h % 16 == 0 && h / 16 * BAND_CL <= 0x7fffffff &&
                      size_t(3) * size_t(ceil_div(a.nseg, 32)) * 4 <= 48 * 1024;
    if (kind == PS_KIND_COLOR) {
        pack_delta_kernel<PS_KIND_COLOR><<<grid, block, 0, stream>>>(a);
    } else if (flat && band) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(h / 16) * BAND_CL);
        cfg.blockDim = dim3(BAND_THREADS);
        cfg.dynamicSmemBytes = size_t(3) * size_t(ceil_div(a.nseg, 32)) * 4;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = BAND_CL;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        check_cuda(cudaLaunchKernelEx(&cfg, pack_delta_vis_band_kernel, a), "launch band kernel");
    } else if (flat) {
        if (skip) {  // SKIP starts at 1 (block identical) and changed bytes clear it
            const int64_t nby = ceil_div(h, TILE_Y);
            check_cuda(cudaMemsetAsync(skip, 1, size_t(3 * nby * a.nseg), stream), "memset skip");
        }
        const int64_t words = h * a.pw / 16;
        const unsigned blocks = unsigned(std::max<int64_t>(
            1, std::min<int64_t>(ceil_div(words, 256), int64_t(sm_count()) * 16)));
        pack_delta_vis_flat_kernel<<<blocks, 256, 0, stream>>>(a);
    } else if (rows_misaligned)
        pack_delta_vis_unaligned_kernel<<<grid, block, 0, stream>>>(a);
    else
        pack_delta_kernel<PS_KIND_VISIBILITY><<<grid, block, 0, stream>>>(a);
    check_launch("pack_delta_kernel");
    return PS_OK;
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" {

const char *ps_last_error(void) { return g_last_error.c_str(); }

int ps_abi_version(void) { return PS_ABI_VERSION; }

int ps_device_sm_count(void) {
    try {
        return sm_count();
    } catch (...) {
        return -1;
    }
}

int64_t ps_widened_width(int64_t w) { return w < 0 ? -1 : (4 * w + 2) / 3; }

int ps_pack_color(const uint32_t *texels, int64_t h, int64_t w, int64_t row_stride,
                  uint16_t *planes, void *stream) {
    PS_ABI_BEGIN
    launch_pack_delta(PS_KIND_COLOR, texels, h, w, row_stride, planes, nullptr, nullptr,
                      nullptr, as_stream(stream));
    PS_ABI_END
}

int ps_pack_visibility(const uint16_t *texels, int64_t h, int64_t w, int64_t row_stride,
                       uint8_t *planes, void *stream) {
    PS_ABI_BEGIN
    launch_pack_delta(PS_KIND_VISIBILITY, texels, h, w, row_stride, planes, nullptr, nullptr,
                      nullptr, as_stream(stream));
    PS_ABI_END
}

int ps_pack_delta(int kind, const void *texels, int64_t h, int64_t w, int64_t row_stride,
                  void *planes_cur, const void *planes_prev, void *residual, uint8_t *skip,
                  const int32_t *key_dev, void *stream) {
    PS_ABI_BEGIN
    launch_pack_delta(kind, texels, h, w, row_stride, planes_cur, planes_prev, residual, skip,
                      as_stream(stream), key_dev);
    PS_ABI_END
}

int ps_temporal_delta(int elem_bytes, const void *cur, const void *prev, int64_t h, int64_t w,
                      void *residual, uint8_t *skip, void *stream) {
    PS_ABI_BEGIN
    if (h < 0 || w < 0) fail(PS_ERR_VALUE, "negative plane shape");
    if (elem_bytes != 1 && elem_bytes != 2) fail(PS_ERR_VALUE, "element bytes must be 1 or 2");
    if (h == 0 || w == 0) return PS_OK;
    const int64_t nseg = ceil_div(w, SEG);
    dim3 block(TILE_X, TILE_Y);
    dim3 grid(unsigned(ceil_div(nseg, TILE_X)), unsigned(ceil_div(h, TILE_Y)), 3);
    auto s = as_stream(stream);
    if (elem_bytes == 2)
        delta_kernel<2><<<grid, block, 0, s>>>(static_cast<const uint8_t *>(cur),
                                                static_cast<const uint8_t *>(prev), h, w, nseg,
                                                static_cast<uint8_t *>(residual), skip);
    else
        delta_kernel<1><<<grid, block, 0, s>>>(static_cast<const uint8_t *>(cur),
                                                static_cast<const uint8_t *>(prev), h, w, nseg,
                                                static_cast<uint8_t *>(residual), skip);
    check_launch("delta_kernel");
    PS_ABI_END
}

int ps_unpack_color(const uint16_t *planes, int64_t h, int64_t w, uint32_t *texels,
                    void *stream) {
    PS_ABI_BEGIN
    if (h < 0 || w < 0) fail(PS_ERR_VALUE, "negative plane shape");
    const int64_t n = h * w;
    if (n == 0) return PS_OK;
    unpack_color_kernel<<<unsigned(std::min<int64_t>(ceil_div(n, 256), 4096)), 256, 0,
                          as_stream(stream)>>>(planes, n, texels);
    check_launch("unpack_color_kernel");
    PS_ABI_END
}

int ps_unpack_visibility(const uint8_t *planes, int64_t h, int64_t w, uint16_t *texels,
                         void *stream) {
    PS_ABI_BEGIN
    if (h < 0 || w < 0) fail(PS_ERR_VALUE, "negative plane shape");
    const int64_t n = h * w;
    if (n == 0) return PS_OK;
    unpack_vis_kernel<<<unsigned(std::min<int64_t>(ceil_div(n, 256), 4096)), 256, 0,
                        as_stream(stream)>>>(planes, h, w, (4 * w + 2) / 3, texels);
    check_launch("unpack_vis_kernel");
    PS_ABI_END
}

}  // extern "C"
