// Stage (3): changed-probe detection (selection.py:284-323) and bitmap
// compaction (np.flatnonzero), sm_100a.
//
// Detection streams both atlases once, in atlas-row order: a CTA owns one
// band of `side` atlas rows (one block row of probes) and 512 consecutive
// texel columns; each thread owns a texel pair (8 bytes, never straddling a
// probe since block sides are even) and ORs its verdict over the band's rows
// with all `side` loads in flight.  Per-probe verdicts are ORed in shared
// memory, ANDed with the active flags and published as a bitmap with one
// atomicOr per 32 probes.  Compaction turns the bitmap into ascending ids
// with a two-kernel count/scan (no host round trip, count stays on device).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>

#include "ps_common.cuh"

namespace ps {
namespace {

constexpr int DET_THREADS = 256;
constexpr int DET_PAIRS = DET_THREADS;  // texel pairs per CTA

enum DetectMode { EXACT = 0, COLOR_CUT = 1, VIS_F32 = 2, VIS_F64 = 3 };

struct DetectArgs {
    const uint2 *a;          // rendered, as texel pairs
    const uint2 *b;          // last_sent
    int64_t pairs_per_row;   // atlas width / 2
    int side;                // block side (10 or 18)
    int64_t ppr;             // probes per row
    int64_t probe_count;
    int64_t probe_begin;     // only probes in [probe_begin, probe_end) are tested
    int64_t probe_end;
    int64_t band0;           // first block row of the range
    const uint8_t *active;   // bool[probe_count] or nullptr (all active)
    uint32_t *bits;          // changed bitmap (zeroed by the launcher)
    uint32_t *const *dst;    // or: publish into these bitmaps (peer memory allowed)
    int ndst;
    int color_cut;           // COLOR_CUT: changed iff max channel delta >= cut
    float thr32;
    double thr64;
};

__device__ __forceinline__ bool color_texel_hit(uint32_t x, uint32_t y, int cut) {
    int dr = abs(int(x & 0x3FFu) - int(y & 0x3FFu));
    int dg = abs(int((x >> 10) & 0x3FFu) - int((y >> 10) & 0x3FFu));
    int db = abs(int((x >> 20) & 0x3FFu) - int((y >> 20) & 0x3FFu));
    return max(dr, max(dg, db)) >= cut;
}

template <int MODE>
__device__ __forceinline__ bool half_hit(uint16_t x, uint16_t y, float t32, double t64) {
    // |f32(a) - f32(b)| computed in float32 exactly as numpy does
    float fx = __half2float(__ushort_as_half(x));
    float fy = __half2float(__ushort_as_half(y));
    float d = fabsf(__fsub_rn(fx, fy));
    bool over = (MODE == VIS_F32) ? (d > t32) : (double(d) > t64);
    return over || (isnan(d) && x != y);
}

template <int MODE>
__device__ __forceinline__ bool word_hit(uint32_t x, uint32_t y, const DetectArgs &a) {
    if (MODE == EXACT) return x != y;
    if (MODE == COLOR_CUT) return color_texel_hit(x, y, a.color_cut);
    return half_hit<MODE>(uint16_t(x), uint16_t(y), a.thr32, a.thr64) ||
           half_hit<MODE>(uint16_t(x >> 16), uint16_t(y >> 16), a.thr32, a.thr64);
}

__device__ __forceinline__ uint2 ldg_stream(const uint2 *p) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];"
                 : "=r"(r.x), "=r"(r.y)
                 : "l"(p));
    return r;
}

template <int MODE, int SIDE>
__global__ void __launch_bounds__(DET_THREADS) detect_kernel(DetectArgs a) {
    __shared__ uint32_t probe_hit[DET_PAIRS * 2 / SIDE + 2];
    const int64_t band = a.band0 + blockIdx.y;
    const int64_t pair0 = int64_t(blockIdx.x) * DET_PAIRS;
    const int64_t col0 = pair0 * 2;               // first texel column of the CTA
    const int64_t bc0 = col0 / SIDE;              // first block column touched
    const int nprobe = int((col0 + 2 * DET_PAIRS - 1) / SIDE - bc0 + 1);
    for (int i = threadIdx.x; i < nprobe; i += DET_THREADS) probe_hit[i] = 0u;
    __syncthreads();

    const int64_t q = pair0 + threadIdx.x;
    if (q < a.pairs_per_row) {
        const int64_t row0 = band * SIDE;
        const uint2 *pa = a.a + row0 * a.pairs_per_row + q;
        const uint2 *pb = a.b + row0 * a.pairs_per_row + q;
        uint2 va[SIDE], vb[SIDE];
#pragma unroll
        for (int r = 0; r < SIDE; ++r) {
            va[r] = ldg_stream(pa + r * a.pairs_per_row);
            vb[r] = ldg_stream(pb + r * a.pairs_per_row);
        }
        bool hit = false;
#pragma unroll
        for (int r = 0; r < SIDE; ++r)
            hit |= word_hit<MODE>(va[r].x, vb[r].x, a) | word_hit<MODE>(va[r].y, vb[r].y, a);
        if (hit) probe_hit[(2 * q) / SIDE - bc0] = 1u;  // benign race: all writers store 1
    }
    __syncthreads();
    // publish: one thread per probe touched by this CTA
    if (!a.dst) {
        for (int i = threadIdx.x; i < nprobe; i += DET_THREADS) {
            const int64_t bc = bc0 + i;
            if (bc >= a.ppr) continue;
            const int64_t p = band * a.ppr + bc;
            if (p < a.probe_begin || p >= a.probe_end || !probe_hit[i]) continue;
            if (a.active && !a.active[p]) continue;
            atomicOr(&a.bits[p >> 5], 1u << (p & 31));
        }
        return;
    }
    // broadcast: the lanes of a bitmap word OR their bits (warp match + reduce) and
    // one lane ORs the word into every destination, peers' bitmaps over NVLink
    for (int i0 = 0; i0 < nprobe; i0 += DET_THREADS) {
        const int i = i0 + threadIdx.x;
        const int64_t bc = bc0 + i;
        const int64_t p = band * a.ppr + bc;
        const bool ok = i < nprobe && bc < a.ppr && p >= a.probe_begin && p < a.probe_end &&
                        probe_hit[i] && (!a.active || a.active[p]);
        const int64_t word = ok ? (p >> 5) : -1;
        const unsigned grp = __match_any_sync(0xffffffffu, word);
        const uint32_t v = __reduce_or_sync(grp, ok ? 1u << (p & 31) : 0u);
        if (ok && (threadIdx.x & 31) == __ffs(grp) - 1)
            for (int d = 0; d < a.ndst; ++d) atomicOr_system(a.dst[d] + word, v);
    }
}

// --- compaction ---------------------------------------------------------------

constexpr int CMP_THREADS = 256;  // words per CTA (8192 probes)

__global__ void __launch_bounds__(CMP_THREADS)
    count_kernel(const uint32_t *bits, int64_t words, int32_t *partial) {
    const int64_t w = int64_t(blockIdx.x) * CMP_THREADS + threadIdx.x;
    int c = (w < words) ? __popc(bits[w]) : 0;
    // block reduce
    __shared__ int red[CMP_THREADS / 32];
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x < 32) {
        int v = threadIdx.x < CMP_THREADS / 32 ? red[threadIdx.x] : 0;
        v = __reduce_add_sync(0xffffffffu, v);
        if (threadIdx.x == 0) partial[blockIdx.x] = v;
    }
}

// mode 0: write ids; mode 1: write (id, aux[id]) pairs (slot entries)
template <int MODE>
__global__ void __launch_bounds__(CMP_THREADS)
    compact_kernel(const uint32_t *bits, int64_t words, int64_t n, const int32_t *partial,
                   int64_t *out, const int32_t *aux, int64_t *out_count) {
    __shared__ int64_t s_base;
    __shared__ int warp_tot[CMP_THREADS / 32];
    if (threadIdx.x < 32) {
        int64_t acc = 0;
        for (int i = threadIdx.x; i < int(blockIdx.x); i += 32) acc += partial[i];
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (threadIdx.x == 0) s_base = acc;
    }
    const int64_t w = int64_t(blockIdx.x) * CMP_THREADS + threadIdx.x;
    uint32_t word = (w < words) ? bits[w] : 0u;
    if (w == words - 1 && (n & 31)) word &= (1u << (n & 31)) - 1u;  // ignore tail bits
    const int c = __popc(word);
    // block exclusive scan of c
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int incl = c;
    for (int o = 1; o < 32; o <<= 1) {
        int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    int wbase = 0;
    for (int i = 0; i < wid; ++i) wbase += warp_tot[i];
    int64_t pos = s_base + wbase + incl - c;
    while (word) {
        const int bit = __ffs(word) - 1;
        word &= word - 1;
        const int64_t id = w * 32 + bit;
        if (MODE == 0) {
            out[pos] = id;
        } else {
            out[2 * pos] = id;
            out[2 * pos + 1] = aux[id];
        }
        ++pos;
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == CMP_THREADS - 1 && out_count) {
        int tot = 0;
        for (int i = 0; i < CMP_THREADS / 32; ++i) tot += warp_tot[i];
        *out_count = s_base + tot;
    }
}

__global__ void ids_to_bits_kernel(const int64_t *ids, const int64_t *n_dev, int64_t n_host,
                                   int64_t probe_count, uint32_t *bits, uint32_t *status) {
    const int64_t n = n_dev ? *n_dev : n_host;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t p = ids[i];
        if (p < 0 || p >= probe_count) {
            if (status) atomicOr(status, PS_DEV_INDEX);
            continue;
        }
        atomicOr(&bits[p >> 5], 1u << (p & 31));
    }
}

}  // namespace

// shared with ps_select.cu
size_t compact_workspace_bytes(int64_t n) {
    const int64_t words = ceil_div(n, 32);
    const int64_t blocks = ceil_div(words, CMP_THREADS);
    return size_t(std::max<int64_t>(blocks, 1)) * sizeof(int32_t) + 256;
}

void compact_bits(const uint32_t *bits, int64_t n, int64_t *out, const int32_t *aux_pairs,
                  int64_t *out_count, void *ws, size_t ws_bytes, cudaStream_t s) {
    const int64_t words = ceil_div(n, 32);
    const int64_t blocks = std::max<int64_t>(ceil_div(words, CMP_THREADS), 1);
    if (ws_bytes < size_t(blocks) * sizeof(int32_t)) fail(PS_ERR_WORKSPACE, "compaction workspace");
    int32_t *partial = static_cast<int32_t *>(ws);
    count_kernel<<<unsigned(blocks), CMP_THREADS, 0, s>>>(bits, words, partial);
    check_launch("count_kernel");
    if (aux_pairs)
        compact_kernel<1><<<unsigned(blocks), CMP_THREADS, 0, s>>>(bits, words, n, partial, out,
                                                                    aux_pairs, out_count);
    else
        compact_kernel<0><<<unsigned(blocks), CMP_THREADS, 0, s>>>(bits, words, n, partial, out,
                                                                    nullptr, out_count);
    check_launch("compact_kernel");
}

void ids_to_bits(const int64_t *ids, const int64_t *n_dev, int64_t n_host, int64_t probe_count,
                 uint32_t *bits, uint32_t *status, cudaStream_t s) {
    const int64_t cap = n_dev ? std::max<int64_t>(n_host, 1) : n_host;
    if (cap <= 0) return;
    const unsigned blocks = unsigned(std::min<int64_t>(ceil_div(cap, 256), 2048));
    ids_to_bits_kernel<<<blocks, 256, 0, s>>>(ids, n_dev, n_host, probe_count, bits, status);
    check_launch("ids_to_bits_kernel");
}

}  // namespace ps

using namespace ps;

static void detect_range_impl(int kind, const void *rendered, const void *last_sent,
                              int64_t probe_count, int64_t probes_per_row, int64_t block_rows,
                              int64_t probe_begin, int64_t probe_end, const uint8_t *active,
                              double threshold, int threshold_is_f64, uint32_t *changed_bits,
                              uint32_t *const *dst, int ndst, cudaStream_t s) {
    if (probe_begin < 0 || probe_end > probe_count || probe_begin > probe_end)
        fail(PS_ERR_INDEX, "probe range outside the volume");
    if (kind != PS_KIND_COLOR && kind != PS_KIND_VISIBILITY) fail(PS_ERR_VALUE, "bad kind");
    if (probe_count < 1) fail(PS_ERR_VALUE, "probe_count must be >= 1");
    if (probes_per_row < 1 || block_rows != ceil_div(probe_count, probes_per_row))
        fail(PS_ERR_LAYOUT, "atlas layout does not match probe count");
    const int side = (kind == PS_KIND_COLOR) ? 10 : 18;
    const int64_t words = ceil_div(probe_count, 32);
    if (!dst) check_cuda(cudaMemsetAsync(changed_bits, 0, size_t(words) * 4, s), "memset bits");

    DetectArgs a;
    a.a = static_cast<const uint2 *>(rendered);
    a.b = static_cast<const uint2 *>(last_sent);
    a.pairs_per_row = probes_per_row * side / 2;
    a.side = side;
    a.ppr = probes_per_row;
    a.probe_count = probe_count;
    a.probe_begin = probe_begin;
    a.probe_end = probe_end;
    a.band0 = probe_begin / probes_per_row;
    a.active = active;
    a.bits = changed_bits;
    a.dst = dst;
    a.ndst = ndst;
    a.color_cut = 1;
    a.thr32 = 0.f;
    a.thr64 = 0.0;
    int mode;
    if (threshold <= 0.0) {
        mode = EXACT;
    } else if (kind == PS_KIND_COLOR) {
        // integer channel delta d (0..1023) compared as float64 `d > thr`
        mode = COLOR_CUT;
        if (std::isnan(threshold) || threshold >= 1023.0)
            a.color_cut = 1024;  // never
        else
            a.color_cut = int(std::floor(threshold)) + 1;
    } else {
        mode = threshold_is_f64 ? VIS_F64 : VIS_F32;
        a.thr32 = float(threshold);  // round-to-nearest, as numpy's weak-scalar cast
        a.thr64 = threshold;
    }
    const int64_t bands = probe_end > probe_begin ? (probe_end - 1) / probes_per_row - a.band0 + 1 : 0;
    if (bands > 65535) fail(PS_ERR_VALUE, "too many block rows");
    dim3 grid(unsigned(ceil_div(a.pairs_per_row, DET_PAIRS)), unsigned(bands));
    if (bands > 0) {
#define PS_DET(M, S) detect_kernel<M, S><<<grid, DET_THREADS, 0, s>>>(a)
    if (side == 10) {
        switch (mode) {
            case EXACT: PS_DET(EXACT, 10); break;
            default: PS_DET(COLOR_CUT, 10); break;
        }
    } else {
        switch (mode) {
            case EXACT: PS_DET(EXACT, 18); break;
            case VIS_F32: PS_DET(VIS_F32, 18); break;
            default: PS_DET(VIS_F64, 18); break;
        }
    }
#undef PS_DET
    check_launch("detect_kernel");
    }
}

extern "C" {

size_t ps_detect_workspace_bytes(int64_t probe_count) {
    return compact_workspace_bytes(std::max<int64_t>(probe_count, 1));
}

size_t ps_compact_workspace_bytes(int64_t probe_count) {
    return compact_workspace_bytes(std::max<int64_t>(probe_count, 1));
}

int ps_detect_changed_bcast(int kind, const void *rendered, const void *last_sent,
                            int64_t probe_count, int64_t probes_per_row, int64_t block_rows,
                            int64_t probe_begin, int64_t probe_end, const uint8_t *active,
                            double threshold, int threshold_is_f64, uint32_t *const *dst_bits,
                            int ndst, void *stream) {
    PS_ABI_BEGIN
    if (!dst_bits || ndst < 1) fail(PS_ERR_VALUE, "need at least one destination bitmap");
    detect_range_impl(kind, rendered, last_sent, probe_count, probes_per_row, block_rows,
                      probe_begin, probe_end, active, threshold, threshold_is_f64, nullptr,
                      dst_bits, ndst, as_stream(stream));
    PS_ABI_END
}

int ps_detect_changed_range(int kind, const void *rendered, const void *last_sent,
                            int64_t probe_count, int64_t probes_per_row, int64_t block_rows,
                            int64_t probe_begin, int64_t probe_end, const uint8_t *active,
                            double threshold, int threshold_is_f64, uint32_t *changed_bits,
                            int64_t *out_ids, int64_t *out_count, void *workspace,
                            size_t workspace_bytes, void *stream) {
    PS_ABI_BEGIN
    auto s = as_stream(stream);
    detect_range_impl(kind, rendered, last_sent, probe_count, probes_per_row, block_rows,
                      probe_begin, probe_end, active, threshold, threshold_is_f64, changed_bits,
                      nullptr, 0, s);
    if (out_ids || out_count)
        compact_bits(changed_bits, probe_count, out_ids, nullptr, out_count, workspace,
                     workspace_bytes, s);
    PS_ABI_END
}

int ps_detect_changed(int kind, const void *rendered, const void *last_sent,
                      int64_t probe_count, int64_t probes_per_row, int64_t block_rows,
                      const uint8_t *active, double threshold, int threshold_is_f64,
                      uint32_t *changed_bits, int64_t *out_ids, int64_t *out_count,
                      void *workspace, size_t workspace_bytes, void *stream) {
    return ps_detect_changed_range(kind, rendered, last_sent, probe_count, probes_per_row,
                                   block_rows, 0, probe_count, active, threshold,
                                   threshold_is_f64, changed_bits, out_ids, out_count, workspace,
                                   workspace_bytes, stream);
}

int ps_ids_to_bits(const int64_t *ids, const int64_t *n_dev, int64_t n_host,
                   int64_t probe_count, uint32_t *bits, uint32_t *status_dev, void *stream) {
    PS_ABI_BEGIN
    ids_to_bits(ids, n_dev, n_host, probe_count, bits, status_dev, as_stream(stream));
    PS_ABI_END
}

int ps_bits_to_ids(const uint32_t *bits, int64_t probe_count, int64_t *out_ids,
                   int64_t *out_count, void *workspace, size_t workspace_bytes, void *stream) {
    PS_ABI_BEGIN
    if (probe_count < 1) fail(PS_ERR_VALUE, "probe_count must be >= 1");
    compact_bits(bits, probe_count, out_ids, nullptr, out_count, workspace, workspace_bytes,
                 as_stream(stream));
    PS_ABI_END
}

}  // extern "C"
