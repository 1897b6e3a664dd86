// Slot assignment straight from a selection bitmap, in two single-pass
// kernels (decoupled look-back scans), for the case the server runs every
// frame: a slot per probe (slot_count >= probe_count), so no eviction is
// reachable and the reference's state machine (packing.py:283-305) reduces to
//
//   new   = selected probes with no cached slot, ascending id;
//   slot(new[k]) = used + k            (the free list pops [used, slot_count)
//                                       in order, packing.py:296-302);
//   last_selected[p] = tick + 1 for every selected p, tick += 1, used += |new|;
//   entries = (slot, probe) for every slot holding a selected probe, by slot.
//
// ps_assign_slots (ps_select.cu) runs the same machine as 16 launches over an
// id list (ids -> bits -> compaction -> plan -> bind -> stamp -> entry bits ->
// compaction); here the selection stays a bitmap:
//
//   bind_kernel    (one pass over the selection words): per 128-probe warp
//                  span, coalesced probe_slot reads -> ballot masks of new
//                  probes; warp / block / cross-tile (look-back) prefix of
//                  (selected, new) counts; then new ids, both slot maps and
//                  the stamps are written coalesced; the last tile publishes
//                  the plan and advances (tick, used);
//   entries_kernel (one pass over the slots): slot_probe + selection bit ->
//                  ballot masks -> the same prefix -> (slot, probe) pairs.
//
// Workspace: one 64-bit status word per tile of each kernel plus two tile
// counters, zeroed by one memset per call (graph-replay safe).
#include <cuda_runtime.h>

#include "ps_common.cuh"

namespace ps {
namespace {

constexpr int AS_THREADS = 256;                 // 8 warps
constexpr int AS_WARPS = AS_THREADS / 32;
// bitmap words per warp (PS_AS_SPAN_WORDS, tuning): 4 words = 128 probes per
// warp puts 128 CTAs on the GPU at C4 instead of 16 with 1,024-probe spans
// (C5 N=131,072 graphed chains, spans of 32 / 8 / 4 words: colour 0.134 /
// 0.129 / 0.125 ms, visibility 0.293 / 0.287 / 0.284 ms)
#ifndef PS_AS_SPAN_WORDS
#define PS_AS_SPAN_WORDS 4
#endif
constexpr int SPAN_WORDS = PS_AS_SPAN_WORDS;
static_assert(SPAN_WORDS >= 1 && SPAN_WORDS <= 32, "span words");
constexpr int64_t AS_SPAN = 32 * SPAN_WORDS;    // probes (or slots) per warp
constexpr int64_t AS_TILE = AS_SPAN * AS_WARPS;  // 1,024 per CTA tile

constexpr uint64_t FLAG_AGG = 1ull << 62, FLAG_PREFIX = 2ull << 62;
constexpr uint64_t VAL_MASK = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t ld_acq(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel(uint64_t *p, uint64_t v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// exclusive prefix of this tile, computed by warp 0 (every lane must call):
// the tile publishes its aggregate, then the warp reads up to 32 predecessors'
// status words at once and sums back to the nearest published prefix -- one
// L2 round trip per 32 tiles instead of one per tile.  Values are packed pairs
// (hi << 31 | lo) that add without carrying between the halves (< 2^31 each).
__device__ uint64_t look_back(uint64_t *status, int64_t tile, uint64_t agg) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) st_rel(status, FLAG_PREFIX | agg);
        return 0;
    }
    if (lane == 0) st_rel(status + tile, FLAG_AGG | agg);
    uint64_t excl = 0;
    for (int64_t base = tile - 1;; base -= 32) {
        const int64_t j = base - lane;
        uint64_t v = FLAG_PREFIX;  // before tile 0: an empty prefix
        if (j >= 0)
            while (((v = ld_acq(status + j)) >> 62) == 0) __nanosleep(32);
        const unsigned pre = __ballot_sync(0xffffffffu, (v >> 62) == 2);
        const int stop = pre ? __ffs(pre) - 1 : 31;  // nearest published prefix
        uint64_t x = lane <= stop ? (v & VAL_MASK) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        excl += x;
        if (pre) break;
    }
    if (lane == 0) st_rel(status + tile, FLAG_PREFIX | (excl + agg));
    return excl;
}

__device__ __forceinline__ uint64_t pack2(uint64_t hi, uint64_t lo) { return (hi << 31) | lo; }

// block-wide exclusive scan of one packed value per warp; returns this warp's
// offset inside the tile and the tile total (smem-broadcast)
__device__ __forceinline__ uint64_t warp_offsets(uint64_t mine, uint64_t *s_warp, uint64_t &total) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) s_warp[warp] = mine;
    __syncthreads();
    uint64_t off = 0, tot = 0;
    for (int w = 0; w < AS_WARPS; ++w) {
        const uint64_t v = s_warp[w];
        if (w < warp) off += v;
        tot += v;
    }
    total = tot;
    return off;
}

// tile ids in launch order from a counter, so a tile's predecessors are running
__device__ __forceinline__ int64_t claim_tile(unsigned long long *counter) {
    __shared__ int64_t s_tile;
    if (threadIdx.x == 0) s_tile = int64_t(atomicAdd(counter, 1ull));
    __syncthreads();
    return s_tile;
}

__global__ void __launch_bounds__(AS_THREADS)
    bind_kernel(const uint32_t *sel_bits, const uint32_t *pvs_bits, int64_t n, int64_t ntiles,
                int32_t *probe_slot, int32_t *slot_probe, int64_t *last_selected, int64_t *meta,
                int64_t *new_ids, int64_t *plan, int64_t *sel_count_out, uint64_t *status,
                unsigned long long *counter) {
    __shared__ uint64_t s_warp[AS_WARPS];
    __shared__ uint64_t s_base;
    const int64_t tile = claim_tile(counter);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t used = meta[1], tick = meta[0] + 1;  // read before this tile publishes
    const int64_t span0 = tile * AS_TILE + int64_t(warp) * AS_SPAN;
    const int64_t words = (n + 31) / 32;
    // lane b holds word b of this warp's span: selection and new-probe masks
    uint32_t selw = 0, neww = 0;
    if (lane < SPAN_WORDS) {
        const int64_t w = span0 / 32 + lane;
        if (w < words) {
            selw = sel_bits[w];
            if (pvs_bits) selw &= pvs_bits[w];
            if (w == words - 1 && (n & 31)) selw &= (1u << (n & 31)) - 1u;
        }
    }
#pragma unroll
    for (int b = 0; b < SPAN_WORDS; ++b) {
        const uint32_t sw = __shfl_sync(0xffffffffu, selw, b);
        const int64_t p = span0 + b * 32 + lane;
        const bool sel = (sw >> lane) & 1u;
        const bool is_new = sel && probe_slot[p] < 0;
        const uint32_t m = __ballot_sync(0xffffffffu, is_new);
        if (lane == b) neww = m;
    }
    const uint64_t mine = pack2(__reduce_add_sync(0xffffffffu, __popc(selw)),
                                __reduce_add_sync(0xffffffffu, __popc(neww)));
    uint64_t tile_total;
    const uint64_t woff = warp_offsets(mine, s_warp, tile_total);
    if (threadIdx.x < 32) {
        const uint64_t excl = look_back(status, tile, tile_total);
        if (threadIdx.x == 0) s_base = excl;
        if (threadIdx.x == 0 && tile == ntiles - 1) {  // totals: plan (plan_kernel layout) + meta
            const uint64_t all = excl + tile_total;
            const int64_t sc = int64_t(all >> 31), nc = int64_t(all & 0x7fffffffu);
            plan[0] = sc;
            plan[1] = nc;
            plan[2] = nc;
            plan[3] = 0;
            plan[4] = 0;
            plan[5] = used;
            plan[6] = tick;
            meta[0] = tick;
            meta[1] = used + nc;
            if (sel_count_out) *sel_count_out = sc;
        }
    }
    __syncthreads();
    int64_t rank = int64_t((s_base + woff) & 0x7fffffffu);  // new probes before this warp
    for (int b = 0; b < SPAN_WORDS; ++b) {
        const uint32_t nm = __shfl_sync(0xffffffffu, neww, b);
        const uint32_t sm = __shfl_sync(0xffffffffu, selw, b);
        const int64_t p = span0 + b * 32 + lane;
        if ((sm >> lane) & 1u) last_selected[p] = tick;  // packing.py:303-304
        if ((nm >> lane) & 1u) {
            const int64_t k = rank + __popc(nm & ((1u << lane) - 1u));
            const int64_t slot = used + k;  // the free list's next slot
            new_ids[k] = p;
            probe_slot[p] = int32_t(slot);
            slot_probe[slot] = int32_t(p);
        }
        rank += __popc(nm);
    }
}

__global__ void __launch_bounds__(AS_THREADS)
    entries_kernel(const int32_t *slot_probe, const uint32_t *sel_bits, const uint32_t *pvs_bits,
                   int64_t n, int64_t slot_count, int64_t ntiles, int64_t *entries,
                   int64_t *entry_count, uint64_t *status, unsigned long long *counter) {
    __shared__ uint64_t s_warp[AS_WARPS];
    __shared__ uint64_t s_base;
    const int64_t tile = claim_tile(counter);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t span0 = tile * AS_TILE + int64_t(warp) * AS_SPAN;
    uint32_t emask = 0;
    int32_t q[SPAN_WORDS];
#pragma unroll
    for (int b = 0; b < SPAN_WORDS; ++b) {
        const int64_t s = span0 + b * 32 + lane;
        q[b] = s < slot_count ? slot_probe[s] : -1;
    }
#pragma unroll
    for (int b = 0; b < SPAN_WORDS; ++b) {
        bool hit = false;
        if (q[b] >= 0 && q[b] < n) {
            uint32_t w = sel_bits[q[b] >> 5];
            if (pvs_bits) w &= pvs_bits[q[b] >> 5];
            hit = (w >> (q[b] & 31)) & 1u;
        }
        const uint32_t m = __ballot_sync(0xffffffffu, hit);
        if (lane == b) emask = m;
    }
    const uint64_t mine = __reduce_add_sync(0xffffffffu, __popc(emask));
    uint64_t tile_total;
    const uint64_t woff = warp_offsets(mine, s_warp, tile_total);
    if (threadIdx.x < 32) {
        const uint64_t excl = look_back(status, tile, tile_total);
        if (threadIdx.x == 0) {
            s_base = excl;
            if (tile == ntiles - 1) *entry_count = int64_t(excl + tile_total);
        }
    }
    __syncthreads();
    int64_t rank = int64_t(s_base + woff);
#pragma unroll
    for (int b = 0; b < SPAN_WORDS; ++b) {
        const uint32_t m = __shfl_sync(0xffffffffu, emask, b);
        if ((m >> lane) & 1u) {
            const int64_t k = rank + __popc(m & ((1u << lane) - 1u));
            entries[2 * k] = span0 + b * 32 + lane;
            entries[2 * k + 1] = q[b];
        }
        rank += __popc(m);
    }
}

struct BitsWs {
    uint64_t *status_bind, *status_entries;
    unsigned long long *counters;
    int64_t *new_ids;
    size_t zero_bytes;
    size_t total;
};

BitsWs carve_bits(void *ws, size_t cap, int64_t n, int64_t sc) {
    Carver c(ws, cap);
    BitsWs w;
    const int64_t tb = ceil_div(std::max<int64_t>(n, 1), AS_TILE);
    const int64_t te = ceil_div(std::max<int64_t>(sc, 1), AS_TILE);
    // status words and counters are contiguous: one memset zeroes them
    w.counters = c.take<unsigned long long>(2);
    w.status_bind = reinterpret_cast<uint64_t *>(c.base ? c.base + c.off : nullptr);
    c.off += size_t(tb) * 8;
    w.status_entries = reinterpret_cast<uint64_t *>(c.base ? c.base + c.off : nullptr);
    c.off += size_t(te) * 8;
    w.zero_bytes = 16 + size_t(tb + te) * 8;
    w.new_ids = c.take<int64_t>(size_t(std::max<int64_t>(n, 1)));
    c.take<char>(1);
    w.total = c.off;
    if (ws) c.check();
    return w;
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" {

size_t ps_assign_bits_workspace_bytes(int64_t probe_count, int64_t slot_count) {
    return carve_bits(nullptr, 0, std::max<int64_t>(probe_count, 1),
                      std::max<int64_t>(slot_count, 1)).total + 256;
}

int ps_assign_slots_bits(const uint32_t *sel_bits, const uint32_t *pvs_bits, int64_t probe_count,
                         int64_t slot_count, int32_t *probe_slot, int32_t *slot_probe,
                         int64_t *last_selected, int64_t *meta, int64_t *entries,
                         int64_t *entry_count, int64_t *plan, int64_t *sel_count,
                         void *workspace, size_t workspace_bytes, void *stream) {
    PS_ABI_BEGIN
    if (probe_count < 1) fail(PS_ERR_VALUE, "probe_count must be >= 1");
    if (slot_count < probe_count)
        fail(PS_ERR_VALUE, "ps_assign_slots_bits needs slot_count >= probe_count (no eviction); "
                           "use ps_assign_slots");
    if (probe_count >= (int64_t(1) << 31)) fail(PS_ERR_VALUE, "probe_count must be < 2^31");
    if (!sel_bits || !probe_slot || !slot_probe || !last_selected || !meta || !entries ||
        !entry_count || !plan)
        fail(PS_ERR_VALUE, "null argument");
    if (workspace_bytes < ps_assign_bits_workspace_bytes(probe_count, slot_count))
        fail(PS_ERR_WORKSPACE, "assign workspace too small");
    auto s = as_stream(stream);
    BitsWs w = carve_bits(workspace, workspace_bytes, probe_count, slot_count);
    check_cuda(cudaMemsetAsync(w.counters, 0, w.zero_bytes, s), "memset");
    const int64_t tb = ceil_div(probe_count, AS_TILE);
    // the last tile's span may run past probe_count: every probe_slot /
    // last_selected access there is guarded by the (tail-masked) selection bit
    bind_kernel<<<unsigned(tb), AS_THREADS, 0, s>>>(sel_bits, pvs_bits, probe_count, tb,
                                                    probe_slot, slot_probe, last_selected, meta,
                                                    w.new_ids, plan, sel_count, w.status_bind,
                                                    w.counters);
    check_launch("bind_kernel(bits)");
    // only slots [0, used) can hold a probe; used <= probe_count
    const int64_t te = ceil_div(std::min<int64_t>(slot_count, probe_count), AS_TILE);
    entries_kernel<<<unsigned(te), AS_THREADS, 0, s>>>(slot_probe, sel_bits, pvs_bits,
                                                       probe_count,
                                                       std::min<int64_t>(slot_count, probe_count),
                                                       te, entries, entry_count,
                                                       w.status_entries, w.counters + 1);
    check_launch("entries_kernel");
    PS_ABI_END
}

}  // extern "C"
