// Stage (3) tail + stage (4) head: budgeted selection (selection.py:413-437),
// the update-atlas slot cache (packing.py:243-317) restated as scan + sort,
// and the update-atlas build with server commit (packing.py:320-338,
// SPEC.md:341).  Everything is stream-ordered with device-resident counts,
// so a whole frame needs no host round trip.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "ps_common.cuh"

namespace ps {

size_t compact_workspace_bytes(int64_t n);
void compact_bits(const uint32_t *bits, int64_t n, int64_t *out, const int32_t *aux_pairs,
                  int64_t *out_count, void *ws, size_t ws_bytes, cudaStream_t s);
void ids_to_bits(const int64_t *ids, const int64_t *n_dev, int64_t n_host, int64_t probe_count,
                 uint32_t *bits, uint32_t *status, cudaStream_t s);

namespace {

constexpr int64_t KEY_PAD = INT64_MAX;

size_t sort_temp_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int64_t *)nullptr, (int64_t *)nullptr,
                                    (const int64_t *)nullptr, (int64_t *)nullptr, int(n));
    return bytes;
}

// candidates = changed & pvs & active, one thread per 32-probe word
__global__ void candidate_kernel(const uint32_t *changed, const uint32_t *pvs,
                                 const uint8_t *active, int64_t n, uint32_t *out) {
    const int64_t words = (n + 31) / 32;
    for (int64_t w = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; w < words;
         w += int64_t(gridDim.x) * blockDim.x) {
        uint32_t m = changed[w];
        if (pvs) m &= pvs[w];
        if (active) {
            uint32_t act = 0;
            for (int b = 0; b < 32; ++b) {
                const int64_t p = w * 32 + b;
                if (p < n && active[p]) act |= 1u << b;
            }
            m &= act;
        }
        if (w == words - 1 && (n & 31)) m &= (1u << (n & 31)) - 1u;
        out[w] = m;
    }
}

// sort keys: staleness order == ascending last_sent_seq (current_seq is a
// common offset), ties by id via the stable sort over ascending ids.
__global__ void select_keys_kernel(const int64_t *ids, const int64_t *count,
                                   const int64_t *last_sent_seq, int64_t n, int64_t *keys,
                                   int64_t *vals) {
    const int64_t c = *count;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        if (i < c) {
            const int64_t p = ids[i];
            keys[i] = last_sent_seq[p];
            vals[i] = p;
        } else {
            keys[i] = KEY_PAD;
            vals[i] = -1;
        }
    }
}

__global__ void budget_kernel(const int64_t *count, int has_budget, int64_t budget,
                              int64_t *out_count) {
    int64_t c = *count;
    if (has_budget) {
        if (budget >= 0)
            c = c < budget ? c : budget;
        else
            c = (c + budget) > 0 ? (c + budget) : 0;  // python slice ids[:budget]
    }
    *out_count = c;
}

// --- slot cache ----------------------------------------------------------------
// meta (persistent, device): [0] tick, [1] used
// plan (per call, device):   [0] sel_count, [1] new_count, [2] F, [3] need,
//                            [4] abort, [5] old_used, [6] tick

__global__ void new_bits_kernel(const uint32_t *sel_bits, const int32_t *probe_slot, int64_t n,
                                uint32_t *new_bits) {
    const int64_t words = (n + 31) / 32;
    for (int64_t w = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; w < words;
         w += int64_t(gridDim.x) * blockDim.x) {
        uint32_t m = sel_bits[w], out = 0;
        while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1;
            if (probe_slot[w * 32 + b] < 0) out |= 1u << b;
        }
        new_bits[w] = out;
    }
}

__global__ void plan_kernel(const int64_t *sel_count, const int64_t *new_count,
                            const uint32_t *status, int64_t slot_count, int64_t *meta,
                            int64_t *plan, uint32_t *status_out) {
    const int64_t sc = *sel_count, nc = *new_count;
    const int64_t used = meta[1];
    int64_t abort = 0;
    if (status && (*status & PS_DEV_INDEX)) {
        abort = 1;  // ids outside the volume: reject before any mutation
        if (status_out) atomicOr(status_out, PS_DEV_INDEX);
    }
    if (sc > slot_count) {
        abort = 1;
        if (status_out) atomicOr(status_out, PS_DEV_SLOT_OVERFLOW);
    }
    const int64_t free_slots = slot_count - used;
    const int64_t f = nc < free_slots ? nc : free_slots;
    plan[0] = sc;
    plan[1] = nc;
    plan[2] = f;
    plan[3] = abort ? 0 : nc - f;
    plan[4] = abort;
    plan[5] = used;
    if (!abort) {
        meta[0] += 1;  // tick (packing.py:292)
        meta[1] = used + f;
    }
    plan[6] = meta[0];
}

// eviction candidates: cached probes outside the selection, keyed by
// (last_selected, slot) -- slot order comes from the stable sort (packing.py:308-312)
__global__ void victim_keys_kernel(const int32_t *slot_probe, const int64_t *last_selected,
                                   const uint32_t *sel_bits, const int64_t *plan,
                                   int64_t slot_count, int64_t *keys, int64_t *vals) {
    const int64_t used = plan[5];
    for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < slot_count;
         s += int64_t(gridDim.x) * blockDim.x) {
        int64_t key = KEY_PAD;
        if (s < used) {
            const int32_t q = slot_probe[s];
            if (q >= 0 && !((sel_bits[q >> 5] >> (q & 31)) & 1u)) key = last_selected[q];
        }
        keys[s] = key;
        vals[s] = s;
    }
}

__global__ void bind_kernel(const int64_t *new_ids, const int64_t *victims, const int64_t *plan,
                            int32_t *probe_slot, int32_t *slot_probe) {
    if (plan[4]) return;
    const int64_t nc = plan[1], f = plan[2], used = plan[5];
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nc;
         k += int64_t(gridDim.x) * blockDim.x) {
        const int64_t p = new_ids[k];
        int64_t slot;
        if (k < f) {
            slot = used + k;
        } else {
            slot = victims[k - f];
            const int32_t q = slot_probe[slot];
            if (q >= 0) probe_slot[q] = -1;
        }
        probe_slot[p] = int32_t(slot);
        slot_probe[slot] = int32_t(p);
    }
}

__global__ void stamp_kernel(const int64_t *sel_ids, const int64_t *plan, int64_t *last_selected) {
    if (plan[4]) return;
    const int64_t c = plan[0], tick = plan[6];
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < c;
         i += int64_t(gridDim.x) * blockDim.x)
        last_selected[sel_ids[i]] = tick;
}

// bitmap over slots holding a selected probe (entries sorted by slot)
__global__ void entry_bits_kernel(const int32_t *slot_probe, const uint32_t *sel_bits,
                                  const int64_t *plan, int64_t slot_count, uint32_t *slot_bits) {
    const int64_t words = (slot_count + 31) / 32;
    const bool abort = plan[4] != 0;
    for (int64_t w = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; w < words;
         w += int64_t(gridDim.x) * blockDim.x) {
        uint32_t m = 0;
        if (!abort)
            for (int b = 0; b < 32; ++b) {
                const int64_t s = w * 32 + b;
                if (s >= slot_count) break;
                const int32_t q = slot_probe[s];
                if (q >= 0 && ((sel_bits[q >> 5] >> (q & 31)) & 1u)) m |= 1u << b;
            }
        slot_bits[w] = m;
    }
}

// --- build + commit --------------------------------------------------------------

// visibility (SIDE 18) at <= 80 registers: 24 warps per SM keep more block
// loads in flight than 16 at 102 registers (0.157 -> 0.127 ms at C4);
// colour keeps its 64
template <int SIDE>
__global__ void __launch_bounds__(256, SIDE == 18 ? 3 : 4)
    build_kernel(const uint32_t *src, int64_t src_w, int64_t ppr, const int64_t *entries,
                 const int64_t *entry_count, int64_t slots_per_row, uint32_t *dst,
                 int64_t dst_w, uint32_t *last_sent, int64_t *last_sent_seq,
                 int64_t current_seq, const int64_t *seq_dev) {
    constexpr int CORE = SIDE - 2;
    const int64_t count = *entry_count;
    if (seq_dev) current_seq = *seq_dev;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    // probe ids and slots are < 2^31: 32-bit divisions (a 64-bit division is a
    // ~70-instruction software sequence, four of them per entry dominated the
    // kernel's instruction count)
    const uint32_t ppr32 = uint32_t(ppr), spr32 = uint32_t(slots_per_row);
    for (int64_t e = warp; e < count; e += nwarps) {
        const uint32_t slot = uint32_t(entries[2 * e]), p = uint32_t(entries[2 * e + 1]);
        const uint32_t py = p / ppr32, sy_ = slot / spr32;
        const int64_t y0 = int64_t(py) * SIDE, x0 = int64_t(p - py * ppr32) * SIDE;
        const int64_t sy = int64_t(sy_) * CORE, sx = int64_t(slot - sy_ * spr32) * CORE;
        warp_copy_block<SIDE>(src, src_w, y0, x0, lane, last_sent, [&](int r, int c, uint32_t v) {
            dst[(sy + r) * dst_w + sx + c] = v;
        });
        if (lane == 0 && last_sent_seq) last_sent_seq[p] = current_seq;
    }
}

// ENT entries per warp iteration: all ENT blocks' loads are issued before the
// first store, so a warp keeps ENT x SIDE^2 / 32 loads per lane in flight
// (the colour blocks are small: one entry is 4 loads per lane)
template <int SIDE, int ENT, int MINB = 4>
__global__ void __launch_bounds__(256, MINB)
    build_multi_kernel(const uint32_t *src, int64_t src_w, int64_t ppr, const int64_t *entries,
                       const int64_t *entry_count, int64_t slots_per_row, uint32_t *dst,
                       int64_t dst_w, uint32_t *last_sent, int64_t *last_sent_seq,
                       int64_t current_seq, const int64_t *seq_dev) {
    constexpr int CORE = SIDE - 2, WORDS = SIDE * SIDE, NW = (WORDS + 31) / 32;
    const int64_t count = *entry_count;
    if (seq_dev) current_seq = *seq_dev;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    const uint32_t ppr32 = uint32_t(ppr), spr32 = uint32_t(slots_per_row);
    const int w32 = int(src_w);
    for (int64_t e0 = warp * ENT; e0 < count; e0 += nwarps * ENT) {
        uint32_t v[ENT][NW];
        int64_t base[ENT];
#pragma unroll
        for (int u = 0; u < ENT; ++u) {
            const int64_t e = e0 + u;
            base[u] = -1;
            if (e < count) {
                const uint32_t p = uint32_t(entries[2 * e + 1]), py = p / ppr32;
                base[u] = int64_t(py) * SIDE * src_w + int64_t(p - py * ppr32) * SIDE;
#pragma unroll
                for (int j = 0; j < NW; ++j) {
                    const int k = lane + 32 * j;
                    if (k < WORDS) v[u][j] = __ldg(src + base[u] + (k / SIDE) * w32 + k % SIDE);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < ENT; ++u) {
            const int64_t e = e0 + u;
            if (base[u] < 0) continue;
            const uint32_t slot = uint32_t(entries[2 * e]), sr = slot / spr32;
            const int64_t sbase = int64_t(sr) * CORE * dst_w + int64_t(slot - sr * spr32) * CORE;
#pragma unroll
            for (int j = 0; j < NW; ++j) {
                const int k = lane + 32 * j;
                if (k < WORDS) {
                    const int r = k / SIDE, c = k % SIDE;
                    if (r >= 1 && r <= CORE && c >= 1 && c <= CORE)
                        dst[sbase + (r - 1) * dst_w + (c - 1)] = v[u][j];
                    if (last_sent) last_sent[base[u] + r * w32 + c] = v[u][j];
                }
            }
            if (lane == 0 && last_sent_seq) last_sent_seq[entries[2 * e + 1]] = current_seq;
        }
    }
}

// Build through shared memory: each warp keeps BUILD_DEPTH blocks in flight
// with 8-byte cp.async copies (a block row is 4 * SIDE bytes at an 8-byte
// aligned offset: 5 / 9 copies per row), so a warp's loads no longer live in
// registers and an SM keeps ~4x more bytes in flight than the register
// version (whose 24 resident warps held one block each).  Once a block has
// landed the warp writes its core to the slot and commits the whole block.
constexpr int BUILD_DEPTH = 4;

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit_group() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int SIDE>
__global__ void __launch_bounds__(256)
    build_async_kernel(const uint32_t *src, int64_t src_w, int64_t ppr, const int64_t *entries,
                       const int64_t *entry_count, int64_t slots_per_row, uint32_t *dst,
                       int64_t dst_w, uint32_t *last_sent, int64_t *last_sent_seq,
                       int64_t current_seq, const int64_t *seq_dev) {
    constexpr int CORE = SIDE - 2, HALF = SIDE / 2, PAIRS = SIDE * HALF, WORDS = SIDE * SIDE;
    __shared__ __align__(16) uint2 ring[8][BUILD_DEPTH][PAIRS];
    const int64_t count = *entry_count;
    if (seq_dev) current_seq = *seq_dev;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    uint2(*my)[PAIRS] = ring[wib];
    auto issue = [&](int64_t e, int slot) {
        if (e < count) {
            const int64_t p = entries[2 * e + 1];
            const uint2 *sb = reinterpret_cast<const uint2 *>(src + (p / ppr) * SIDE * src_w +
                                                              (p % ppr) * SIDE);
            const int64_t wp = src_w / 2;  // row stride in pairs (src_w is even: ppr * SIDE)
            for (int k = lane; k < PAIRS; k += 32) cp_async8(&my[slot][k], sb + (k / HALF) * wp + k % HALF);
        }
        cp_async_commit_group();
    };
#pragma unroll
    for (int d = 0; d < BUILD_DEPTH - 1; ++d) issue(warp + d * nwarps, d);
    int slot = 0;
    for (int64_t e = warp; e < count; e += nwarps) {
        issue(e + (BUILD_DEPTH - 1) * nwarps, (slot + BUILD_DEPTH - 1) % BUILD_DEPTH);
        cp_async_wait_group<BUILD_DEPTH - 1>();
        __syncwarp();
        const int64_t s_ = entries[2 * e], p = entries[2 * e + 1];
        const uint32_t *blk = reinterpret_cast<const uint32_t *>(my[slot]);
        int64_t y0, x0;
        block_origin(p, ppr, SIDE, y0, x0);
        int64_t sy, sx;
        block_origin(s_, slots_per_row, CORE, sy, sx);
        for (int k = lane; k < CORE * CORE; k += 32) {
            const int r = k / CORE, c = k % CORE;
            dst[(sy + r) * dst_w + sx + c] = blk[(r + 1) * SIDE + c + 1];
        }
        if (last_sent) {
            uint2 *ls = reinterpret_cast<uint2 *>(last_sent + y0 * src_w + x0);
            const int64_t wp = src_w / 2;
            for (int k = lane; k < PAIRS; k += 32) ls[(k / HALF) * wp + k % HALF] = my[slot][k];
        }
        if (lane == 0 && last_sent_seq) last_sent_seq[p] = current_seq;
        __syncwarp();  // the slot is refilled by the next iteration's issue
        slot = (slot + 1) % BUILD_DEPTH;
        (void)WORDS;
    }
    cp_async_wait_group<0>();
}

// slab-sharded build: export own probes' cores into a per-rank payload
template <int SIDE>
__global__ void __launch_bounds__(256)
    export_kernel(const uint32_t *src, int64_t src_w, int64_t ppr, const int64_t *entries,
                  const int64_t *entry_count, int64_t probe_begin, int64_t probe_end,
                  uint32_t *payload, uint32_t *last_sent, int64_t *last_sent_seq,
                  int64_t current_seq, const int64_t *seq_dev) {
    constexpr int CORE = SIDE - 2;
    const int64_t count = *entry_count;
    if (seq_dev) current_seq = *seq_dev;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t e = warp; e < count; e += nwarps) {
        const int64_t p = entries[2 * e + 1];
        if (lane == 0 && last_sent_seq) last_sent_seq[p] = current_seq;  // replicated stamp
        if (p < probe_begin || p >= probe_end) continue;
        int64_t y0, x0;
        block_origin(p, ppr, SIDE, y0, x0);
        uint32_t *dst = payload + (p - probe_begin) * (CORE * CORE);
        warp_copy_block<SIDE>(src, src_w, y0, x0, lane, last_sent,
                              [&](int r, int c, uint32_t v) { dst[r * CORE + c] = v; });
    }
}

// encoder rank: gathered payloads -> slot regions of the update atlas
template <int CORE>
__global__ void __launch_bounds__(256)
    import_kernel(const uint32_t *payloads, int64_t payload_stride, const int64_t *rank_begin,
                  int world, const int64_t *entries, const int64_t *entry_count,
                  int64_t slots_per_row, uint32_t *dst, int64_t dst_w) {
    __shared__ int64_t s_begin[65];
    for (int i = threadIdx.x; i <= world; i += blockDim.x) s_begin[i] = rank_begin[i];
    __syncthreads();
    const int64_t count = *entry_count;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t e = warp; e < count; e += nwarps) {
        const int64_t slot = entries[2 * e], p = entries[2 * e + 1];
        int r = 0;
        while (r + 1 < world && p >= s_begin[r + 1]) ++r;
        const uint32_t *srcp = payloads + (int64_t(r) * payload_stride + (p - s_begin[r])) * (CORE * CORE);
        int64_t sy, sx;
        block_origin(slot, slots_per_row, CORE, sy, sx);
#pragma unroll 4
        for (int k = lane; k < CORE * CORE; k += 32) {
            const int rr = k / CORE, cc = k % CORE;
            dst[(sy + rr) * dst_w + sx + cc] = srcp[k];
        }
    }
}

// probe index buffer: count, then per entry the slot delta
// and the zig-zag probe delta as LEB128 varints (pass 1: byte counts)
__device__ __forceinline__ int ib_vlen(uint64_t v) {
    int n = 1;
    while (v >= 128) {
        v >>= 7;
        ++n;
    }
    return n;
}

__device__ __forceinline__ void ib_deltas(const int64_t *entries, int64_t e, uint64_t &ds,
                                          uint64_t &dp) {
    const int64_t ps = e ? entries[2 * (e - 1)] : 0, pp = e ? entries[2 * (e - 1) + 1] : 0;
    ds = uint64_t(entries[2 * e] - ps);
    const int64_t d = entries[2 * e + 1] - pp;
    dp = (uint64_t(d) << 1) ^ uint64_t(d >> 63);
}

__global__ void index_len_kernel(const int64_t *entries, const int64_t *count, int64_t cap,
                                 uint32_t *lens) {
    const int64_t c = *count;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < cap;
         e += int64_t(gridDim.x) * blockDim.x) {
        if (e >= c) {
            lens[e] = 0;
            continue;
        }
        uint64_t ds, dp;
        ib_deltas(entries, e, ds, dp);
        lens[e] = uint32_t(ib_vlen(ds) + ib_vlen(dp));
    }
}

__device__ __forceinline__ int ib_put(uint8_t *dst, uint64_t v) {
    int k = 0;
    while (v >= 128) {
        dst[k++] = uint8_t(v | 0x80);
        v >>= 7;
    }
    dst[k++] = uint8_t(v);
    return k;
}

__global__ void index_write_kernel(const int64_t *entries, const int64_t *count,
                                   const uint64_t *offsets, const uint32_t *lens, int64_t cap,
                                   uint8_t *out, int64_t *out_len) {
    const int64_t c = *count;
    const int head = ib_vlen(uint64_t(c));
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < c;
         e += int64_t(gridDim.x) * blockDim.x) {
        uint64_t ds, dp;
        ib_deltas(entries, e, ds, dp);
        uint8_t *d = out + head + offsets[e];
        d += ib_put(d, ds);
        ib_put(d, dp);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ib_put(out, uint64_t(c));
        *out_len = head + (c ? int64_t(offsets[c - 1] + lens[c - 1]) : 0);
    }
}

// guard band of every probe block from its core (packing.py:180-196)
template <int SIDE>
__global__ void guard_kernel(uint32_t *atlas, int64_t w, int64_t ppr, int64_t probe_count) {
    constexpr int N = SIDE - 2;
    constexpr int BORDER = 4 * SIDE - 4;
    const int64_t total = probe_count * BORDER;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t p = i / BORDER;
        const int k = int(i % BORDER);
        int r, c, sr, sc;  // border texel (r, c) copies core texel (sr, sc), block coords
        if (k < SIDE) {  // top row incl. corners
            r = 0;
            c = k;
        } else if (k < 2 * SIDE) {  // bottom row incl. corners
            r = SIDE - 1;
            c = k - SIDE;
        } else if (k < 2 * SIDE + N) {  // left column
            r = 1 + (k - 2 * SIDE);
            c = 0;
        } else {  // right column
            r = 1 + (k - 2 * SIDE - N);
            c = SIDE - 1;
        }
        if (r == 0 && c == 0) { sr = N; sc = N; }
        else if (r == 0 && c == SIDE - 1) { sr = N; sc = 1; }
        else if (r == SIDE - 1 && c == 0) { sr = 1; sc = N; }
        else if (r == SIDE - 1 && c == SIDE - 1) { sr = 1; sc = 1; }
        else if (r == 0) { sr = 1; sc = SIDE - 1 - c; }
        else if (r == SIDE - 1) { sr = N; sc = SIDE - 1 - c; }
        else if (c == 0) { sr = SIDE - 1 - r; sc = 1; }
        else { sr = SIDE - 1 - r; sc = N; }
        int64_t y0, x0;
        block_origin(p, ppr, SIDE, y0, x0);
        atlas[(y0 + r) * w + x0 + c] = atlas[(y0 + sr) * w + x0 + sc];
    }
}

inline unsigned grid_for(int64_t n, int threads = 256) {
    return unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), 4 * 148 * 8)));
}

struct SelectWs {
    uint32_t *cand;
    int64_t *ids, *count, *keys_in, *keys_out, *vals_in;
    void *cub_tmp;
    size_t cub_bytes;
    void *cmp;
    size_t cmp_bytes;
    size_t total;
};

SelectWs carve_select(void *ws, size_t bytes, int64_t n) {
    Carver c(ws, bytes);
    SelectWs w;
    w.cand = c.take<uint32_t>(size_t(ceil_div(n, 32)));
    w.ids = c.take<int64_t>(size_t(n));
    w.count = c.take<int64_t>(1);
    w.keys_in = c.take<int64_t>(size_t(n));
    w.keys_out = c.take<int64_t>(size_t(n));
    w.vals_in = c.take<int64_t>(size_t(n));
    w.cub_bytes = sort_temp_bytes(n);
    w.cub_tmp = c.take<char>(w.cub_bytes);
    w.cmp_bytes = compact_workspace_bytes(n);
    w.cmp = c.take<char>(w.cmp_bytes);
    c.take<char>(1);
    w.total = c.off;
    if (ws) c.check();
    return w;
}

struct AssignWs {
    uint32_t *sel_bits, *new_bits, *slot_bits;
    int64_t *sel_ids, *sel_count, *new_ids, *new_count, *plan;
    int64_t *keys_in, *keys_out, *vals_in, *vals_out;
    void *cub_tmp;
    size_t cub_bytes;
    void *cmp;
    size_t cmp_bytes;
    size_t total;
};

AssignWs carve_assign(void *ws, size_t bytes, int64_t n, int64_t slots) {
    Carver c(ws, bytes);
    AssignWs w;
    w.sel_bits = c.take<uint32_t>(size_t(ceil_div(n, 32)));
    w.new_bits = c.take<uint32_t>(size_t(ceil_div(n, 32)));
    w.slot_bits = c.take<uint32_t>(size_t(ceil_div(slots, 32)));
    w.sel_ids = c.take<int64_t>(size_t(n));
    w.sel_count = c.take<int64_t>(1);
    w.new_ids = c.take<int64_t>(size_t(n));
    w.new_count = c.take<int64_t>(1);
    w.plan = c.take<int64_t>(8);
    const bool may_evict = slots < n;
    const int64_t ns = may_evict ? slots : 1;
    w.keys_in = c.take<int64_t>(size_t(ns));
    w.keys_out = c.take<int64_t>(size_t(ns));
    w.vals_in = c.take<int64_t>(size_t(ns));
    w.vals_out = c.take<int64_t>(size_t(ns));
    w.cub_bytes = may_evict ? sort_temp_bytes(ns) : 0;
    w.cub_tmp = c.take<char>(std::max<size_t>(w.cub_bytes, 1));
    w.cmp_bytes = compact_workspace_bytes(std::max(n, slots));
    w.cmp = c.take<char>(w.cmp_bytes);
    c.take<char>(1);
    w.total = c.off;
    if (ws) c.check();
    return w;
}

}  // namespace
}  // namespace ps

namespace ps {
__global__ void frame_advance_kernel(int64_t *state, int64_t gop) {
    const int64_t fc = state[1] + 1;
    state[0] += 1;
    state[1] = fc;
    state[2] = (fc % gop == 0) ? 1 : 0;
}
}  // namespace ps

using namespace ps;

extern "C" {

size_t ps_select_workspace_bytes(int64_t probe_count) {
    return carve_select(nullptr, 0, std::max<int64_t>(probe_count, 1)).total + 256;
}

int ps_select(const uint32_t *changed_bits, const uint32_t *pvs_bits, const uint8_t *active,
              const int64_t *last_sent_seq, int64_t current_seq, int64_t probe_count,
              int has_budget, int64_t budget, int ordered, int64_t *out_ids,
              int64_t *out_count, void *workspace, size_t workspace_bytes, void *stream) {
    PS_ABI_BEGIN
    (void)current_seq;  // staleness order is invariant to the common offset
    if (probe_count < 1) fail(PS_ERR_VALUE, "probe_count must be >= 1");
    if (workspace_bytes < ps_select_workspace_bytes(probe_count))
        fail(PS_ERR_WORKSPACE, "select workspace too small");
    auto s = as_stream(stream);
    const int64_t n = probe_count;
    SelectWs w = carve_select(workspace, workspace_bytes, n);
    candidate_kernel<<<grid_for(ceil_div(n, 32)), 256, 0, s>>>(changed_bits, pvs_bits, active, n,
                                                                w.cand);
    check_launch("candidate_kernel");
    if (!ordered && !has_budget) {
        // the whole candidate set is selected and the caller only needs the set (the
        // slot assignment orders by id anyway): ascending ids, no staleness sort
        compact_bits(w.cand, n, out_ids, nullptr, out_count, w.cmp, w.cmp_bytes, s);
        return PS_OK;
    }
    compact_bits(w.cand, n, w.ids, nullptr, w.count, w.cmp, w.cmp_bytes, s);
    select_keys_kernel<<<grid_for(n), 256, 0, s>>>(w.ids, w.count, last_sent_seq, n, w.keys_in,
                                                   w.vals_in);
    check_launch("select_keys_kernel");
    size_t tmp = w.cub_bytes;
    check_cuda(cub::DeviceRadixSort::SortPairs(w.cub_tmp, tmp, w.keys_in, w.keys_out, w.vals_in,
                                               out_ids, int(n), 0, 64, s),
               "cub SortPairs (select)");
    budget_kernel<<<1, 1, 0, s>>>(w.count, has_budget, budget, out_count);
    check_launch("budget_kernel");
    PS_ABI_END
}

size_t ps_assign_workspace_bytes(int64_t probe_count, int64_t slot_count) {
    const int64_t n = std::max<int64_t>(probe_count, 1);
    const int64_t sl = std::max<int64_t>(slot_count, 1);
    return carve_assign(nullptr, 0, n, sl).total + 256;
}

int ps_assign_slots(const int64_t *selected, const int64_t *n_dev, int64_t n_host,
                    int64_t probe_count, int64_t slot_count, int32_t *probe_slot,
                    int32_t *slot_probe, int64_t *last_selected, int64_t *meta,
                    int64_t *entries, int64_t *entry_count, uint32_t *status_dev,
                    void *workspace, size_t workspace_bytes, void *stream) {
    PS_ABI_BEGIN
    if (probe_count < 1) fail(PS_ERR_VALUE, "probe_count must be >= 1");
    if (slot_count < 1) fail(PS_ERR_VALUE, "slot_count must be >= 1");
    if (workspace_bytes < ps_assign_workspace_bytes(probe_count, slot_count))
        fail(PS_ERR_WORKSPACE, "assign workspace too small");
    auto s = as_stream(stream);
    const int64_t n = probe_count, sc = slot_count;
    AssignWs w = carve_assign(workspace, workspace_bytes, n, sc);
    check_cuda(cudaMemsetAsync(w.sel_bits, 0, size_t(ceil_div(n, 32)) * 4, s), "memset");
    // local status word for index errors so a stale caller flag cannot abort us
    uint32_t *local_status = reinterpret_cast<uint32_t *>(w.plan + 7);
    check_cuda(cudaMemsetAsync(local_status, 0, 4, s), "memset");
    ids_to_bits(selected, n_dev, n_host, n, w.sel_bits, local_status, s);
    compact_bits(w.sel_bits, n, w.sel_ids, nullptr, w.sel_count, w.cmp, w.cmp_bytes, s);
    new_bits_kernel<<<grid_for(ceil_div(n, 32)), 256, 0, s>>>(w.sel_bits, probe_slot, n,
                                                               w.new_bits);
    check_launch("new_bits_kernel");
    compact_bits(w.new_bits, n, w.new_ids, nullptr, w.new_count, w.cmp, w.cmp_bytes, s);
    plan_kernel<<<1, 1, 0, s>>>(w.sel_count, w.new_count, local_status, sc, meta, w.plan,
                                status_dev);
    check_launch("plan_kernel");
    const int64_t *victims = nullptr;
    if (sc < n) {  // eviction is only reachable when slots < probes
        victim_keys_kernel<<<grid_for(sc), 256, 0, s>>>(slot_probe, last_selected, w.sel_bits,
                                                        w.plan, sc, w.keys_in, w.vals_in);
        check_launch("victim_keys_kernel");
        size_t tmp = w.cub_bytes;
        check_cuda(cub::DeviceRadixSort::SortPairs(w.cub_tmp, tmp, w.keys_in, w.keys_out,
                                                   w.vals_in, w.vals_out, int(sc), 0, 64, s),
                   "cub SortPairs (evict)");
        victims = w.vals_out;
    }
    bind_kernel<<<grid_for(n), 256, 0, s>>>(w.new_ids, victims, w.plan, probe_slot, slot_probe);
    check_launch("bind_kernel");
    stamp_kernel<<<grid_for(n), 256, 0, s>>>(w.sel_ids, w.plan, last_selected);
    check_launch("stamp_kernel");
    entry_bits_kernel<<<grid_for(ceil_div(sc, 32)), 256, 0, s>>>(slot_probe, w.sel_bits, w.plan,
                                                                   sc, w.slot_bits);
    check_launch("entry_bits_kernel");
    compact_bits(w.slot_bits, sc, entries, slot_probe, entry_count, w.cmp, w.cmp_bytes, s);
    PS_ABI_END
}

int ps_build_update(int kind, const void *source, int64_t probe_count, int64_t probes_per_row,
                    const int64_t *entries, const int64_t *entry_count, int64_t max_entries,
                    int64_t slots_per_row, void *update_texels, int64_t update_row_stride,
                    void *last_sent, int64_t *last_sent_seq, int64_t current_seq,
                    const int64_t *current_seq_dev, void *stream) {
    PS_ABI_BEGIN
    if (kind != PS_KIND_COLOR && kind != PS_KIND_VISIBILITY) fail(PS_ERR_VALUE, "bad kind");
    if (probes_per_row < 1 || slots_per_row < 1) fail(PS_ERR_VALUE, "bad layout");
    if (max_entries <= 0) return PS_OK;
    auto s = as_stream(stream);
    const int side = kind == PS_KIND_COLOR ? 10 : 18;
    const int64_t src_w = probes_per_row * side;
    const unsigned blocks = unsigned(std::max<int64_t>(
        1, std::min<int64_t>(ceil_div(max_entries, 8), int64_t(sm_count()) * 16)));
    // tuning knob: the cp.async variant measured equal (visibility) or slower
    // (colour 0.056 -> 0.062 ms at C4), so the register version is the default
    static const bool async_build = getenv("PS_BUILD_ASYNC") != nullptr;
    if (async_build) {
        const unsigned ab = unsigned(std::max<int64_t>(
            1, std::min<int64_t>(ceil_div(max_entries, 8 * BUILD_DEPTH), int64_t(sm_count()) * 8)));
        if (kind == PS_KIND_COLOR)
            build_async_kernel<10><<<ab, 256, 0, s>>>(
                static_cast<const uint32_t *>(source), src_w, probes_per_row, entries,
                entry_count, slots_per_row, static_cast<uint32_t *>(update_texels),
                update_row_stride, static_cast<uint32_t *>(last_sent), last_sent_seq,
                current_seq, current_seq_dev);
        else
            build_async_kernel<18><<<ab, 256, 0, s>>>(
                static_cast<const uint32_t *>(source), src_w, probes_per_row, entries,
                entry_count, slots_per_row, static_cast<uint32_t *>(update_texels),
                update_row_stride, static_cast<uint32_t *>(last_sent), last_sent_seq,
                current_seq, current_seq_dev);
        check_launch("build_async_kernel");
        return PS_OK;
    }
    static const int multi = getenv("PS_BUILD_MULTI") ? atoi(getenv("PS_BUILD_MULTI")) : 4;
    // colour: 4 entries per warp iteration (C5 N=131,072: 0.058 -> 0.044 ms)
    if (kind == PS_KIND_COLOR && multi > 1) {
        const unsigned mb = unsigned(std::max<int64_t>(
            1, std::min<int64_t>(ceil_div(max_entries, 8 * 4), int64_t(sm_count()) * 16)));
        build_multi_kernel<10, 4><<<mb, 256, 0, s>>>(
            static_cast<const uint32_t *>(source), src_w, probes_per_row, entries, entry_count,
            slots_per_row, static_cast<uint32_t *>(update_texels), update_row_stride,
            static_cast<uint32_t *>(last_sent), last_sent_seq, current_seq, current_seq_dev);
        check_launch("build_multi_kernel");
        return PS_OK;
    }
    // visibility: 2 entries per warp iteration at 2 CTAs per SM (C5 N=131,072:
    // 0.121 -> 0.117 ms); PS_BUILD_MULTI=1 selects the one-entry kernels (tuning)
    if (kind == PS_KIND_VISIBILITY && multi > 1) {
        const unsigned mb = unsigned(std::max<int64_t>(
            1, std::min<int64_t>(ceil_div(max_entries, 8 * 2), int64_t(sm_count()) * 16)));
        build_multi_kernel<18, 2, 2><<<mb, 256, 0, s>>>(
            static_cast<const uint32_t *>(source), src_w, probes_per_row, entries, entry_count,
            slots_per_row, static_cast<uint32_t *>(update_texels), update_row_stride,
            static_cast<uint32_t *>(last_sent), last_sent_seq, current_seq, current_seq_dev);
        check_launch("build_multi_kernel");
        return PS_OK;
    }
    if (kind == PS_KIND_COLOR)
        build_kernel<10><<<blocks, 256, 0, s>>>(
            static_cast<const uint32_t *>(source), src_w, probes_per_row, entries, entry_count,
            slots_per_row, static_cast<uint32_t *>(update_texels), update_row_stride,
            static_cast<uint32_t *>(last_sent), last_sent_seq, current_seq, current_seq_dev);
    else
        build_kernel<18><<<blocks, 256, 0, s>>>(
            static_cast<const uint32_t *>(source), src_w, probes_per_row, entries, entry_count,
            slots_per_row, static_cast<uint32_t *>(update_texels), update_row_stride,
            static_cast<uint32_t *>(last_sent), last_sent_seq, current_seq, current_seq_dev);
    check_launch("build_kernel");
    PS_ABI_END
}

int ps_export_tiles(int kind, const void *source, int64_t probe_count, int64_t probes_per_row,
                    const int64_t *entries, const int64_t *entry_count, int64_t max_entries,
                    int64_t probe_begin, int64_t probe_end, void *payload, void *last_sent,
                    int64_t *last_sent_seq, int64_t current_seq,
                    const int64_t *current_seq_dev, void *stream) {
    PS_ABI_BEGIN
    if (kind != PS_KIND_COLOR && kind != PS_KIND_VISIBILITY) fail(PS_ERR_VALUE, "bad kind");
    if (probe_begin < 0 || probe_end > probe_count || probe_begin > probe_end)
        fail(PS_ERR_INDEX, "probe range outside the volume");
    if (max_entries <= 0) return PS_OK;
    auto s = as_stream(stream);
    const unsigned blocks = unsigned(std::max<int64_t>(
        1, std::min<int64_t>(ceil_div(max_entries, 8), int64_t(sm_count()) * 16)));
    if (kind == PS_KIND_COLOR)
        export_kernel<10><<<blocks, 256, 0, s>>>(
            static_cast<const uint32_t *>(source), probes_per_row * 10, probes_per_row, entries,
            entry_count, probe_begin, probe_end, static_cast<uint32_t *>(payload),
            static_cast<uint32_t *>(last_sent), last_sent_seq, current_seq, current_seq_dev);
    else
        export_kernel<18><<<blocks, 256, 0, s>>>(
            static_cast<const uint32_t *>(source), probes_per_row * 18, probes_per_row, entries,
            entry_count, probe_begin, probe_end, static_cast<uint32_t *>(payload),
            static_cast<uint32_t *>(last_sent), last_sent_seq, current_seq, current_seq_dev);
    check_launch("export_kernel");
    PS_ABI_END
}

int ps_frame_advance(int64_t *state, int64_t gop_length, void *stream) {
    PS_ABI_BEGIN
    if (!state) fail(PS_ERR_VALUE, "state must not be NULL");
    if (gop_length < 1) fail(PS_ERR_VALUE, "gop_length must be >= 1");
    frame_advance_kernel<<<1, 1, 0, as_stream(stream)>>>(state, gop_length);
    check_launch("frame_advance_kernel");
    PS_ABI_END
}

int ps_import_tiles(int kind, const void *payloads, int64_t payload_stride,
                    const int64_t *rank_begin, int32_t world, const int64_t *entries,
                    const int64_t *entry_count, int64_t max_entries, int64_t slots_per_row,
                    void *update_texels, int64_t update_row_stride, void *stream) {
    PS_ABI_BEGIN
    if (kind != PS_KIND_COLOR && kind != PS_KIND_VISIBILITY) fail(PS_ERR_VALUE, "bad kind");
    if (world < 1 || world > 64) fail(PS_ERR_VALUE, "world size in [1, 64]");
    if (max_entries <= 0) return PS_OK;
    auto s = as_stream(stream);
    const unsigned blocks = unsigned(std::max<int64_t>(
        1, std::min<int64_t>(ceil_div(max_entries, 8), int64_t(sm_count()) * 16)));
    if (kind == PS_KIND_COLOR)
        import_kernel<8><<<blocks, 256, 0, s>>>(static_cast<const uint32_t *>(payloads),
                                                payload_stride, rank_begin, world, entries,
                                                entry_count, slots_per_row,
                                                static_cast<uint32_t *>(update_texels),
                                                update_row_stride);
    else
        import_kernel<16><<<blocks, 256, 0, s>>>(static_cast<const uint32_t *>(payloads),
                                                 payload_stride, rank_begin, world, entries,
                                                 entry_count, slots_per_row,
                                                 static_cast<uint32_t *>(update_texels),
                                                 update_row_stride);
    check_launch("import_kernel");
    PS_ABI_END
}

size_t ps_index_workspace_bytes(int64_t max_entries) {
    const int64_t n = std::max<int64_t>(max_entries, 1);
    size_t scan = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan, (const uint32_t *)nullptr, (uint64_t *)nullptr, int(n));
    return size_t(n) * (4 + 8) + scan + 1024;
}

int ps_encode_index(const int64_t *entries, const int64_t *entry_count, int64_t max_entries,
                    uint8_t *out, int64_t *out_len, void *workspace, size_t workspace_bytes,
                    void *stream) {
    PS_ABI_BEGIN
    const int64_t n = std::max<int64_t>(max_entries, 1);
    if (workspace_bytes < ps_index_workspace_bytes(max_entries)) fail(PS_ERR_WORKSPACE, "index workspace");
    Carver c(workspace, workspace_bytes);
    uint32_t *lens = c.take<uint32_t>(size_t(n));
    uint64_t *offsets = c.take<uint64_t>(size_t(n));
    size_t scan = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan, lens, offsets, int(n));
    void *tmp = c.take<char>(scan);
    c.check();
    auto s = as_stream(stream);
    index_len_kernel<<<grid_for(n), 256, 0, s>>>(entries, entry_count, n, lens);
    check_launch("index_len_kernel");
    check_cuda(cub::DeviceScan::ExclusiveSum(tmp, scan, lens, offsets, int(n), s), "index scan");
    index_write_kernel<<<grid_for(n), 256, 0, s>>>(entries, entry_count, offsets, lens, n, out, out_len);
    check_launch("index_write_kernel");
    PS_ABI_END
}

int ps_reconstruct_guard_bands(int kind, void *atlas, int64_t probe_count,
                               int64_t probes_per_row, void *stream) {
    PS_ABI_BEGIN
    if (kind != PS_KIND_COLOR && kind != PS_KIND_VISIBILITY) fail(PS_ERR_VALUE, "bad kind");
    auto s = as_stream(stream);
    if (kind == PS_KIND_COLOR)
        guard_kernel<10><<<grid_for(probe_count * 36), 256, 0, s>>>(
            static_cast<uint32_t *>(atlas), probes_per_row * 10, probes_per_row, probe_count);
    else
        guard_kernel<18><<<grid_for(probe_count * 68), 256, 0, s>>>(
            static_cast<uint32_t *>(atlas), probes_per_row * 18, probes_per_row, probe_count);
    check_launch("guard_kernel");
    PS_ABI_END
}

}  // extern "C"
