// Stage (2) on the 5th-generation tensor cores: the DDGI blend as dense
// products issued with tcgen05.mma (kind::tf32, fp32 accumulators in TMEM).
//
// Per frame every probe blends its R rays into 64 colour texels and 256 depth
// texels with weights that are shared by all probes (cosine / cosine^s of the
// texel and ray directions).  For a CTA of P = 32 probes that is
//
//   D_depth[t, n] = sum_r Wd[r, t] * Bd[r, n]     t < 256, n = (d | d^2, probe)
//   D_col  [t, n] = sum_r Wc[r, t] * Bc[r, n]     t < 64,  n = (r | g | b, probe)
//
// i.e. M = texels (two M=128 tiles for depth, one M=128 tile for colour),
// N = 64 / 96 probe channels, K = rays in steps of 8.  TMEM holds all three
// accumulators (64 + 64 + 96 = 224 of a 256-column allocation), so two CTAs
// share an SM and one's epilogue overlaps the other's MMAs.
//
// Precision (parity bar: 1e-4 relative / 1e-5 absolute vs the fp32 oracle,
// BASELINE.json north_star): 3xTF32.  Weights and probe channels are plain
// fp32; each is split x = hi + lo, hi = x with its low 13 mantissa bits
// cleared (exact in tf32), lo = x - hi (exact in fp32), and every product is
// issued as W_hi*B_hi + W_hi*B_lo + W_lo*B_hi.  What is lost is W_lo*B_lo and
// the tf32 truncation of the lo terms, <= 2^-20 relative per product: the
// sums are fp32-accurate.
//   * depth: 3 MMAs per 128-texel tile and k-step (A = W_hi, W_hi, W_lo);
//   * colour: the 64 live texels use rows 0-63 of the M=128 tile for W_hi and
//     rows 64-127 for W_lo, so A_c x B_hi yields W_hi*B_hi (rows 0-63) and
//     W_lo*B_hi (rows 64-127) in one MMA, and A_c x B_lo adds W_hi*B_lo (and
//     W_lo*B_lo) -- 2 MMAs; the epilogue adds TMEM lanes t and t + 64.
//
// Warp-specialised pipeline over k-steps of 8 rays, STAGES shared-memory
// stages of 30 KB, mbarriers between the roles:
//   * warp 5 (one thread) streams the weights (5 operand images, 20 KB per
//     k-step, one TMA bulk copy) from a per-frame image the weights pass
//     writes in the canonical K-major no-swizzle UMMA layout;
//   * warps 0-3 stream their ray records through a cp.async ring (RING - 1
//     k-steps ahead) and convert them into the B images (channels d, d^2, r,
//     g, b), hi and lo;
//   * warp 4 (one thread) issues 8 MMAs per k-step and commits them to the
//     stage's "empty" barrier.
// The epilogue reads the accumulators with tcgen05.ld (one texel per TMEM
// lane), applies the normalisation / hysteresis / quantisation of the
// CUDA-core blend and writes the guard-banded atlas blocks.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <type_traits>

#include "ps_common.cuh"
#include "ps_guard.cuh"

namespace ps {
namespace tc {

constexpr int P = 32;         // probes per CTA (two CTAs per SM: one's epilogue overlaps
                              // the other's MMAs)
constexpr int THREADS = 256;  // warps 0-3 convert records, 4 issues MMAs, 5 loads weights
constexpr int PRODUCERS = 128;
#ifndef PS_BLEND_STAGES
#define PS_BLEND_STAGES 3
#endif
#ifndef PS_BLEND_RING
#define PS_BLEND_RING 5
#endif
constexpr int STAGES = PS_BLEND_STAGES;
constexpr int PART = 128 * 8;  // floats of one 128-row x 8-k operand image
// A images of a k-step: depth hi tile 0, depth hi tile 1, depth lo tile 0,
// depth lo tile 1, colour (rows 0-63 hi, 64-127 lo)
constexpr int A_DHI = 0, A_DLO = 2 * PART, A_COL = 4 * PART;
constexpr int A_FLOATS = 5 * PART;
constexpr int BD_ROWS = 2 * P;                // d (probe q) then d^2 (probe q)
constexpr int BC_ROWS = 3 * P;                // r, g, b
constexpr int BD = BD_ROWS * 8;               // floats of one depth B image
constexpr int BC = BC_ROWS * 8;
constexpr int STAGE = A_FLOATS + 2 * BD + 2 * BC;  // 7680 floats = 30 KB
constexpr uint32_t A_LOAD_BYTES = A_FLOATS * 4;
constexpr int RAW = P * 8 * 4;  // floats of one k-step's raw ray records (4 KB)
constexpr int RING = PS_BLEND_RING;  // raw record ring: records stream RING - 1 k-steps ahead
constexpr size_t SMEM_BYTES = (size_t(STAGES) * STAGE + size_t(RING) * RAW) * 4 + 1024;
// epilogue: quantised cores + the colour lo partials handed from TMEM lanes 64-127
constexpr int XBUF = 2 * 3 * 64 * 16;  // [half][ch][texel][probe of the half]
constexpr uint32_t COL_D0 = 0, COL_D1 = BD_ROWS, COL_C = 2 * BD_ROWS, TMEM_COLS = 256;

static_assert(COL_C + BC_ROWS <= TMEM_COLS, "accumulators must fit the TMEM allocation");
static_assert(P * 64 + P * 256 + XBUF <= STAGES * STAGE + RING * RAW,
              "epilogue staging must fit the stages and the ring");
#ifndef PS_BLEND_CTAS
#define PS_BLEND_CTAS 2  // CTAs per SM (tuning: 1 allows deeper stage / ring pipelines)
#endif
static_assert(PS_BLEND_CTAS * (SMEM_BYTES + 1024) + 1024 <= 233472, "CTAs per SM vs shared memory");

// canonical K-major, no-swizzle operand image: 8-row x 16-byte core matrices,
// row groups 128 B apart (SBO), the two 4-wide k halves rows*16 B apart (LBO);
// within a k half, row m starts at float 4m
__host__ __device__ constexpr int img_off(int rows, int m, int k) {
    return (k >> 2) * rows * 4 + (m >> 3) * 32 + (m & 7) * 4 + (k & 3);
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t smem_desc(const float *p, uint32_t rows) {
    uint64_t d = uint64_t((smem_u32(p) >> 4) & 0x3FFFu);
    d |= uint64_t((rows * 16u >> 4) & 0x3FFFu) << 16;  // leading byte offset (k halves)
    d |= uint64_t((128u >> 4) & 0x3FFFu) << 32;        // stride byte offset (row groups)
    d |= uint64_t(1) << 46;                            // descriptor version (sm_100)
    return d;                                          // base 0, swizzle none
}

// instruction descriptor: D f32, A/B tf32, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc(int m, int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t id,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(id), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE;\n\t"
        "bra LAB_WAIT;\n\t"
        "DONE:\n\t}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// 16 consecutive accumulator columns of this warp's 32 TMEM lanes
__device__ __forceinline__ void tmem_ld16(uint32_t addr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float tf32_hi(float x) {
    return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

// weights pass: the per-frame A image, (R/8) k-steps x 5 operand images of
// the fp32 weights split hi + lo
__global__ void weight_image_kernel(const float *w_color, const float *w_depth, int R,
                                    float *img) {
    const int total = (R / 8) * A_FLOATS;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int s = i / A_FLOATS, rem = i - s * A_FLOATS;
        const int part = rem / PART, off = rem - part * PART;
        // invert img_off(128, m, k)
        const int kh = off / 512, in = off - kh * 512;
        const int m = (in >> 5) * 8 + ((in & 31) >> 2);
        const int k = kh * 4 + (in & 3);
        const int r = s * 8 + k;
        bool lo;
        float w;
        if (part == 4) {  // colour: rows 0-63 hi, rows 64-127 lo of texel m & 63
            w = w_color[r * 64 + (m & 63)];
            lo = m >= 64;
        } else {
            w = w_depth[r * 256 + (part & 1) * 128 + m];
            lo = part >= 2;
        }
        const float hi = tf32_hi(w);
        img[i] = lo ? w - hi : hi;
    }
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

// TMA bulk copy global -> shared, completing `bytes` of the barrier's transaction count
// bulk prefetch of a global range into L2 (16-byte aligned, multiple of 16 bytes)
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// one producer thread's share of a k-step: rays (8c + 2j, 8c + 2j + 1) of probe q,
// copied raw (2 float4) into its ring slot
__device__ __forceinline__ void issue_raw(float *slot, const float4 *records, int R, int q,
                                          int nq, int c, int j) {
    if (q < nq) {
        const float4 *src = records + size_t(q) * R + c * 8 + 2 * j;
        float *dst = slot + (q * 8 + 2 * j) * 4;
        cp_async16(dst, src);
        cp_async16(dst + 4, src + 1);
    }
}

struct Rec2 {
    float4 a, b;
};

__device__ __forceinline__ Rec2 read_raw(const float *slot, int q, int nq, int j) {
    Rec2 v;
    if (q < nq) {
        const float4 *src = reinterpret_cast<const float4 *>(slot) + q * 8 + 2 * j;
        v.a = src[0];
        v.b = src[1];
    } else {
        v.a = v.b = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    return v;
}

__device__ __forceinline__ void put2(float *img, int rows, int m, int k, float x0, float x1) {
    *reinterpret_cast<float2 *>(img + img_off(rows, m, k)) = make_float2(x0, x1);
}

// records -> B images (hi, lo) of the stage: channels d, d^2 (depth), r, g, b
__device__ __forceinline__ void stage_b(float *st, const Rec2 &v, int q, int j) {
    float *bdh = st + A_FLOATS, *bdl = bdh + BD, *bch = bdl + BD, *bcl = bch + BC;
    const int k = 2 * j;
    const float x0[5] = {v.a.w, v.a.w * v.a.w, v.a.x, v.a.y, v.a.z};
    const float x1[5] = {v.b.w, v.b.w * v.b.w, v.b.x, v.b.y, v.b.z};
#pragma unroll
    for (int ch = 0; ch < 5; ++ch) {
        const float h0 = tf32_hi(x0[ch]), h1 = tf32_hi(x1[ch]);
        if (ch < 2) {
            put2(bdh, BD_ROWS, ch * P + q, k, h0, h1);
            put2(bdl, BD_ROWS, ch * P + q, k, x0[ch] - h0, x1[ch] - h1);
        } else {
            put2(bch, BC_ROWS, (ch - 2) * P + q, k, h0, h1);
            put2(bcl, BC_ROWS, (ch - 2) * P + q, k, x0[ch] - h0, x1[ch] - h1);
        }
    }
}

__device__ __forceinline__ void issue_mma(const float *st, uint32_t tmem, int c) {
    const float *a = st;
    const float *bdh = st + A_FLOATS, *bdl = bdh + BD, *bch = bdl + BD, *bcl = bch + BC;
    const uint32_t acc = c > 0 ? 1u : 0u;
    constexpr uint32_t ID_D = idesc(128, BD_ROWS), ID_C = idesc(128, BC_ROWS);
    const uint64_t b_dh = smem_desc(bdh, BD_ROWS), b_dl = smem_desc(bdl, BD_ROWS);
    const uint64_t b_ch = smem_desc(bch, BC_ROWS), b_cl = smem_desc(bcl, BC_ROWS);
#pragma unroll
    for (int t = 0; t < 2; ++t) {  // depth tiles (texels 0-127, 128-255)
        const uint64_t a_hi = smem_desc(a + A_DHI + t * PART, 128);
        const uint64_t a_lo = smem_desc(a + A_DLO + t * PART, 128);
        const uint32_t d = tmem + (t ? COL_D1 : COL_D0);
        mma_tf32(d, a_hi, b_dh, ID_D, acc);
        mma_tf32(d, a_hi, b_dl, ID_D, 1u);
        mma_tf32(d, a_lo, b_dh, ID_D, 1u);
    }
    const uint64_t a_c = smem_desc(a + A_COL, 128);
    mma_tf32(tmem + COL_C, a_c, b_ch, ID_C, acc);
    mma_tf32(tmem + COL_C, a_c, b_cl, ID_C, 1u);
}

// the guard-banded SIDE x SIDE blocks of probes p0 .. p0 + nq - 1, from their
// quantised cores staged in shared memory (core[q * CORE_WORDS + i])
template <int SIDE, int NJ>
__device__ __forceinline__ void write_blocks(uint32_t *atlas, int ppr, int p0, int nq,
                                             const uint32_t *core, int core_words, int warp,
                                             int lane) {
    static_assert(NJ * 32 >= SIDE * SIDE, "NJ words per lane cover the block");
    int src[NJ], off[NJ];
    const int W = ppr * SIDE;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        const int k = lane + 32 * j;
        const int r = k / SIDE, c = k - (k / SIDE) * SIDE;
        src[j] = k < SIDE * SIDE ? guard_source(r, c, SIDE) : -1;
        off[j] = r * W + c;
    }
    for (int q = warp; q < nq; q += THREADS / 32) {
        const int p = p0 + q, by = p / ppr;
        uint32_t *blk = atlas + size_t(by) * SIDE * W + size_t(p - by * ppr) * SIDE;
        const uint32_t *cq = core + q * core_words;
#pragma unroll
        for (int j = 0; j < NJ; ++j)
            if (src[j] >= 0) blk[off[j]] = cq[src[j]];
    }
}

__global__ void __launch_bounds__(THREADS, PS_BLEND_CTAS)
    blend_tc_kernel(ps_trace_params prm, int rotate) {
    extern __shared__ unsigned char smem_raw[];
    // 1024-byte aligned by offsetting the shared array itself (an integer round
    // trip through uintptr_t would lose the shared address space and turn every
    // ring read, operand-image write and epilogue staging access into a
    // generic 64-bit LD / ST instead of LDS / STS)
    float *stages = reinterpret_cast<float *>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    __shared__ __align__(8) uint64_t a_full[STAGES], b_full[STAGES], empty[STAGES], done;
    __shared__ uint32_t s_tmem;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int R = prm.rays_per_probe, NK = R / 8;
    const int64_t p0 = int64_t(prm.probe_begin) + int64_t(blockIdx.x) * P;
    const int64_t left = int64_t(prm.probe_end) - p0;
    const int nq = int(left < P ? left : P);
    const int64_t pl0 = p0 - prm.probe_begin;
    // rotate: CTA b walks its k-steps from (b mod NK), so the CTAs in flight read
    // different weight-image k-steps instead of all the same L2 lines at once
    const int kr = rotate ? int(blockIdx.x % unsigned(NK)) : 0;
    auto kstep = [&](int c) { return c + kr < NK ? c + kr : c + kr - NK; };

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&a_full[s], 1);
            mbar_init(&b_full[s], PRODUCERS);
            mbar_init(&empty[s], 1);
        }
        mbar_init(&done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&s_tmem)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;

    // ---- main loop: k-steps of 8 rays, warp-specialised ------------------------------------
    // stage s, use u = c / STAGES: a_full / b_full complete phase u when the weights /
    // probe channels of k-step c are in place; empty completes phase u when the MMAs of
    // k-step c have drained the stage.
    if (warp < PRODUCERS / 32) {
        // each thread streams its own 32 B of every k-step through the raw ring (no
        // cross-thread hand-off), RING - 1 k-steps ahead of its conversion
        const float4 *records = reinterpret_cast<const float4 *>(prm.records) + pl0 * R;
        float *ring = stages + STAGES * STAGE;
        const int q = tid >> 2, j = tid & 3;
#pragma unroll
        for (int c = 0; c < RING - 1; ++c) {
            if (c < NK) issue_raw(ring + c * RAW, records, R, q, nq, kstep(c), j);
            cp_async_commit();
        }
#pragma unroll 1
        for (int c = 0; c < NK; ++c) {
            const int s = c % STAGES, u = c / STAGES;
            if (c + RING - 1 < NK)
                issue_raw(ring + ((c + RING - 1) % RING) * RAW, records, R, q, nq,
                          kstep(c + RING - 1), j);
            cp_async_commit();
            cp_async_wait<RING - 1>();  // k-step c's records have landed
            const Rec2 rv = read_raw(ring + (c % RING) * RAW, q, nq, j);
            if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
            stage_b(stages + s * STAGE, rv, q, j);
            fence_async_smem();  // generic-proxy stores -> visible to the tensor core
            mbar_arrive(&b_full[s]);
        }
        cp_async_wait<0>();
    } else if (warp == 4) {
        if (lane == 0) {
#pragma unroll 1
            for (int c = 0; c < NK; ++c) {
                const int s = c % STAGES, u = c / STAGES;
                mbar_wait(&a_full[s], u & 1);
                mbar_wait(&b_full[s], u & 1);
                tc_fence_after();
                issue_mma(stages + s * STAGE, tmem, c);
                mma_commit(&empty[s]);
            }
            mma_commit(&done);  // arrives once every MMA of the CTA has completed
        }
        __syncwarp();
    } else if (warp == 5) {
        if (lane == 0) {
            if (prm.hysteresis != 0.f) {
                // the epilogue reads this CTA's old state: pull it into L2 while the
                // MMAs run, so the epilogue's loads are L2 hits, not HBM round trips
                bulk_prefetch_l2(reinterpret_cast<const float2 *>(prm.moments) + pl0 * 256,
                                 uint32_t(nq) * 256 * 8);
                bulk_prefetch_l2(prm.irradiance + pl0 * 64 * 3, uint32_t(nq) * 64 * 3 * 4);
            }
#pragma unroll 1
            for (int c = 0; c < NK; ++c) {
                const int s = c % STAGES, u = c / STAGES;
                if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
                // the k-step's five operand images are contiguous in the weight image
#ifdef PS_BLEND_NO_WEIGHT_TRAFFIC  // tuning only (wrong results): weights loaded once
                if (c >= STAGES) {
                    mbar_arrive(&a_full[s]);
                    continue;
                }
#endif
                mbar_expect_tx(&a_full[s], A_LOAD_BYTES);
                bulk_g2s(stages + s * STAGE, prm.w_image + size_t(kstep(c)) * A_FLOATS,
                         A_LOAD_BYTES, &a_full[s]);
            }
        }
        __syncwarp();
    }
    // (a parity wait on a stage barrier could alias a phase two behind: use `done`)
    mbar_wait(&done, 0);
    tc_fence_after();

#ifdef PS_BLEND_NO_EPILOGUE  // tuning: time the main loop alone
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(TMEM_COLS));
    }
    return;
#endif
    // ---- epilogue: TMEM -> state + quantised cores (staged in the freed stages) -----------
    uint32_t *s_ccore = reinterpret_cast<uint32_t *>(stages);  // [P][64]
    uint32_t *s_vcore = s_ccore + P * 64;                      // [P][256]
    const float h = prm.hysteresis;
    const float qs = prm.irradiance_scale > 0.f ? 1.0f / prm.irradiance_scale : 0.f;
    const int sub = warp & 3, half = warp >> 2;
    const uint32_t lane_base = tmem + (uint32_t(sub * 32) << 16);
    {  // depth moments: warp half h owns tile h, one texel per lane
        const int t = half * 128 + sub * 32 + lane;
        const float inv = __ldg(prm.inv_wsum + 64 + t);
        const uint32_t base = lane_base + (half ? COL_D1 : COL_D0);
        float2 *mom = reinterpret_cast<float2 *>(prm.moments) + pl0 * 256 + t;
        const bool need_old = inv == 0.f || h != 0.f;
#pragma unroll 1
        for (int q0 = 0; q0 < P; q0 += 16) {
            float2 old[16];  // independent loads first: the state read is latency bound
#pragma unroll
            for (int i = 0; i < 16; ++i)
                old[i] = (need_old && q0 + i < nq) ? __ldcs(mom + (q0 + i) * 256)
                                                   : make_float2(0.f, 0.f);
            float m1[16], m2[16];
            tmem_ld16(base + q0, m1);
            tmem_ld16(base + P + q0, m2);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int qq = q0 + i;
                if (qq >= nq) break;
                float a = m1[i] * inv, b = m2[i] * inv;
                if (inv == 0.f) {
                    a = old[i].x;
                    b = old[i].y;
                } else if (h != 0.f) {
                    a = fmaf(h, old[i].x - a, a);
                    b = fmaf(h, old[i].y - b, b);
                }
                __stcs(mom + qq * 256, make_float2(a, b));
                s_vcore[qq * 256 + t] = uint32_t(__half_as_ushort(__float2half_rn(a))) |
                                        (uint32_t(__half_as_ushort(__float2half_rn(b))) << 16);
            }
        }
    }
    // colour: TMEM lanes 0-63 hold W_hi*B (+ W_hi*B_lo) of the 64 texels, lanes
    // 64-127 the W_lo*B_hi terms of the same texels; warp half h owns probes
    // h*16..h*16+15.  A warp can only read its own TMEM lane quarter, so the
    // hi warps (quarters 0-1) and the lo warps (quarters 2-3) trade halves
    // through shared memory: the hi warps finish probes 0-7 of the half, the
    // lo warps probes 8-15 -- every warp finishes 8 probes of 32 texels.
    float *xbuf = reinterpret_cast<float *>(s_vcore + P * 256);  // [half][hi|lo][ch][t][8]
    const int q0c = half * (P / 2);
    static_assert(P / 2 == 16, "one 16-column TMEM load per channel");
    const uint32_t cbase = lane_base + COL_C;
    const bool hi_warp = sub < 2;
    const int tcol = (sub & 1) * 32 + lane;  // this lane's colour texel (both roles)
    float own[3][16];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) tmem_ld16(cbase + ch * P + q0c, own[ch]);
    // own[] is indexed with compile-time offsets only (a run-time offset would
    // put the array in local memory): the two roles are two instantiations
    auto give_half = [&](auto GIVE) {  // hi warps give probes 8-15, lo warps 0-7
        constexpr int give = decltype(GIVE)::value;
        float *xo = xbuf + ((half * 2 + (give ? 0 : 1)) * 3) * 64 * 8;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch)
#pragma unroll
            for (int i = 0; i < 8; ++i) xo[(ch * 64 + tcol) * 8 + i] = own[ch][give + i];
    };
    if (hi_warp)
        give_half(std::integral_constant<int, 8>());
    else
        give_half(std::integral_constant<int, 0>());
    const int keep = hi_warp ? 0 : 8;  // probes this warp finishes: q0c + keep + 0..7
    const float inv_c = __ldg(prm.inv_wsum + tcol);
    const bool need_old_c = inv_c == 0.f || h != 0.f;
    float old[8][3];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int qq = q0c + keep + i;
        const float *st = prm.irradiance + ((pl0 + qq) * 64 + tcol) * 3;
        const bool ld = need_old_c && qq < nq;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) old[i][ch] = ld ? __ldcs(st + ch) : 0.f;
    }
    __syncthreads();  // both halves are in xbuf
    auto finish = [&](auto KEEP) {
        constexpr int kp = decltype(KEEP)::value;
        const float *xi = xbuf + ((half * 2 + (kp ? 0 : 1)) * 3) * 64 * 8;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int qq = q0c + kp + i;
            if (qq >= nq) break;
            float *st = prm.irradiance + ((pl0 + qq) * 64 + tcol) * 3;
            uint32_t texel = 0;
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
                const float acc = own[ch][kp + i] + xi[(ch * 64 + tcol) * 8 + i];
                float v = acc * inv_c;
                if (inv_c == 0.f) v = old[i][ch];  // no ray sees this texel: keep the state
                else if (h != 0.f) v = fmaf(h, old[i][ch] - v, v);
                __stcs(st + ch, v);
                const float x = fminf(fmaxf(v * qs, 0.0f), 1.0f);
                texel |= __float2uint_rn(x * 1023.0f) << (10 * ch);
            }
            s_ccore[qq * 64 + tcol] = texel;
        }
    };
    if (hi_warp)
        finish(std::integral_constant<int, 0>());
    else
        finish(std::integral_constant<int, 8>());
    tc_fence_before();
    __syncthreads();

    // ---- atlas blocks with guard bands -------------------------------------------------------
    // a warp writes whole probe blocks: one block-origin division per probe,
    // and each lane's guard-band source indices (its words k = lane + 32 j of
    // the 10 x 10 / 18 x 18 block) computed once, not per word
    write_blocks<10, 4>(prm.color_atlas, prm.probes_per_row_color, int(p0), nq, s_ccore, 64, warp,
                        lane);
    write_blocks<18, 11>(reinterpret_cast<uint32_t *>(prm.vis_atlas), prm.probes_per_row_vis,
                         int(p0), nq, s_vcore, 256, warp, lane);
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(TMEM_COLS));
    }
}

}  // namespace tc

size_t weight_image_floats(int rays_per_probe) {
    return rays_per_probe % 8 == 0 ? size_t(rays_per_probe / 8) * tc::A_FLOATS : 0;
}

void launch_weight_image(const float *w_color, const float *w_depth, int R, float *img,
                         cudaStream_t s) {
    const int total = (R / 8) * tc::A_FLOATS;
    tc::weight_image_kernel<<<unsigned(ceil_div(total, 256)), 256, 0, s>>>(w_color, w_depth, R, img);
    check_launch("weight_image_kernel");
}

bool blend_tc_usable(const ps_trace_params &p) {
    static const bool off = [] {
        const char *e = getenv("PS_BLEND");
        return e && e[0] == 's';  // PS_BLEND=simt forces the CUDA-core blend
    }();
    return !off && p.w_image && p.rays_per_probe % 8 == 0;
}

void launch_blend_tc(const ps_trace_params &p, int64_t nloc, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        check_cuda(cudaFuncSetAttribute(tc::blend_tc_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(tc::SMEM_BYTES)),
                   "cudaFuncSetAttribute(blend_tc)");
        attr = true;
    }
    static const int rotate = getenv("PS_BLEND_ROTATE") ? atoi(getenv("PS_BLEND_ROTATE")) : 0;
    tc::blend_tc_kernel<<<unsigned(ceil_div(nloc, tc::P)), tc::THREADS, tc::SMEM_BYTES, s>>>(
        p, rotate);
    check_launch("blend_tc_kernel");
}

}  // namespace ps
