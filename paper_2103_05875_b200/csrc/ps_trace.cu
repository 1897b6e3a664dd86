// Stages (1)+(2): probe ray tracing (BVH2 stack traversal, no RT cores on
// B200) fused with the DDGI irradiance / depth-moment blend, hysteresis,
// quantisation to the reference's atlas formats and the guard-band copy.
//
// The reference has no implementation of these stages; the
// pinned pieces it does have and that this kernel follows are:
//   ray/primitive semantics   SceneGeometry.raycast, selection.py:66-149
//                             (nearest hit with t > 1e-6, double-sided
//                             Moller-Trumbore with |det| > 1e-6 and
//                             u, v >= -1e-6, u + v <= 1 + 1e-6; normal faces
//                             the ray)
//   base ray set              fibonacci_sphere, selection.py:241-249 (rotated
//                             per frame on the host, shared by every probe)
//   probe positions           volume.py:127-138
//   texel directions          texel_center_uv + oct_decode, volume.py:286-314
//   texel formats             colour A2RGB10 r|g<<10|b<<20 (volume.py:221-226),
//                             visibility raw RG16F halves (volume.py:150-153)
//   guard band                reconstruct_guard_band, packing.py:180-196
//
// One CTA handles P consecutive probes: phase 1 traces all P*R rays (one
// warp = 32 neighbouring directions of one probe) and stages the per-ray
// radiance and depth in shared memory; phase 2 blends them into the 64
// colour and 256 depth texels of each probe.  The per-frame weights
// (cos and cos^sharpness between texel and ray directions) are shared by all
// probes, so phase 2 is a small dense product per CTA: each thread owns one
// texel and walks the rays with the weight row loaded once per ray and the
// ray data broadcast from shared memory.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>

#include "ps_common.cuh"
#include "ps_traverse.cuh"
#include "ps_guard.cuh"

namespace ps {

// ps_blend_tc.cu
size_t weight_image_floats(int rays_per_probe);
void launch_weight_image(const float *w_color, const float *w_depth, int R, float *img,
                         cudaStream_t s);
bool blend_tc_usable(const ps_trace_params &p);
void launch_blend_tc(const ps_trace_params &p, int64_t nloc, cudaStream_t s);
namespace {

constexpr int THREADS = 256;
using namespace trav;

struct Shade {
    float r, g, b, depth, t;
    int prim;
    int shadow_mask;
};

// cube shadow map face / texel of a light-to-point vector (see shadow_map_kernel)
__device__ __forceinline__ int cube_texel(float vx, float vy, float vz, int S) {
    const float ax = fabsf(vx), ay = fabsf(vy), az = fabsf(vz);
    int a;
    float m, u, w, sgn;
    if (ax >= ay && ax >= az) {
        a = 0; m = ax; sgn = vx; u = vy; w = vz;
    } else if (ay >= az) {
        a = 1; m = ay; sgn = vy; u = vz; w = vx;
    } else {
        a = 2; m = az; sgn = vz; u = vx; w = vy;
    }
    const int f = 2 * a + (sgn < 0.0f ? 1 : 0);
    const float inv = 1.0f / m;
    int i = int(floorf(fmaf(u * inv, 0.5f, 0.5f) * float(S)));
    int j = int(floorf(fmaf(w * inv, 0.5f, 0.5f) * float(S)));
    i = min(max(i, 0), S - 1);
    j = min(max(j, 0), S - 1);
    return (f * S + j) * S + i;
}

template <int SHADOW, int WIDTH>
__device__ Shade shade_hit(const ps_trace_params &p, const float4 *nodes, const float4 *tris,
                           const Ray &ray, int slot, float t, float3 shift);

// the ray is moved into the BVH frame once; only that copy lives through the
// traversal, and the hit point goes back to world coordinates by the frame
// origin, reloaded afterwards (keeps the loop at 48 registers without spills)
template <int SHADOW, int LEAFV, int WIDTH, int STATS = 0>
__device__ Shade shade_ray(const ps_trace_params &p, const float4 *nodes, const float4 *tris,
                           const Ray &ray) {
    float t;
    const Ray rt = to_bvh_frame(nodes, ray);
    const int slot = traverse_impl<false, LEAFV, WIDTH, STATS>(nodes, tris, rt, INFINITY, t);
    const float4 org = __ldg(nodes - 4);
    return shade_hit<SHADOW, WIDTH>(p, nodes, tris, rt, slot, t, make_float3(org.x, org.y, org.z));
}

// radiance + depth of a ray given its nearest hit (slot < 0: miss); the hit
// point is ray.o + t ray.d + shift in world coordinates
template <int SHADOW, int WIDTH>
__device__ Shade shade_hit(const ps_trace_params &p, const float4 *nodes, const float4 *tris,
                           const Ray &ray, int slot, float t, float3 shift) {
    Shade s;
    s.shadow_mask = 0;
    if (slot < 0) {
        s.r = p.sky[0];
        s.g = p.sky[1];
        s.b = p.sky[2];
        s.depth = p.max_distance;
        s.t = INFINITY;
        s.prim = -1;
        return s;
    }
    const int prim = __float_as_int(__ldg(tris + 3 * slot).w);
    const float4 *mat = reinterpret_cast<const float4 *>(p.materials) + 3 * prim;
    const float4 alb = __ldg(mat), emi = __ldg(mat + 1), nrm = __ldg(mat + 2);
    // normal faces the incoming ray (selection.py:147-148)
    float nx = nrm.x, ny = nrm.y, nz = nrm.z;
    if (dot3(nx, ny, nz, ray.dx, ray.dy, ray.dz) > 0.0f) {
        nx = -nx;
        ny = -ny;
        nz = -nz;
    }
    const float hx = fmaf(ray.dx, t, ray.ox) + shift.x, hy = fmaf(ray.dy, t, ray.oy) + shift.y,
                hz = fmaf(ray.dz, t, ray.oz) + shift.z;
    const float sx = fmaf(nx, p.normal_bias, hx), sy = fmaf(ny, p.normal_bias, hy),
                sz = fmaf(nz, p.normal_bias, hz);
    float lr = 0.f, lg = 0.f, lb = 0.f;
    const float *L = p.lights;
    const int S = p.shadow_map_size;
    for (int l = 0; l < p.light_count; ++l) {
        const float px = __ldg(L + 6 * l), py = __ldg(L + 6 * l + 1), pz = __ldg(L + 6 * l + 2);
        const float lx = px - sx, ly = py - sy, lz = pz - sz;
        const float d2 = dot3(lx, ly, lz, lx, ly, lz);
        if (!(d2 > 0.0f)) continue;
        const float dist = sqrtf(d2);
        const float inv = 1.0f / dist;
        const float ux = lx * inv, uy = ly * inv, uz = lz * inv;
        const float cosv = dot3(nx, ny, nz, ux, uy, uz);
        if (!(cosv > 0.0f)) continue;
        if (SHADOW == PS_SHADOW_RAYS) {
            Ray sh{sx, sy, sz, ux, uy, uz};
            float ts;
            if (traverse<true, 1, WIDTH>(nodes, tris, sh, dist, ts) >= 0) continue;
        } else if (SHADOW == PS_SHADOW_MAP) {
            const float dm = __ldg(p.shadow_maps + int64_t(l) * 6 * S * S +
                                   cube_texel(-lx, -ly, -lz, S));
            if (dist > dm * (1.0f + p.shadow_bias)) continue;
        }
        s.shadow_mask |= 1 << l;
        const float k = cosv / d2;
        lr = fmaf(__ldg(L + 6 * l + 3), k, lr);
        lg = fmaf(__ldg(L + 6 * l + 4), k, lg);
        lb = fmaf(__ldg(L + 6 * l + 5), k, lb);
    }
    s.r = fmaf(alb.x, lr, emi.x);
    s.g = fmaf(alb.y, lg, emi.y);
    s.b = fmaf(alb.z, lb, emi.z);
    s.depth = fminf(t, p.max_distance);
    s.t = t;
    s.prim = prim;
    return s;
}

// ---- pass 0: cube distance maps traced from each light ------------------------------
// face f: axis a = f / 2, sign = f % 2 ? -1 : +1, (b, c) = ((a+1)%3, (a+2)%3);
// texel (i, j): direction e_a*sign + e_b*u + e_c*w with u = (i+.5)/S*2-1,
// w = (j+.5)/S*2-1, normalised; value = nearest hit distance (inf on a miss).
template <int WIDTH>
__global__ void __launch_bounds__(256) shadow_map_kernel(ps_trace_params prm) {
    const int S = prm.shadow_map_size;
    const int64_t per_light = int64_t(6) * S * S;
    const int64_t all = per_light * prm.light_count;
    const int64_t total = prm.shadow_texel_end > 0 && prm.shadow_texel_end < all
                              ? prm.shadow_texel_end : all;
    const float4 *nodes = reinterpret_cast<const float4 *>(prm.nodes);
    const float4 *tris = reinterpret_cast<const float4 *>(prm.tris);
    // a warp traces an 8 x 4 texel block of one face (a compact cone of
    // directions from the light) when the whole map is traced and S allows it;
    // otherwise consecutive texels of a row
    const bool blocked = prm.shadow_texel_begin == 0 && total == all && S % 8 == 0;
    // index splits by run-time constants as multiply-high divisions (all < 2^31
    // for maps up to 30 lights x 6 x 3,344^2; larger maps take 64-bit divides)
    const bool fast = all < (int64_t(1) << 31);
    const FastDiv div_light{uint32_t(fast ? per_light : 1)}, div_face{uint32_t(S * S)},
        div_s{uint32_t(S)}, div_bs{uint32_t(S >= 8 ? S / 8 : 1)};
    for (int64_t wi = prm.shadow_texel_begin + blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
         wi < total; wi += int64_t(gridDim.x) * blockDim.x) {
        int l, rem, f, i, j;
        if (fast) {
            l = int(div_light.div(uint32_t(wi)));
            rem = int(uint32_t(wi) - uint32_t(l) * div_light.d);
            f = int(div_face.div(uint32_t(rem)));
            const uint32_t r2 = uint32_t(rem) - uint32_t(f) * div_face.d;
            const uint32_t row = div_s.div(r2);
            j = int(row);
            i = int(r2 - row * div_s.d);
            if (blocked) {
                const uint32_t blk = r2 >> 5, ln = r2 & 31, by = div_bs.div(blk);
                i = int(blk - by * div_bs.d) * 8 + int(ln & 7);
                j = int(by) * 4 + int(ln >> 3);
            }
        } else {
            l = int(wi / per_light);
            rem = int(wi - int64_t(l) * per_light);
            f = rem / (S * S);
            j = (rem / S) % S;
            i = rem % S;
            if (blocked) {
                const int r2 = rem - f * S * S, blk = r2 >> 5, ln = r2 & 31;
                i = (blk % (S / 8)) * 8 + (ln & 7);
                j = (blk / (S / 8)) * 4 + (ln >> 3);
            }
        }
        const int64_t idx = int64_t(l) * per_light + int64_t(f) * S * S + int64_t(j) * S + i;
        const int a = f >> 1;
        const float sgn = (f & 1) ? -1.0f : 1.0f;
        const float u = (float(i) + 0.5f) / float(S) * 2.0f - 1.0f;
        const float w = (float(j) + 0.5f) / float(S) * 2.0f - 1.0f;
        float d[3];
        d[a] = sgn;
        d[(a + 1) % 3] = u;
        d[(a + 2) % 3] = w;
        const float inv = 1.0f / sqrtf(dot3(d[0], d[1], d[2], d[0], d[1], d[2]));
        Ray ray{__ldg(prm.lights + 6 * l), __ldg(prm.lights + 6 * l + 1),
                __ldg(prm.lights + 6 * l + 2), d[0] * inv, d[1] * inv, d[2] * inv};
        float t;
        const int slot = traverse<false, 1, WIDTH>(nodes, tris, ray, INFINITY, t);
        const float v = slot < 0 ? INFINITY : t;
        if (prm.shadow_dst)
            for (int d = 0; d < prm.shadow_ndst; ++d) prm.shadow_dst[d][idx] = v;  // peers too
        else
            prm.shadow_maps[idx] = v;
    }
}

// ---- pass 1: probe rays -> per-ray records (persistent, dynamic chunks) -----------------
// A warp claims a chunk of 32 rays from a global counter, traces + shades them
// and writes {rgb, depth}; dynamic claiming keeps every SM busy regardless of
// the large per-chunk cost differences.  The chunk shape is the kernel's main
// lever (PROBE_PARALLEL): every probe shoots the same frame-rotated ray set, so
// the default chunk is ONE direction for a compact tile of probes (2 x 2 x 8
// when the slab is 8 planes deep) -- 32 near-parallel rays from neighbouring
// origins that walk largely the same BVH nodes, so a warp's node fetches hit
// few lines
// (6.18 ms per C4 trace + blend for a 2 x 2 x 8 tile vs 7.90 ms for 32
// neighbouring directions of one probe and 8.70 ms for a row of 32 probes;
// more than one direction per warp was slower).
// TPB = 640 (two CTAs per SM, 48 registers, 40 warps) is the default launch;
// TPB = 1024 is the "SM-sized" launch used when SMs are reserved for
// concurrent streams: one CTA fills an SM (64 registers x 1024 threads), so a
// grid of sms - reserve CTAs leaves whole SMs free (a grid of 256-thread CTAs
// would be spread over every SM and leave only fragments, too small for NCCL's
// kernels).  The kernel is per-warp, so the block size is free.
// CLAIM > 0: chunks are claimed per CTA in blocks of CLAIM consecutive tasks
// (one probe tile x CLAIM consecutive directions of the Morton-ordered ray
// set): the CTA's warps trace neighbouring directions from the same origins
// at the same time, so their node fetches share the SM's L1.  A CTA-shared
// 64-bit word holds (block << 32 | next); the warp that draws next == CLAIM
// fetches the CTA's next block from the global counter.
template <int SHADOW, int LEAFV, int MINB, int PROBE_PARALLEL, int WIDTH, int TPB = THREADS,
          int STATS = 0, int CLAIM = 0>
__global__ void __launch_bounds__(TPB, TPB == THREADS ? MINB : (TPB == 1024 ? 1 : 2))
    trace_kernel(ps_trace_params prm) {
    __shared__ unsigned long long s_claim;
    if (CLAIM > 0) {
        if (threadIdx.x == 0) s_claim = CLAIM;  // block 0 "exhausted": first claim fetches
        __syncthreads();
    }
    const float4 *nodes = reinterpret_cast<const float4 *>(prm.nodes);
    const float4 *tris = reinterpret_cast<const float4 *>(prm.tris);
    const float4 *dirs = reinterpret_cast<const float4 *>(prm.ray_dirs);
    const int R = prm.rays_per_probe;
    const int64_t nloc = int64_t(prm.probe_end) - prm.probe_begin;
    const int64_t total_rays = nloc * R;
    const int64_t chunks_per_probe = (R + 31) / 32;
    // PROBE_PARALLEL: a chunk is one direction for 32 consecutive probes
    // (parallel rays from neighbouring origins) instead of 32 directions of
    // one probe
    const int64_t probe_groups = (nloc + 31) / 32;
    // PROBE_PARALLEL == 2: one direction for a compact 4 x 4 x 2 tile of probes
    // (near-parallel rays from origins <= 2 spacings apart walk the same nodes)
    const int64_t plane = int64_t(prm.nx) * prm.ny;
    const int64_t k0 = prm.probe_begin / plane;
    const int64_t k1 = nloc > 0 ? (prm.probe_end - 1) / plane : k0;
    // tile shapes (x, y, z probes) x D neighbouring directions = 32 rays
    constexpr int PPV = PROBE_PARALLEL;
    constexpr int TX = PPV == 11 ? 1 : (PPV == 3 || PPV == 6) ? 8 : (PPV == 4 || PPV >= 8) ? 2 : 4;
    constexpr int TY = PPV == 11 ? 4 : PPV == 13 ? 8 : (PPV == 5 || PPV == 6 || PPV >= 8) ? 2 : 4;
    constexpr int DD = PPV == 8 ? 2 : PPV == 9 ? 4 : PPV == 10 ? 8 : 1;  // 11-13: 1
    constexpr int TZ = 32 / (TX * TY * DD);
    constexpr bool TILED = PROBE_PARALLEL >= 2;
    const int64_t tiles_x = (prm.nx + TX - 1) / TX, tiles_y = (prm.ny + TY - 1) / TY;
    const int64_t tiles_z = (k1 - k0 + TZ) / TZ;
    const int64_t tiles = tiles_x * tiles_y * tiles_z;
    const int64_t dgroups = (R + DD - 1) / DD;
    const int64_t total_chunks = TILED ? tiles * dgroups
                               : PROBE_PARALLEL ? probe_groups * R : nloc * chunks_per_probe;
    const int lane = threadIdx.x & 31;
    float4 *records = reinterpret_cast<float4 *>(prm.records);
    // run-time divisors of the tiled chunk decode (task -> tile, direction ->
    // probe i, j, k): multiply-high divisions instead of per-ray divisions
    const FastDiv div_dg{uint32_t(dgroups > 0 ? dgroups : 1)},
        div_tx{uint32_t(tiles_x > 0 ? tiles_x : 1)}, div_ty{uint32_t(tiles_y > 0 ? tiles_y : 1)};
    while (true) {
        uint32_t task = 0;
        if (lane == 0) {
            if (CLAIM > 0) {
                while (true) {
                    const unsigned long long old = atomicAdd(&s_claim, 1ull);
                    const uint32_t idx = uint32_t(old);
                    if (idx < uint32_t(CLAIM)) {
                        task = uint32_t(old >> 32) * CLAIM + idx;
                        break;
                    }
                    if (idx == uint32_t(CLAIM)) {
                        const uint32_t nb = atomicAdd(prm.work_counter, 1u);
                        atomicExch(&s_claim, (unsigned long long)nb << 32);
                    } else {
                        __nanosleep(64);
                    }
                }
            } else {
                task = atomicAdd(prm.work_counter, 1u);
            }
        }
        task = __shfl_sync(0xffffffffu, task, 0);
        if (int64_t(task) >= total_chunks) break;
        int64_t q;
        int r;
        int64_t i = 0, j = 0, k = 0;  // grid coordinates (TILED: from the tile)
        if (TILED) {
            uint32_t t;
            if (PROBE_PARALLEL == 7) {  // direction-major: all tiles for one direction
                r = int(int64_t(task) / tiles);
                t = uint32_t(int64_t(task) - int64_t(r) * tiles);
            } else {
                t = div_dg.div(task);
                r = int(task - t * div_dg.d) * DD + lane / (TX * TY * TZ);
                if (r >= R) continue;
            }
            const int pl = lane % (TX * TY * TZ);
            const uint32_t txy = div_tx.div(t), tz = div_ty.div(txy);
            const uint32_t tx = t - txy * div_tx.d, ty = txy - tz * div_ty.d;
            i = int64_t(tx) * TX + (pl % TX);
            j = int64_t(ty) * TY + ((pl / TX) % TY);
            k = k0 + int64_t(tz) * TZ + pl / (TX * TY);
            const int64_t pp = i + prm.nx * (j + prm.ny * k);
            if (i >= prm.nx || j >= prm.ny || pp < prm.probe_begin || pp >= prm.probe_end) continue;
            q = pp - prm.probe_begin;
        } else if (PROBE_PARALLEL) {
            const int64_t g = int64_t(task) / R;
            r = int(int64_t(task) - g * R);
            q = g * 32 + lane;
            if (q >= nloc) continue;
        } else {
            q = int64_t(task) / chunks_per_probe;
            r = int(int64_t(task) - q * chunks_per_probe) * 32 + lane;
            if (r >= R) continue;
        }
        if (!TILED) {
            const int64_t p = prm.probe_begin + q;
            i = p % prm.nx;
            j = (p / prm.nx) % prm.ny;
            k = p / (int64_t(prm.nx) * prm.ny);
        }
        Ray ray;
        // origin + spacing * (i, j, k) in double, rounded once (no FMA
        // contraction, as numpy evaluates volume.py:138)
        ray.ox = float(__dadd_rn(prm.origin[0], __dmul_rn(prm.spacing[0], double(i))));
        ray.oy = float(__dadd_rn(prm.origin[1], __dmul_rn(prm.spacing[1], double(j))));
        ray.oz = float(__dadd_rn(prm.origin[2], __dmul_rn(prm.spacing[2], double(k))));
        const float4 d = __ldg(dirs + r);
        ray.dx = d.x;
        ray.dy = d.y;
        ray.dz = d.z;
        const Shade s = shade_ray<SHADOW, LEAFV, WIDTH, STATS>(prm, nodes, tris, ray);
        const int64_t ray_id = q * R + r;
        // streaming store (evict-first): the 537 MB of records pass through L2
        // without evicting the BVH the traversal keeps re-reading
        __stcs(records + ray_id, make_float4(s.r, s.g, s.b, s.depth));
        if (prm.ray_records) {
            float4 *rec = reinterpret_cast<float4 *>(prm.ray_records) + 2 * ray_id;
            rec[0] = make_float4(s.r, s.g, s.b, s.depth);
            rec[1] = make_float4(s.t, __int_as_float(s.prim), __int_as_float(s.shadow_mask), 0.f);
        }
        (void)total_rays;
    }
}

// ---- pass 1 (alternative): persistent while-while traversal with per-lane refill -------
// Aila & Laine style: every lane owns one ray; a lane that finds a leaf
// postpones it and keeps walking inner nodes until all active lanes hold a
// leaf (speculative traversal), then the warp tests leaves together.  When
// fewer than DYN_FETCH lanes are still busy the warp shades the finished rays
// and refills those lanes from the global ray counter (warp-aggregated
// atomic), so SIMT lanes stay occupied despite the very uneven ray costs.
constexpr int WW_SENTINEL = 0x7fffffff;
constexpr int DYN_FETCH = 20;

__device__ __forceinline__ int ww_pop(const int2 *stack, int &sp, float tb) {
    while (sp > 0) {
        const int2 e = stack[--sp];
        if (__int_as_float(e.y) <= tb) return e.x;
    }
    return WW_SENTINEL;
}

template <int SHADOW, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) trace_ww_kernel(ps_trace_params prm) {
    const float4 *nodes = reinterpret_cast<const float4 *>(prm.nodes);
    const float4 *tris = reinterpret_cast<const float4 *>(prm.tris);
    const float4 *dirs = reinterpret_cast<const float4 *>(prm.ray_dirs);
    const int R = prm.rays_per_probe;
    const int64_t nloc = int64_t(prm.probe_end) - prm.probe_begin;
    const uint32_t total = uint32_t(nloc * R);
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    float4 *records = reinterpret_cast<float4 *>(prm.records);

    uint32_t ray_id = 0;
    bool has_ray = false;
    bool queue_done = false;
    Ray ray{0.f, 0.f, 0.f, 0.f, 0.f, 1.f};
    Ray rt = ray;  // the ray in the BVH frame (ps_traverse.cuh to_bvh_frame)
    float ix = 0.f, iy = 0.f, iz = 0.f, oix = 0.f, oiy = 0.f, oiz = 0.f, tb = 0.f;
    int hit = -1;
    int node = WW_SENTINEL, leaf = 0, sp = 0;
    int2 stack[STACK];

    while (true) {
        // ---- finished rays: shade + write; then refill from the queue ----------------
        const bool idle = node == WW_SENTINEL;
        if (idle && has_ray) {
            const Shade sh = shade_hit<SHADOW, 2>(prm, nodes, tris, ray, hit, tb,
                                                  make_float3(0.f, 0.f, 0.f));
            records[ray_id] = make_float4(sh.r, sh.g, sh.b, sh.depth);
            if (prm.ray_records) {
                float4 *rec = reinterpret_cast<float4 *>(prm.ray_records) + 2 * int64_t(ray_id);
                rec[0] = make_float4(sh.r, sh.g, sh.b, sh.depth);
                rec[1] = make_float4(sh.t, __int_as_float(sh.prim), __int_as_float(sh.shadow_mask), 0.f);
            }
            has_ray = false;
        }
        const unsigned need = __ballot_sync(FULL, idle);
        if (need && !queue_done) {
            const int leader = __ffs(need) - 1;
            uint32_t base = 0;
            if (lane == leader) base = atomicAdd(prm.work_counter, uint32_t(__popc(need)));
            base = __shfl_sync(FULL, base, leader);
            if (base + uint32_t(__popc(need)) >= total) queue_done = true;  // warp-uniform
            if (idle) {
                const uint32_t id = base + uint32_t(__popc(need & lt_mask));
                if (id < total) {
                    ray_id = id;
                    has_ray = true;
                    const int64_t q = id / uint32_t(R);
                    const int r = int(id - uint32_t(q) * uint32_t(R));
                    const int64_t p = prm.probe_begin + q;
                    const int64_t i = p % prm.nx, j = (p / prm.nx) % prm.ny,
                                  k = p / (int64_t(prm.nx) * prm.ny);
                    ray.ox = float(__dadd_rn(prm.origin[0], __dmul_rn(prm.spacing[0], double(i))));
                    ray.oy = float(__dadd_rn(prm.origin[1], __dmul_rn(prm.spacing[1], double(j))));
                    ray.oz = float(__dadd_rn(prm.origin[2], __dmul_rn(prm.spacing[2], double(k))));
                    const float4 d = __ldg(dirs + r);
                    ray.dx = d.x;
                    ray.dy = d.y;
                    ray.dz = d.z;
                    const float sx = fabsf(d.x) < 1e-12f ? copysignf(1e-12f, d.x) : d.x;
                    const float sy = fabsf(d.y) < 1e-12f ? copysignf(1e-12f, d.y) : d.y;
                    const float sz = fabsf(d.z) < 1e-12f ? copysignf(1e-12f, d.z) : d.z;
                    ix = 1.0f / sx;
                    iy = 1.0f / sy;
                    iz = 1.0f / sz;
                    rt = to_bvh_frame(nodes, ray);
                    oix = rt.ox * ix;
                    oiy = rt.oy * iy;
                    oiz = rt.oz * iz;
                    tb = INFINITY;
                    hit = -1;
                    node = 0;
                    leaf = 0;
                    sp = 0;
                }
            }
        }
        if (__all_sync(FULL, node == WW_SENTINEL)) break;

        // ---- while-while traversal -----------------------------------------------------
        while (node != WW_SENTINEL) {
            // inner nodes, postponing the first leaf found
            while (node >= 0 && node != WW_SENTINEL) {
                bool h0, h1;
                float t0, t1;
                int c0, c1;
                node_hits(nodes, node, ix, iy, iz, oix, oiy, oiz, tb, h0, h1, t0, t1, c0, c1);
                if (h0 && h1) {
                    const bool swap = t1 < t0;
                    node = swap ? c1 : c0;
                    stack[sp++] = make_int2(swap ? c0 : c1, __float_as_int(swap ? t0 : t1));
                } else if (h0 || h1) {
                    node = h0 ? c0 : c1;
                } else {
                    node = ww_pop(stack, sp, tb);
                }
                if (node < 0 && leaf == 0) {  // postpone the leaf, keep walking
                    leaf = node;
                    node = ww_pop(stack, sp, tb);
                }
                if (!__any_sync(__activemask(), leaf == 0)) break;
            }
            // leaves
            while (leaf < 0) {
                const int ref = ~leaf;
                const int first = ref >> 3, cnt = ref & 7;
                for (int k = 0; k < cnt; k += 2) {
                    const float4 a0 = __ldg(tris + 3 * (first + k));
                    const float4 a1 = __ldg(tris + 3 * (first + k) + 1);
                    const float4 a2 = __ldg(tris + 3 * (first + k) + 2);
                    float4 b0, b1, b2;
                    const bool two = k + 1 < cnt;
                    if (two) {
                        b0 = __ldg(tris + 3 * (first + k + 1));
                        b1 = __ldg(tris + 3 * (first + k + 1) + 1);
                        b2 = __ldg(tris + 3 * (first + k + 1) + 2);
                    }
                    float t = tri_hit(rt, a0, a1, a2);
                    if (t < tb) {
                        tb = t;
                        hit = first + k;
                    }
                    if (two) {
                        t = tri_hit(rt, b0, b1, b2);
                        if (t < tb) {
                            tb = t;
                            hit = first + k + 1;
                        }
                    }
                }
                leaf = 0;
                if (node < 0 && node != WW_SENTINEL) {  // another leaf popped: take it now
                    leaf = node;
                    node = ww_pop(stack, sp, tb);
                }
            }
            if (__popc(__activemask()) < DYN_FETCH) break;  // refill idle lanes
        }
    }
}

// ---- pass 2: DDGI blend, register-blocked over P = 16 probes per CTA ----------------------
// Per probe the blend is two small dense products with per-frame weights
// shared by every probe: irradiance (64 x R) . (R x 3) and depth moments
// (256 x R) . (R x 2).  A CTA stages the ray records of 16 probes in shared
// memory and streams the weight rows through it in chunks of RC rays; each
// thread owns 4 depth texels x 4 probes (32 accumulators: one LDS.128 of
// weights + two broadcast LDS.128 of (d, d^2) feed 32 FFMA) and 1 colour
// texel x 4 probes (12 accumulators).
constexpr int BP = 16;  // probes per CTA
constexpr int RC = 16;  // rays per weight chunk

__device__ __forceinline__ void finalize_color(const ps_trace_params &prm, int64_t p_local, int t,
                                               const float acc[3], float inv, float h, float qs,
                                               uint32_t *core) {
    float *st = prm.irradiance + (p_local * 64 + t) * 3;
    uint32_t texel = 0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        float v = acc[c] * inv;
        if (inv == 0.f) v = st[c];  // no ray sees this texel: keep the state
        else if (h != 0.f) v = fmaf(h, st[c] - v, v);
        st[c] = v;
        const float x = fminf(fmaxf(v * qs, 0.0f), 1.0f);
        texel |= __float2uint_rn(x * 1023.0f) << (10 * c);
    }
    *core = texel;
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

constexpr int RGB_STRIDE = BP * 3 + 4;  // padded [r] row of 16 probes x rgb (208 B)
constexpr int DEP_STRIDE = BP + 4;      // padded [r] row of 16 probe depths (80 B)
constexpr int W_CHUNK = RC * (256 + 64);  // floats per weight chunk

__device__ __forceinline__ void issue_weight_chunk(float *dst, const float *wd, const float *wc,
                                                   int r0, int rc, int tid) {
    for (int i = tid; i < rc * 64; i += THREADS)  // depth weights: rc x 256 floats
        cp_async16(dst + 4 * i, wd + size_t(r0) * 256 + 4 * i);
    for (int i = tid; i < rc * 16; i += THREADS)  // colour weights: rc x 64 floats
        cp_async16(dst + RC * 256 + 4 * i, wc + size_t(r0) * 64 + 4 * i);
    cp_async_commit();
}

__global__ void __launch_bounds__(THREADS, 2) blend_kernel(ps_trace_params prm) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int R = prm.rays_per_probe;
    float *s_rgb = reinterpret_cast<float *>(smem_raw);  // [R][RGB_STRIDE]
    float *s_dep = s_rgb + R * RGB_STRIDE;                // [R][DEP_STRIDE]
    float *s_w = s_dep + R * DEP_STRIDE;                  // 2 x [RC][256 + 64]
    uint32_t *s_ccore = reinterpret_cast<uint32_t *>(s_w);  // [BP][64]  (aliases W after the loop)
    uint32_t *s_vcore = s_ccore + BP * 64;                   // [BP][256]

    const int tid = threadIdx.x;
    const int64_t p0 = int64_t(prm.probe_begin) + int64_t(blockIdx.x) * BP;
    const int64_t left = int64_t(prm.probe_end) - p0;
    const int nq = int(left < BP ? left : BP);
    const int64_t pl0 = p0 - prm.probe_begin;
    const int nchunks = (R + RC - 1) / RC;
    // weights of the first chunk fly while the ray records are staged
    issue_weight_chunk(s_w, prm.w_depth, prm.w_color, 0, min(RC, R), tid);
    const float4 *records = reinterpret_cast<const float4 *>(prm.records) + pl0 * R;
    for (int g = tid; g < BP * R; g += THREADS) {
        const int q = g / R, r = g - q * R;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (q < nq) v = __ldcs(records + g);  // streamed once
        float *dst = s_rgb + r * RGB_STRIDE + q * 3;
        dst[0] = v.x;
        dst[1] = v.y;
        dst[2] = v.z;
        s_dep[r * DEP_STRIDE + q] = v.w;
    }

    const int tg = tid & 63;  // colour texel / depth texel group
    const int qg = tid >> 6;  // probe group (4 probes)
    float cacc[4][3];
    float dacc[4][4][2];  // [texel][probe][moment]
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        cacc[q][0] = cacc[q][1] = cacc[q][2] = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) dacc[k][q][0] = dacc[k][q][1] = 0.f;
    }
    for (int c = 0; c < nchunks; ++c) {
        const int r0 = c * RC;
        const int rc = min(RC, R - r0);
        if (c + 1 < nchunks) {
            issue_weight_chunk(s_w + ((c + 1) & 1) * W_CHUNK, prm.w_depth, prm.w_color, r0 + RC,
                               min(RC, R - r0 - RC), tid);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();  // chunk c landed for every thread (and the records are staged)
        const float *wd = s_w + (c & 1) * W_CHUNK;
        const float *wcol = wd + RC * 256;
#pragma unroll 4
        for (int rr = 0; rr < rc; ++rr) {
            const int r = r0 + rr;
            const float4 w4 = reinterpret_cast<const float4 *>(wd + rr * 256)[tg];
            const float4 dq = *reinterpret_cast<const float4 *>(s_dep + r * DEP_STRIDE + 4 * qg);
            const float dv[4] = {dq.x, dq.y, dq.z, dq.w};
            const float wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float d2 = dv[q] * dv[q];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    dacc[k][q][0] = fmaf(wv[k], dv[q], dacc[k][q][0]);
                    dacc[k][q][1] = fmaf(wv[k], d2, dacc[k][q][1]);
                }
            }
            const float wc = wcol[rr * 64 + tg];
            const float4 *cp = reinterpret_cast<const float4 *>(s_rgb + r * RGB_STRIDE + 12 * qg);
            const float4 c0 = cp[0], c1 = cp[1], c2 = cp[2];
            const float cv[12] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w, c2.x, c2.y, c2.z, c2.w};
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int k = 0; k < 3; ++k) cacc[q][k] = fmaf(wc, cv[3 * q + k], cacc[q][k]);
        }
        __syncthreads();  // buffer (c & 1) is refilled by the issue two chunks later
    }

    const float h = prm.hysteresis;
    const float qs = prm.irradiance_scale > 0.f ? 1.0f / prm.irradiance_scale : 0.f;
    {
        const float inv = __ldg(prm.inv_wsum + tg);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int qq = 4 * qg + q;
            if (qq < nq) finalize_color(prm, pl0 + qq, tg, cacc[q], inv, h, qs, s_ccore + qq * 64 + tg);
        }
    }
    {
        const float4 inv4 = __ldg(reinterpret_cast<const float4 *>(prm.inv_wsum + 64) + tg);
        const float inv[4] = {inv4.x, inv4.y, inv4.z, inv4.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int qq = 4 * qg + q;
            if (qq >= nq) continue;
            float4 *st = reinterpret_cast<float4 *>(prm.moments + ((pl0 + qq) * 256 + 4 * tg) * 2);
            float4 o01 = make_float4(0.f, 0.f, 0.f, 0.f), o23 = o01;
            if (h != 0.f || inv[0] == 0.f || inv[1] == 0.f || inv[2] == 0.f || inv[3] == 0.f) {
                o01 = st[0];
                o23 = st[1];
            }
            const float old[4][2] = {{o01.x, o01.y}, {o01.z, o01.w}, {o23.x, o23.y}, {o23.z, o23.w}};
            float nv[4][2];
            uint4 packed;
            uint32_t *pk = reinterpret_cast<uint32_t *>(&packed);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float a = dacc[k][q][0] * inv[k], b = dacc[k][q][1] * inv[k];
                if (inv[k] == 0.f) {
                    a = old[k][0];
                    b = old[k][1];
                } else if (h != 0.f) {
                    a = fmaf(h, old[k][0] - a, a);
                    b = fmaf(h, old[k][1] - b, b);
                }
                nv[k][0] = a;
                nv[k][1] = b;
                pk[k] = uint32_t(__half_as_ushort(__float2half_rn(a))) |
                        (uint32_t(__half_as_ushort(__float2half_rn(b))) << 16);
            }
            st[0] = make_float4(nv[0][0], nv[0][1], nv[1][0], nv[1][1]);
            st[1] = make_float4(nv[2][0], nv[2][1], nv[3][0], nv[3][1]);
            reinterpret_cast<uint4 *>(s_vcore + qq * 256)[tg] = packed;
        }
    }
    __syncthreads();

    // ---- atlas blocks with guard bands (32-bit index math: atlases < 2^31 texels) ----------
    {
        const int ppr = prm.probes_per_row_color;
        const int W = ppr * 10;
        const int pb = int(p0);
        for (int idx = tid; idx < nq * 100; idx += THREADS) {
            const int q = idx / 100, k = idx - q * 100;
            const int r = k / 10, c = k - r * 10;
            const int p = pb + q;
            const int by = p / ppr;
            const int y0 = by * 10, x0 = (p - by * ppr) * 10;
            prm.color_atlas[size_t(y0 + r) * W + x0 + c] = s_ccore[q * 64 + guard_source(r, c, 10)];
        }
    }
    {
        const int ppr = prm.probes_per_row_vis;
        const int W = ppr * 18;
        const int pb = int(p0);
        uint32_t *vis = reinterpret_cast<uint32_t *>(prm.vis_atlas);
        for (int idx = tid; idx < nq * 324; idx += THREADS) {
            const int q = idx / 324, k = idx - q * 324;
            const int r = k / 18, c = k - r * 18;
            const int p = pb + q;
            const int by = p / ppr;
            const int y0 = by * 18, x0 = (p - by * ppr) * 18;
            vis[size_t(y0 + r) * W + x0 + c] = s_vcore[q * 256 + guard_source(r, c, 18)];
        }
    }
}

// per-frame blend weights (plain fp32): w_color[r][t] = max(0, n_t . d_r),
// w_depth[r][t] = max(0, n_t . d_r)^sharpness, inv_wsum[t] = 1 / sum_r w
__global__ void weights_kernel(const float4 *dirs, int R, const float4 *texdir, float sharpness,
                               float *w_color, float *w_depth) {
    const int total = R * 320;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int r = i / 320, t = i - r * 320;
        const float4 d = dirs[r], n = texdir[t];
        const float c = fmaxf(dot3(n.x, n.y, n.z, d.x, d.y, d.z), 0.0f);
        if (t < 64)
            w_color[r * 64 + t] = c;
        else
            w_depth[r * 256 + (t - 64)] = powf(c, sharpness);
    }
}

__global__ void wsum_kernel(int R, const float *w_color, const float *w_depth, float *inv_wsum) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 320) return;
    float s = 0.f;
    if (t < 64)
        for (int r = 0; r < R; ++r) s += w_color[r * 64 + t];
    else
        for (int r = 0; r < R; ++r) s += w_depth[r * 256 + (t - 64)];
    inv_wsum[t] = s > 0.f ? 1.0f / s : 0.0f;
}

size_t blend_smem_bytes(int R) {
    const size_t w = size_t(2) * W_CHUNK * 4;
    const size_t cores = size_t(BP) * (64 + 256) * 4;
    return size_t(R) * (RGB_STRIDE + DEP_STRIDE) * 4 + (w > cores ? w : cores);
}

template <class K>
int resident_blocks(K kernel, int threads, size_t smem) {
    int n = 0;
    check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem),
               "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
    return n > 0 ? n : 1;
}

template <int SHADOW, int LEAFV, int MINB, int PP, int WIDTH>
void launch_trace_t(const ps_trace_params &p, int sms, cudaStream_t s, bool sm_sized) {
    if (sm_sized) {
        trace_kernel<SHADOW, LEAFV, MINB, PP, WIDTH, 1024><<<sms, 1024, 0, s>>>(p);
        return;
    }
    const int per_sm = resident_blocks(trace_kernel<SHADOW, LEAFV, MINB, PP, WIDTH>, THREADS, 0);
    trace_kernel<SHADOW, LEAFV, MINB, PP, WIDTH><<<sms * per_sm, THREADS, 0, s>>>(p);
}

// two 640-thread CTAs per SM (40 warps at <= 48 registers) on all but the
// reserved SMs
template <int SHADOW, int LEAFV, int PP, int WIDTH, int CLAIM = 0>
void launch_trace_640(const ps_trace_params &p, int sms, cudaStream_t s) {
    static const int carve = [] {  // tuning knob: L1 / shared-memory carveout (percent)
        const char *e = getenv("PS_L1_CARVE");
        return e ? atoi(e) : -1;
    }();
    static bool set = false;
    if (carve >= 0 && !set) {
        check_cuda(cudaFuncSetAttribute(trace_kernel<SHADOW, LEAFV, 1, PP, WIDTH, 640, 0, CLAIM>,
                                        cudaFuncAttributePreferredSharedMemoryCarveout, carve),
                   "carveout");
        set = true;
    }
    trace_kernel<SHADOW, LEAFV, 1, PP, WIDTH, 640, 0, CLAIM><<<2 * sms, 640, 0, s>>>(p);
}

template <int SHADOW, int MINB>
void launch_trace_ww(const ps_trace_params &p, int sms, cudaStream_t s) {
    const int per_sm = resident_blocks(trace_ww_kernel<SHADOW, MINB>, THREADS, 0);
    trace_ww_kernel<SHADOW, MINB><<<sms * per_sm, THREADS, 0, s>>>(p);
}

template <int SHADOW>
void launch_trace_s(const ps_trace_params &p, int variant, int sms, cudaStream_t s, bool big) {
    if (p.bvh_width == 3) {  // BVH4, origin-relative fp16 boxes (WIDTH 17)
        switch (variant) {
            case 64: launch_trace_640<SHADOW, 0, 4, 17>(p, sms, s); break;
            case 65: launch_trace_640<SHADOW, 0, 2, 17>(p, sms, s); break;
            case 90: {  // traversal statistics (tuning only)
                trace_kernel<SHADOW, 0, 1, 12, 17, 640, 1><<<2 * sms, 640, 0, s>>>(p);
                break;
            }
            default: launch_trace_640<SHADOW, 0, 12, 17>(p, sms, s); break;
        }
        return;
    }
    if (p.bvh_width == 8) {  // BVH8, quantised boxes (WIDTH 16)
        switch (variant) {
            case 64: launch_trace_640<SHADOW, 0, 4, 16>(p, sms, s); break;
            case 65: launch_trace_640<SHADOW, 0, 2, 16>(p, sms, s); break;
            case 90: {  // traversal statistics (tuning only)
                trace_kernel<SHADOW, 0, 1, 12, 16, 640, 1><<<2 * sms, 640, 0, s>>>(p);
                break;
            }
            default: launch_trace_640<SHADOW, 0, 12, 16>(p, sms, s); break;
        }
        return;
    }
    if (p.bvh_width == 5) {
        switch (variant) {
            case 11: launch_trace_t<SHADOW, 1, 4, 0, 5>(p, sms, s, big); break;
            case 12: launch_trace_t<SHADOW, 1, 1, 0, 5>(p, sms, s, big); break;
            // fp16 boxes, octant tests, two 256-bit loads per node
            case 64: launch_trace_640<SHADOW, 0, 4, 23>(p, sms, s); break;  // 2x4x4 tiles
            case 86: launch_trace_640<SHADOW, 0, 4, 3>(p, sms, s); break;
            case 70: launch_trace_640<SHADOW, 0, 12, 18>(p, sms, s); break;  // word selects
            case 71: launch_trace_t<SHADOW, 0, 1, 12, 3>(p, sms, s, true); break;  // 1024 x 1
            case 72: launch_trace_640<SHADOW, 1, 12, 3>(p, sms, s); break;  // leaf pairs
            case 65: launch_trace_640<SHADOW, 0, 2, 23>(p, sms, s); break;  // 4x4x2 tiles
            case 66: launch_trace_640<SHADOW, 0, 4, 19>(p, sms, s); break;  // fp32 slabs
            case 67: launch_trace_640<SHADOW, 0, 2, 19>(p, sms, s); break;
            case 87: launch_trace_640<SHADOW, 0, 2, 3>(p, sms, s); break;
            // CTA-level claiming: one tile x CLAIM neighbouring directions
            case 80: launch_trace_640<SHADOW, 0, 12, 3, 16>(p, sms, s); break;
            case 81: launch_trace_640<SHADOW, 0, 12, 3, 32>(p, sms, s); break;
            case 82: launch_trace_640<SHADOW, 0, 12, 3, 64>(p, sms, s); break;
            case 83: launch_trace_640<SHADOW, 0, 12, 3, 256>(p, sms, s); break;
            // speculative while-while traversal (parked leaves, warp vote)
            case 84: launch_trace_640<SHADOW, 0, 12, 19>(p, sms, s); break;
            case 88: launch_trace_640<SHADOW, 0, 12, 20>(p, sms, s); break;  // word selects
            case 89: launch_trace_640<SHADOW, 0, 12, 21>(p, sms, s); break;  // vote >= 3/4
            case 91: launch_trace_640<SHADOW, 0, 12, 22>(p, sms, s); break;  // vote >= 1/2
            case 92: launch_trace_640<SHADOW, 0, 12, 23>(p, sms, s); break;  // half2 slabs
            // traversal statistics of 84 / 92 (tuning only, ps_trace_stats)
            case 93: launch_trace_640<SHADOW, 0, 12, 24>(p, sms, s); break;
            case 94: launch_trace_640<SHADOW, 0, 12, 25>(p, sms, s); break;
            case 85: launch_trace_640<SHADOW, 0, 12, 3>(p, sms, s); break;  // plain loop
            // default: packed half2 slab tests (WIDTH 23), conservative, so the
            // nearest hits match the fp32 test's; with the scene-centred BVH
            // frame C4 traces in 3.960 vs 4.004 ms (84 = fp32 slabs) on one
            // frame's rotation, 4.042 vs 4.050 on the bench's; directions with
            // a near-zero component take the fp32 test (warp-uniform)
            default: launch_trace_640<SHADOW, 0, 12, 23>(p, sms, s); break;
        }
        return;
    }
    if (p.bvh_width == 4) {
        switch (variant) {
            case 0: launch_trace_t<SHADOW, 0, 1, 0, 4>(p, sms, s, big); break;
            case 10: launch_trace_t<SHADOW, 0, 4, 0, 4>(p, sms, s, big); break;
            case 11: launch_trace_t<SHADOW, 1, 4, 0, 4>(p, sms, s, big); break;
            case 30: launch_trace_t<SHADOW, 1, 1, 1, 4>(p, sms, s, big); break;
            case 32: launch_trace_t<SHADOW, 1, 1, 2, 4>(p, sms, s, big); break;
            case 33: launch_trace_t<SHADOW, 1, 1, 3, 4>(p, sms, s, big); break;
            case 35: launch_trace_t<SHADOW, 1, 1, 5, 4>(p, sms, s, big); break;
            case 36: launch_trace_t<SHADOW, 1, 1, 6, 4>(p, sms, s, big); break;
            case 37: launch_trace_t<SHADOW, 1, 1, 7, 4>(p, sms, s, big); break;
            case 38: launch_trace_t<SHADOW, 1, 1, 8, 4>(p, sms, s, big); break;
            case 39: launch_trace_t<SHADOW, 1, 1, 9, 4>(p, sms, s, big); break;
            case 40: launch_trace_t<SHADOW, 1, 1, 10, 4>(p, sms, s, big); break;
            case 41: launch_trace_t<SHADOW, 1, 1, 11, 4>(p, sms, s, big); break;  // 1x4x8
            case 42: launch_trace_t<SHADOW, 1, 1, 12, 4>(p, sms, s, big); break;  // 2x2x8
            case 43: launch_trace_t<SHADOW, 1, 1, 13, 4>(p, sms, s, big); break;  // 2x8x2
            case 44: launch_trace_t<SHADOW, 0, 1, 4, 4>(p, sms, s, big); break;   // 2x4x4, seq leaf
            case 45: launch_trace_t<SHADOW, 1, 4, 4, 4>(p, sms, s, big); break;   // 2x4x4, 4 CTAs/SM
            case 46: launch_trace_t<SHADOW, 0, 1, 12, 4>(p, sms, s, big); break;  // 2x2x8, seq leaf
            case 47: launch_trace_t<SHADOW, 0, 1, 11, 4>(p, sms, s, big); break;  // 1x4x8, seq leaf
            case 48: launch_trace_t<SHADOW, 2, 1, 12, 4>(p, sms, s, big); break;  // 2x2x8, 4-wide leaf
            case 49: launch_trace_t<SHADOW, 2, 1, 4, 4>(p, sms, s, big); break;   // 2x4x4, 4-wide leaf
            case 50: launch_trace_t<SHADOW, 0, 1, 2, 4>(p, sms, s, big); break;   // 4x4x2, seq leaf
            // octant-specialised node tests: per node (6) / per ray (7)
            case 56: launch_trace_t<SHADOW, 0, 1, 12, 6>(p, sms, s, big); break;  // 2x2x8
            case 57: launch_trace_t<SHADOW, 0, 1, 12, 7>(p, sms, s, big); break;
            case 58: launch_trace_t<SHADOW, 0, 1, 4, 6>(p, sms, s, big); break;   // 2x4x4
            case 59: launch_trace_t<SHADOW, 0, 1, 4, 7>(p, sms, s, big); break;
            case 60: launch_trace_t<SHADOW, 0, 1, 2, 6>(p, sms, s, big); break;   // 4x4x2
            case 61: launch_trace_t<SHADOW, 0, 5, 12, 6>(p, sms, s, false); break;  // 40 warps/SM
            case 62: launch_trace_t<SHADOW, 0, 6, 12, 6>(p, sms, s, false); break;  // 48 warps/SM
            case 63: launch_trace_640<SHADOW, 0, 12, 6>(p, sms, s); break;  // 2 x 640 per SM
            case 64: launch_trace_640<SHADOW, 0, 4, 6>(p, sms, s); break;
            case 65: launch_trace_640<SHADOW, 0, 2, 6>(p, sms, s); break;
            case 90: {  // traversal statistics (tuning only)
                const int per_sm = resident_blocks(trace_kernel<SHADOW, 1, 1, 0, 4, THREADS, 1>, THREADS, 0);
                trace_kernel<SHADOW, 1, 1, 0, 4, THREADS, 1><<<sms * per_sm, THREADS, 0, s>>>(p);
                break;
            }
            case 34: launch_trace_t<SHADOW, 1, 1, 4, 4>(p, sms, s, big); break;
            default: launch_trace_t<SHADOW, 1, 1, 0, 4>(p, sms, s, big); break;
        }
        return;
    }
    switch (variant) {
        case 20: launch_trace_ww<SHADOW, 1>(p, sms, s); break;
        case 22: launch_trace_ww<SHADOW, 4>(p, sms, s); break;
        case 30: launch_trace_t<SHADOW, 1, 1, 1, 2>(p, sms, s, big); break;
        case 0: launch_trace_t<SHADOW, 0, 1, 0, 2>(p, sms, s, big); break;
        case 10: launch_trace_t<SHADOW, 0, 4, 0, 2>(p, sms, s, big); break;
        default: launch_trace_t<SHADOW, 1, 1, 0, 2>(p, sms, s, big); break;
    }
}

void launch_trace(const ps_trace_params &p, int variant, int sms, cudaStream_t s, bool big) {
    switch (p.shadow_mode) {
        case PS_SHADOW_NONE: launch_trace_s<PS_SHADOW_NONE>(p, variant, sms, s, big); break;
        case PS_SHADOW_RAYS: launch_trace_s<PS_SHADOW_RAYS>(p, variant, sms, s, big); break;
        default: launch_trace_s<PS_SHADOW_MAP>(p, variant, sms, s, big); break;
    }
    check_launch("trace_kernel");
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" {

// traversal statistics of PS_TRACE_VARIANT=90 (tuning only): {inner-node
// visits, leaf visits, triangle tests, rays}; reset after reading
int ps_trace_stats(unsigned long long *out) {
    PS_ABI_BEGIN
    check_cuda(cudaMemcpyFromSymbol(out, trav::g_trav_stats, sizeof(unsigned long long) * 4),
               "read stats");
    const unsigned long long zero[4] = {0, 0, 0, 0};
    check_cuda(cudaMemcpyToSymbol(trav::g_trav_stats, zero, sizeof(zero)), "reset stats");
    PS_ABI_END
}

size_t ps_blend_weight_image_floats(int32_t rays_per_probe) {
    return weight_image_floats(rays_per_probe);
}

int ps_blend_weights(const float *ray_dirs, int32_t rays_per_probe, const float *texdir,
                     float sharpness, float *w_color, float *w_depth, float *inv_wsum,
                     float *w_image, void *stream) {
    PS_ABI_BEGIN
    if (rays_per_probe < 1) fail(PS_ERR_VALUE, "rays_per_probe must be >= 1");
    auto s = as_stream(stream);
    const int total = rays_per_probe * 320;
    weights_kernel<<<unsigned(ceil_div(total, 256)), 256, 0, s>>>(
        reinterpret_cast<const float4 *>(ray_dirs), rays_per_probe,
        reinterpret_cast<const float4 *>(texdir), sharpness, w_color, w_depth);
    check_launch("weights_kernel");
    wsum_kernel<<<2, 256, 0, s>>>(rays_per_probe, w_color, w_depth, inv_wsum);
    check_launch("wsum_kernel");
    if (w_image) {
        if (rays_per_probe % 8) fail(PS_ERR_VALUE, "the weight image needs rays_per_probe % 8 == 0");
        launch_weight_image(w_color, w_depth, rays_per_probe, w_image, s);
    }
    PS_ABI_END
}

int ps_trace_blend(const ps_trace_params *params, void *stream) {
    PS_ABI_BEGIN
    if (!params) fail(PS_ERR_VALUE, "params must not be NULL");
    const ps_trace_params &p = *params;
    if (p.nx < 1 || p.ny < 1 || p.nz < 1) fail(PS_ERR_VALUE, "volume dims must be >= 1");
    const int64_t n = int64_t(p.nx) * p.ny * p.nz;
    if (p.probe_begin < 0 || p.probe_end > n || p.probe_begin > p.probe_end)
        fail(PS_ERR_INDEX, "probe range outside the volume");
    if (p.rays_per_probe < 1 || p.rays_per_probe > 2048) fail(PS_ERR_VALUE, "rays_per_probe in [1, 2048]");
    if (p.light_count < 0 || p.light_count > 30) fail(PS_ERR_VALUE, "light_count in [0, 30]");
    if (p.probes_per_row_color < 1 || p.probes_per_row_vis < 1) fail(PS_ERR_LAYOUT, "bad atlas layout");
    if (p.shadow_mode < PS_SHADOW_NONE || p.shadow_mode > PS_SHADOW_MAP) fail(PS_ERR_VALUE, "bad shadow_mode");
    if (p.bvh_width != 2 && p.bvh_width != 3 && p.bvh_width != 4 && p.bvh_width != 5 &&
        p.bvh_width != 8)
        fail(PS_ERR_VALUE, "bvh_width must be 2, 4, 5 (BVH4 with fp16 boxes) or 8 (BVH8, 8-bit boxes)");
    if (p.bvh_width == 4 && (p.shadow_mode == PS_SHADOW_RAYS || false)) {
        // any-hit shadow rays use the same templated traversal: fine
    }
    if (p.shadow_mode == PS_SHADOW_MAP && p.light_count > 0 &&
        (p.shadow_map_size < 1 || p.shadow_map_size > 4096 || !p.shadow_maps))
        fail(PS_ERR_VALUE, "shadow map size / buffer missing");
    if (!p.records || !p.work_counter) fail(PS_ERR_VALUE, "records / work_counter scratch missing");
    const int64_t nloc = p.probe_end - p.probe_begin;
    auto s = as_stream(stream);
    const int sms = sm_count();
    const int passes = p.passes ? p.passes : 7;
    if (p.shadow_texel_begin < 0 || p.shadow_texel_end < 0 ||
        (p.shadow_texel_end > 0 && p.shadow_texel_end < p.shadow_texel_begin))
        fail(PS_ERR_VALUE, "bad shadow texel range");
    // pass 0: shadow maps
    if ((passes & 1) && p.shadow_mode == PS_SHADOW_MAP && p.light_count > 0) {
        const int64_t all = int64_t(p.light_count) * 6 * p.shadow_map_size * p.shadow_map_size;
        const int64_t end = p.shadow_texel_end > 0 && p.shadow_texel_end < all ? p.shadow_texel_end : all;
        const int64_t texels = end > p.shadow_texel_begin ? end - p.shadow_texel_begin : 0;
        const unsigned blocks = unsigned(std::max<int64_t>(
            1, std::min<int64_t>(ceil_div(texels, 256), int64_t(sms) * 32)));
        if (p.bvh_width == 3)
            shadow_map_kernel<17><<<blocks, 256, 0, s>>>(p);
        else if (p.bvh_width == 8)
            shadow_map_kernel<16><<<blocks, 256, 0, s>>>(p);
        else if (p.bvh_width == 5 && getenv("PS_SHADOW_PLAIN"))
            shadow_map_kernel<3><<<blocks, 256, 0, s>>>(p);
        else if (p.bvh_width == 5 && getenv("PS_SHADOW_HALF"))  // half2 slab tests (tuning:
            shadow_map_kernel<23><<<blocks, 256, 0, s>>>(p);      // 0.156 vs 0.151 ms at C4)
        else if (p.bvh_width == 5)  // speculative while-while traversal (traverse_spec)
            shadow_map_kernel<19><<<blocks, 256, 0, s>>>(p);
        else if (p.bvh_width == 4)
            shadow_map_kernel<6><<<blocks, 256, 0, s>>>(p);  // octant-specialised BVH4 tests
        else
            shadow_map_kernel<2><<<blocks, 256, 0, s>>>(p);
        check_launch("shadow_map_kernel");
    }
    if (nloc == 0) return PS_OK;
    // pass 1: persistent trace with dynamic chunk claiming
    if (passes & 2) {
        check_cuda(cudaMemsetAsync(p.work_counter, 0, sizeof(uint32_t), s), "memset counter");
        // PS_TRACE_VARIANT (tuning knob): leaf fetch 0 = sequential, 1 = pairs,
        // 2 = four in flight; +10 = cap registers for 4 resident CTAs per SM
        static const int forced = [] {
            const char *e = getenv("PS_TRACE_VARIANT");
            return e ? atoi(e) : -1;
        }();
        // default (BVH4): one direction per warp over the deepest probe tile the
        // slab holds -- 2x2x8 (C4 trace + blend 6.18 ms), 2x4x4 (6.39), 4x4x2 --
        // with leaves tested one triangle at a time (LEAFV 0 beats pairs once the
        // warp's rays are coherent) and octant-specialised node tests picked per
        // node (trace 5.39 -> 5.27 ms; one traversal per octant, 57, thrashes
        // the instruction cache: 7.58 ms), launched as two 640-thread CTAs per
        // SM at <= 48 registers (40 warps instead of 32: 5.27 -> 5.08 ms)
        const int64_t plane = int64_t(p.nx) * p.ny;
        const int64_t depth = (p.probe_end - 1) / plane - p.probe_begin / plane + 1;
        const int variant = forced >= 0 ? forced : depth >= 8 ? 63 : depth >= 4 ? 64 : 65;
        const int keep = p.reserve_sms > 0 && p.reserve_sms < sms / 2 ? p.reserve_sms : 0;
        launch_trace(p, variant, sms - keep, s, keep > 0);
    }
    if (!(passes & 4)) return PS_OK;
    // pass 2: blend -- tcgen05 tensor cores (ps_blend_tc.cu), or the CUDA-core kernel
    if (blend_tc_usable(p)) {
        launch_blend_tc(p, nloc, s);
        return PS_OK;
    }
    const size_t smem = blend_smem_bytes(p.rays_per_probe);
    static bool attr_set = false;
    if (!attr_set) {
        check_cuda(cudaFuncSetAttribute(blend_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        200 * 1024),
                   "cudaFuncSetAttribute");
        attr_set = true;
    }
    if (smem > 200 * 1024) fail(PS_ERR_VALUE, "too many rays per probe for shared memory");
    blend_kernel<<<unsigned(ceil_div(nloc, BP)), THREADS, smem, s>>>(p);
    check_launch("blend_kernel");
    PS_ABI_END
}

}  // extern "C"
