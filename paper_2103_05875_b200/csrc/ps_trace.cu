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

#include "ps_common.cuh"

namespace ps {
namespace {

constexpr int THREADS = 256;
constexpr int STACK = 64;
constexpr float RAY_EPS = 1e-6f;  // selection.py:22

struct Ray {
    float ox, oy, oz, dx, dy, dz;
};

__device__ __forceinline__ float3 f3(float4 v) { return make_float3(v.x, v.y, v.z); }

__device__ __forceinline__ float dot3(float ax, float ay, float az, float bx, float by, float bz) {
    return fmaf(az, bz, fmaf(ay, by, ax * bx));
}

// Moller-Trumbore with the reference's epsilons; returns t or +inf
__device__ __forceinline__ float tri_hit(const Ray &r, float4 v0, float4 e1, float4 e2) {
    const float px = r.dy * e2.z - r.dz * e2.y;
    const float py = r.dz * e2.x - r.dx * e2.z;
    const float pz = r.dx * e2.y - r.dy * e2.x;
    const float det = dot3(e1.x, e1.y, e1.z, px, py, pz);
    if (!(fabsf(det) > RAY_EPS)) return INFINITY;
    const float inv = 1.0f / det;
    const float tx = r.ox - v0.x, ty = r.oy - v0.y, tz = r.oz - v0.z;
    const float u = dot3(tx, ty, tz, px, py, pz) * inv;
    const float qx = ty * e1.z - tz * e1.y;
    const float qy = tz * e1.x - tx * e1.z;
    const float qz = tx * e1.y - ty * e1.x;
    const float v = dot3(r.dx, r.dy, r.dz, qx, qy, qz) * inv;
    const float t = dot3(e2.x, e2.y, e2.z, qx, qy, qz) * inv;
    const bool ok = (u >= -RAY_EPS) && (v >= -RAY_EPS) && (u + v <= 1.0f + RAY_EPS) && (t > RAY_EPS);
    return ok ? t : INFINITY;
}

// slab test against the two child boxes of a node
__device__ __forceinline__ void node_hits(const float4 *nodes, int node, float ix, float iy,
                                          float iz, float oix, float oiy, float oiz, float tmax,
                                          bool &h0, bool &h1, float &t0, float &t1, int &c0,
                                          int &c1) {
    const float4 a = __ldg(nodes + 4 * node + 0);
    const float4 b = __ldg(nodes + 4 * node + 1);
    const float4 z = __ldg(nodes + 4 * node + 2);
    const float4 c = __ldg(nodes + 4 * node + 3);
    // child 0
    float lx = fmaf(a.x, ix, -oix), hx = fmaf(a.y, ix, -oix);
    float ly = fmaf(a.z, iy, -oiy), hy = fmaf(a.w, iy, -oiy);
    float lz = fmaf(z.x, iz, -oiz), hz = fmaf(z.y, iz, -oiz);
    float n0 = fmaxf(fmaxf(fminf(lx, hx), fminf(ly, hy)), fmaxf(fminf(lz, hz), 0.0f));
    float f0 = fminf(fminf(fmaxf(lx, hx), fmaxf(ly, hy)), fminf(fmaxf(lz, hz), tmax));
    // child 1
    lx = fmaf(b.x, ix, -oix);
    hx = fmaf(b.y, ix, -oix);
    ly = fmaf(b.z, iy, -oiy);
    hy = fmaf(b.w, iy, -oiy);
    lz = fmaf(z.z, iz, -oiz);
    hz = fmaf(z.w, iz, -oiz);
    float n1 = fmaxf(fmaxf(fminf(lx, hx), fminf(ly, hy)), fmaxf(fminf(lz, hz), 0.0f));
    float f1 = fminf(fminf(fmaxf(lx, hx), fmaxf(ly, hy)), fminf(fmaxf(lz, hz), tmax));
    h0 = n0 <= f0;
    h1 = n1 <= f1;
    t0 = n0;
    t1 = n1;
    c0 = __float_as_int(c.x);
    c1 = __float_as_int(c.y);
}

// Nearest hit (ANY_HIT = false) or occlusion test (ANY_HIT = true) with a
// per-thread stack.  Returns the hit record slot (or -1) and the distance.
template <bool ANY_HIT>
__device__ int traverse(const float4 *__restrict__ nodes, const float4 *__restrict__ tris,
                        const Ray &r, float tmax, float &t_best) {
    // reciprocal direction; tiny components replaced so the slabs stay finite
    const float sx = fabsf(r.dx) < 1e-12f ? copysignf(1e-12f, r.dx) : r.dx;
    const float sy = fabsf(r.dy) < 1e-12f ? copysignf(1e-12f, r.dy) : r.dy;
    const float sz = fabsf(r.dz) < 1e-12f ? copysignf(1e-12f, r.dz) : r.dz;
    const float ix = 1.0f / sx, iy = 1.0f / sy, iz = 1.0f / sz;
    const float oix = r.ox * ix, oiy = r.oy * iy, oiz = r.oz * iz;
    int stack[STACK];
    int sp = 0;
    int node = 0;
    int hit_slot = -1;
    t_best = tmax;
    while (true) {
        if (node >= 0) {
            bool h0, h1;
            float t0, t1;
            int c0, c1;
            node_hits(nodes, node, ix, iy, iz, oix, oiy, oiz, t_best, h0, h1, t0, t1, c0, c1);
            if (h0 && h1) {
                const bool swap = t1 < t0;
                node = swap ? c1 : c0;
                stack[sp++] = swap ? c0 : c1;
                continue;
            }
            if (h0 || h1) {
                node = h0 ? c0 : c1;
                continue;
            }
        } else {
            for (int s = ~node;; ++s) {
                const float4 v0 = __ldg(tris + 3 * s);
                const int prim = __float_as_int(v0.w);
                if (prim < 0) break;
                const float t = tri_hit(r, v0, __ldg(tris + 3 * s + 1), __ldg(tris + 3 * s + 2));
                if (t < t_best) {
                    t_best = t;
                    hit_slot = s;
                    if (ANY_HIT) return hit_slot;
                }
            }
        }
        if (sp == 0) break;
        node = stack[--sp];
    }
    return hit_slot;
}

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

template <int SHADOW>
__device__ Shade shade_ray(const ps_trace_params &p, const float4 *nodes, const float4 *tris,
                           const Ray &ray) {
    Shade s;
    float t;
    const int slot = traverse<false>(nodes, tris, ray, INFINITY, t);
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
    const float hx = fmaf(ray.dx, t, ray.ox), hy = fmaf(ray.dy, t, ray.oy), hz = fmaf(ray.dz, t, ray.oz);
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
            if (traverse<true>(nodes, tris, sh, dist, ts) >= 0) continue;
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

// ---- pass 0: cube distance maps traced from each light ------------------------------
// face f: axis a = f / 2, sign = f % 2 ? -1 : +1, (b, c) = ((a+1)%3, (a+2)%3);
// texel (i, j): direction e_a*sign + e_b*u + e_c*w with u = (i+.5)/S*2-1,
// w = (j+.5)/S*2-1, normalised; value = nearest hit distance (inf on a miss).
__global__ void __launch_bounds__(256) shadow_map_kernel(ps_trace_params prm) {
    const int S = prm.shadow_map_size;
    const int64_t per_light = int64_t(6) * S * S;
    const int64_t total = per_light * prm.light_count;
    const float4 *nodes = reinterpret_cast<const float4 *>(prm.nodes);
    const float4 *tris = reinterpret_cast<const float4 *>(prm.tris);
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int l = int(idx / per_light);
        const int rem = int(idx - int64_t(l) * per_light);
        const int f = rem / (S * S);
        const int j = (rem / S) % S, i = rem % S;
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
        const int slot = traverse<false>(nodes, tris, ray, INFINITY, t);
        prm.shadow_maps[idx] = slot < 0 ? INFINITY : t;
    }
}

// ---- pass 1: probe rays -> per-ray records (persistent, dynamic chunks) -----------------
// A warp claims 32 consecutive rays of one probe (neighbouring directions in
// the coherence-ordered set) from a global counter, traces + shades them and
// writes {rgb, depth}.  Dynamic claiming keeps every SM busy regardless of the
// large per-direction cost differences.
template <int SHADOW>
__global__ void __launch_bounds__(THREADS) trace_kernel(ps_trace_params prm) {
    const float4 *nodes = reinterpret_cast<const float4 *>(prm.nodes);
    const float4 *tris = reinterpret_cast<const float4 *>(prm.tris);
    const float4 *dirs = reinterpret_cast<const float4 *>(prm.ray_dirs);
    const int R = prm.rays_per_probe;
    const int64_t nloc = int64_t(prm.probe_end) - prm.probe_begin;
    const int64_t total_rays = nloc * R;
    const int64_t chunks_per_probe = (R + 31) / 32;
    const int64_t total_chunks = nloc * chunks_per_probe;
    const int lane = threadIdx.x & 31;
    float4 *records = reinterpret_cast<float4 *>(prm.records);
    while (true) {
        uint32_t task = 0;
        if (lane == 0) task = atomicAdd(prm.work_counter, 1u);
        task = __shfl_sync(0xffffffffu, task, 0);
        if (int64_t(task) >= total_chunks) break;
        const int64_t q = int64_t(task) / chunks_per_probe;
        const int r = int(int64_t(task) - q * chunks_per_probe) * 32 + lane;
        if (r >= R) continue;
        const int64_t p = prm.probe_begin + q;
        const int64_t i = p % prm.nx, j = (p / prm.nx) % prm.ny, k = p / (int64_t(prm.nx) * prm.ny);
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
        const Shade s = shade_ray<SHADOW>(prm, nodes, tris, ray);
        const int64_t ray_id = q * R + r;
        records[ray_id] = make_float4(s.r, s.g, s.b, s.depth);
        if (prm.ray_records) {
            float4 *rec = reinterpret_cast<float4 *>(prm.ray_records) + 2 * ray_id;
            rec[0] = make_float4(s.r, s.g, s.b, s.depth);
            rec[1] = make_float4(s.t, __int_as_float(s.prim), __int_as_float(s.shadow_mask), 0.f);
        }
        (void)total_rays;
    }
}

// ---- pass 2: DDGI blend of P probes per CTA ---------------------------------------------
template <int P>
__global__ void __launch_bounds__(THREADS) blend_kernel(ps_trace_params prm) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int R = prm.rays_per_probe;
    float4 *s_rgb = reinterpret_cast<float4 *>(smem_raw);            // R * P   [r][q]
    float2 *s_dep = reinterpret_cast<float2 *>(s_rgb + R * P);       // R * P   [r][q] (d, d^2)
    uint32_t *s_ccore = reinterpret_cast<uint32_t *>(s_dep + R * P); // P * 64
    uint32_t *s_vcore = s_ccore + P * 64;                            // P * 256

    const int tid = threadIdx.x;
    const int64_t p0 = int64_t(prm.probe_begin) + int64_t(blockIdx.x) * P;
    const int64_t left = int64_t(prm.probe_end) - p0;
    const int nq = int(left < P ? left : P);
    const float4 *records = reinterpret_cast<const float4 *>(prm.records) +
                            (p0 - prm.probe_begin) * R;
    for (int g = tid; g < P * R; g += THREADS) {
        const int q = g / R, r = g - q * R;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (q < nq) v = __ldcs(records + g);  // streamed once
        s_rgb[r * P + q] = make_float4(v.x, v.y, v.z, 0.f);
        s_dep[r * P + q] = make_float2(v.w, v.w * v.w);
    }
    __syncthreads();

    // ---- irradiance (64 texels x P probes) --------------------------------------------
    {
        constexpr int QPT = (P + 3) / 4;  // probes per thread
        const int t = tid & 63, qg = tid >> 6;
        float acc[QPT][3];
#pragma unroll
        for (int a = 0; a < QPT; ++a) acc[a][0] = acc[a][1] = acc[a][2] = 0.f;
        const float *wc = prm.w_color + t;
        for (int r = 0; r < R; ++r) {
            const float w = __ldg(wc + r * 64);
#pragma unroll
            for (int a = 0; a < QPT; ++a) {
                const int q = qg + 4 * a;
                if (q < P) {
                    const float4 L = s_rgb[r * P + q];
                    acc[a][0] = fmaf(w, L.x, acc[a][0]);
                    acc[a][1] = fmaf(w, L.y, acc[a][1]);
                    acc[a][2] = fmaf(w, L.z, acc[a][2]);
                }
            }
        }
        const float inv = __ldg(prm.inv_wsum + t);
        const float h = prm.hysteresis;
        const float qs = prm.irradiance_scale > 0.f ? 1.0f / prm.irradiance_scale : 0.f;
#pragma unroll
        for (int a = 0; a < QPT; ++a) {
            const int q = qg + 4 * a;
            if (q >= nq) continue;
            float *st = prm.irradiance + ((p0 - prm.probe_begin + q) * 64 + t) * 3;
            uint32_t texel = 0;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                float v = acc[a][c] * inv;
                if (inv == 0.f) v = st[c];  // no ray sees this texel: keep the state
                else if (h != 0.f) v = fmaf(h, st[c] - v, v);
                st[c] = v;
                float x = fminf(fmaxf(v * qs, 0.0f), 1.0f);
                texel |= __float2uint_rn(x * 1023.0f) << (10 * c);
            }
            s_ccore[q * 64 + t] = texel;
        }
    }
    // ---- depth moments (256 texels x P probes) ------------------------------------------
    {
        const int t = tid;
        float m1[P], m2[P];
#pragma unroll
        for (int q = 0; q < P; ++q) m1[q] = m2[q] = 0.f;
        const float *wd = prm.w_depth + t;
        for (int r = 0; r < R; ++r) {
            const float w = __ldg(wd + r * 256);
#pragma unroll
            for (int q = 0; q < P; ++q) {
                const float2 d = s_dep[r * P + q];
                m1[q] = fmaf(w, d.x, m1[q]);
                m2[q] = fmaf(w, d.y, m2[q]);
            }
        }
        const float inv = __ldg(prm.inv_wsum + 64 + t);
        const float h = prm.hysteresis;
#pragma unroll
        for (int q = 0; q < P; ++q) {
            if (q >= nq) continue;
            float2 *st = reinterpret_cast<float2 *>(prm.moments) + (p0 - prm.probe_begin + q) * 256 + t;
            float a = m1[q] * inv, b = m2[q] * inv;
            if (inv == 0.f) {
                const float2 o = *st;
                a = o.x;
                b = o.y;
            } else if (h != 0.f) {
                const float2 o = *st;
                a = fmaf(h, o.x - a, a);
                b = fmaf(h, o.y - b, b);
            }
            *st = make_float2(a, b);
            const uint32_t lo = __half_as_ushort(__float2half_rn(a));
            const uint32_t hi = __half_as_ushort(__float2half_rn(b));
            s_vcore[q * 256 + t] = lo | (hi << 16);
        }
    }
    __syncthreads();

    // ---- atlas blocks with guard bands ----------------------------------------------------
    {
        const int ppr = prm.probes_per_row_color;
        const int64_t W = int64_t(ppr) * 10;
        for (int idx = tid; idx < nq * 100; idx += THREADS) {
            const int q = idx / 100, k = idx - q * 100;
            const int r = k / 10, c = k - r * 10;
            const int64_t p = p0 + q;
            const int64_t y0 = (p / ppr) * 10, x0 = (p % ppr) * 10;
            prm.color_atlas[(y0 + r) * W + x0 + c] = s_ccore[q * 64 + guard_source(r, c, 10)];
        }
    }
    {
        const int ppr = prm.probes_per_row_vis;
        const int64_t W = int64_t(ppr) * 18;
        uint32_t *vis = reinterpret_cast<uint32_t *>(prm.vis_atlas);
        for (int idx = tid; idx < nq * 324; idx += THREADS) {
            const int q = idx / 324, k = idx - q * 324;
            const int r = k / 18, c = k - r * 18;
            const int64_t p = p0 + q;
            const int64_t y0 = (p / ppr) * 18, x0 = (p % ppr) * 18;
            vis[(y0 + r) * W + x0 + c] = s_vcore[q * 256 + guard_source(r, c, 18)];
        }
    }
}

// per-frame blend weights: w_color[r][t] = max(0, n_t . d_r),
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

constexpr int PROBES_PER_CTA = 8;

size_t blend_smem_bytes(int R, int P) {
    return size_t(R) * P * 16 + size_t(R) * P * 8 + size_t(P) * (64 + 256) * 4;
}

template <class K>
int resident_blocks(K kernel, int threads, size_t smem) {
    int n = 0;
    check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem),
               "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
    return n > 0 ? n : 1;
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" {

int ps_blend_weights(const float *ray_dirs, int32_t rays_per_probe, const float *texdir,
                     float sharpness, float *w_color, float *w_depth, float *inv_wsum,
                     void *stream) {
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
    if (p.shadow_mode == PS_SHADOW_MAP && p.light_count > 0 &&
        (p.shadow_map_size < 1 || p.shadow_map_size > 4096 || !p.shadow_maps))
        fail(PS_ERR_VALUE, "shadow map size / buffer missing");
    if (!p.records || !p.work_counter) fail(PS_ERR_VALUE, "records / work_counter scratch missing");
    const int64_t nloc = p.probe_end - p.probe_begin;
    if (nloc == 0) return PS_OK;
    auto s = as_stream(stream);
    const int sms = sm_count();
    // pass 0: shadow maps
    if (p.shadow_mode == PS_SHADOW_MAP && p.light_count > 0) {
        const int64_t texels = int64_t(p.light_count) * 6 * p.shadow_map_size * p.shadow_map_size;
        const unsigned blocks = unsigned(std::min<int64_t>(ceil_div(texels, 256), int64_t(sms) * 32));
        shadow_map_kernel<<<blocks, 256, 0, s>>>(p);
        check_launch("shadow_map_kernel");
    }
    // pass 1: persistent trace with dynamic chunk claiming
    check_cuda(cudaMemsetAsync(p.work_counter, 0, sizeof(uint32_t), s), "memset counter");
    {
        int per_sm;
        switch (p.shadow_mode) {
            case PS_SHADOW_NONE:
                per_sm = resident_blocks(trace_kernel<PS_SHADOW_NONE>, THREADS, 0);
                trace_kernel<PS_SHADOW_NONE><<<sms * per_sm, THREADS, 0, s>>>(p);
                break;
            case PS_SHADOW_RAYS:
                per_sm = resident_blocks(trace_kernel<PS_SHADOW_RAYS>, THREADS, 0);
                trace_kernel<PS_SHADOW_RAYS><<<sms * per_sm, THREADS, 0, s>>>(p);
                break;
            default:
                per_sm = resident_blocks(trace_kernel<PS_SHADOW_MAP>, THREADS, 0);
                trace_kernel<PS_SHADOW_MAP><<<sms * per_sm, THREADS, 0, s>>>(p);
                break;
        }
        check_launch("trace_kernel");
    }
    // pass 2: blend
    const size_t smem = blend_smem_bytes(p.rays_per_probe, PROBES_PER_CTA);
    static bool attr_set = false;
    if (!attr_set) {
        check_cuda(cudaFuncSetAttribute(blend_kernel<PROBES_PER_CTA>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024),
                   "cudaFuncSetAttribute");
        attr_set = true;
    }
    if (smem > 200 * 1024) fail(PS_ERR_VALUE, "too many rays per probe for shared memory");
    blend_kernel<PROBES_PER_CTA><<<unsigned(ceil_div(nloc, PROBES_PER_CTA)), THREADS, smem, s>>>(p);
    check_launch("blend_kernel");
    PS_ABI_END
}

}  // extern "C"
