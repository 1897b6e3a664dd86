// BVH traversal shared by the probe tracer (ps_trace.cu) and the PVS kernel
// (ps_pvs.cu): ray/triangle test with the reference's semantics
// (selection.py:123-139), BVH2 and BVH4 node tests, stack traversal.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cuda_fp16.h>

namespace ps {
namespace trav {

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
    // MUFU.RCP alone (<= 1 ulp): |det| > 1e-6 keeps it far from the range
    // where the IEEE division's slow path matters, so the rn fix-up and its
    // slow-path branch are dropped from every triangle test
    const float inv = __fdividef(1.0f, det);
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

// BVH4 node: four child slab tests from one 128-byte node (SoA boxes), the
// hit children sorted by entry distance with a 5-comparator network.
constexpr int EMPTY_CHILD = 0x7fffffff;

__device__ __forceinline__ void cswap(float &da, int &ca, float &db, int &cb) {
    const bool sw = db < da;
    const float td = sw ? db : da;
    const int tc = sw ? cb : ca;
    db = sw ? da : db;
    cb = sw ? ca : cb;
    da = td;
    ca = tc;
}

// 32-byte read-only load (sm_100 LDG.256): a 128-byte BVH4 node is four of
// them instead of seven 16-byte loads; with coherent warps (one ray direction
// over a probe tile) the lanes share node lines, so fewer load instructions
// per node are fewer L1 wavefronts
__device__ __forceinline__ void ldg256(const void *p, float (&v)[8]) {
    asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
          "=f"(v[7])
        : "l"(p));
}

__device__ __forceinline__ void node4_hits(const float4 *nodes, int node, float ix, float iy,
                                           float iz, float oix, float oiy, float oiz, float tmax,
                                           float d[4], int c[4]) {
    const float4 *nd = nodes + 8 * node;
    float x[8], y[8], z[8], w[8];
    ldg256(nd + 0, x);
    ldg256(nd + 2, y);
    ldg256(nd + 4, z);
    ldg256(nd + 6, w);
    const float lxa[4] = {x[0], x[1], x[2], x[3]}, hxa[4] = {x[4], x[5], x[6], x[7]};
    const float lya[4] = {y[0], y[1], y[2], y[3]}, hya[4] = {y[4], y[5], y[6], y[7]};
    const float lza[4] = {z[0], z[1], z[2], z[3]}, hza[4] = {z[4], z[5], z[6], z[7]};
    const int ca[4] = {__float_as_int(w[0]), __float_as_int(w[1]), __float_as_int(w[2]),
                       __float_as_int(w[3])};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float ax = fmaf(lxa[k], ix, -oix), bx = fmaf(hxa[k], ix, -oix);
        const float ay = fmaf(lya[k], iy, -oiy), by = fmaf(hya[k], iy, -oiy);
        const float az = fmaf(lza[k], iz, -oiz), bz = fmaf(hza[k], iz, -oiz);
        const float tn = fmaxf(fmaxf(fminf(ax, bx), fminf(ay, by)), fmaxf(fminf(az, bz), 0.0f));
        const float tf = fminf(fminf(fmaxf(ax, bx), fmaxf(ay, by)), fminf(fmaxf(az, bz), tmax));
        const bool hit = tn <= tf && ca[k] != EMPTY_CHILD;
        d[k] = hit ? tn : INFINITY;
        c[k] = ca[k];
    }
    cswap(d[0], c[0], d[1], c[1]);
    cswap(d[2], c[2], d[3], c[3]);
    cswap(d[0], c[0], d[2], c[2]);
    cswap(d[1], c[1], d[3], c[3]);
    cswap(d[1], c[1], d[2], c[2]);
}

// Nearest hit (ANY_HIT = false) or occlusion test (ANY_HIT = true) with a
// per-thread stack of (node, entry distance) pairs: popped entries farther
// than the current hit are skipped.  Leaves carry their triangle count
// (~ref = first << 3 | count), so all of a leaf's triangle records are
// fetched before the first test.  Returns the hit record index (or -1).
// BVH4 with fp16 child boxes (64-byte nodes, "width" 5): boxes were rounded
// outward on the host, so the half box contains the float box.
__device__ __forceinline__ void node4h_hits(const float4 *nodes, int node, float ix, float iy,
                                            float iz, float oix, float oiy, float oiz, float tmax,
                                            float d[4], int c[4]) {
    const uint4 *nd = reinterpret_cast<const uint4 *>(nodes) + 4 * node;
    const uint4 qx = __ldg(nd + 0), qy = __ldg(nd + 1), qz = __ldg(nd + 2);
    const int4 ch = __ldg(reinterpret_cast<const int4 *>(nd + 3));
    float lx[4], hx[4], ly[4], hy[4], lz[4], hz[4];
    auto unpack = [](uint32_t w, float &a, float &b) {
        const float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&w));
        a = f.x;
        b = f.y;
    };
    unpack(qx.x, lx[0], lx[1]); unpack(qx.y, lx[2], lx[3]);
    unpack(qx.z, hx[0], hx[1]); unpack(qx.w, hx[2], hx[3]);
    unpack(qy.x, ly[0], ly[1]); unpack(qy.y, ly[2], ly[3]);
    unpack(qy.z, hy[0], hy[1]); unpack(qy.w, hy[2], hy[3]);
    unpack(qz.x, lz[0], lz[1]); unpack(qz.y, lz[2], lz[3]);
    unpack(qz.z, hz[0], hz[1]); unpack(qz.w, hz[2], hz[3]);
    const int ca[4] = {ch.x, ch.y, ch.z, ch.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float ax = fmaf(lx[k], ix, -oix), bx = fmaf(hx[k], ix, -oix);
        const float ay = fmaf(ly[k], iy, -oiy), by = fmaf(hy[k], iy, -oiy);
        const float az = fmaf(lz[k], iz, -oiz), bz = fmaf(hz[k], iz, -oiz);
        const float tn = fmaxf(fmaxf(fminf(ax, bx), fminf(ay, by)), fmaxf(fminf(az, bz), 0.0f));
        const float tf = fminf(fminf(fmaxf(ax, bx), fmaxf(ay, by)), fminf(fmaxf(az, bz), tmax));
        const bool hit = tn <= tf && ca[k] != EMPTY_CHILD;
        d[k] = hit ? tn : INFINITY;
        c[k] = ca[k];
    }
    cswap(d[0], c[0], d[1], c[1]);
    cswap(d[2], c[2], d[3], c[3]);
    cswap(d[0], c[0], d[2], c[2]);
    cswap(d[1], c[1], d[3], c[3]);
    cswap(d[1], c[1], d[2], c[2]);
}

// traversal statistics of the STATS variant (tuning only): inner-node visits,
// BVH4 node test for a ray octant known at compile time (OCT bit a set = the
// direction's axis-a component is negative): the entry / exit planes of each
// slab are picked by the octant instead of a min / max pair per axis, so a
// child costs 6 FFMA + 4 min/max instead of 6 FFMA + 10 min/max.  For l <= h
// and i > 0, fma(l, i, -oi) <= fma(h, i, -oi) (fma is monotone in l), so the
// picked planes are exactly min / max of the generic test: identical results.
template <int OCT>
__device__ __forceinline__ void node4o_hits(const float4 *nodes, int node, float ix, float iy,
                                            float iz, float oix, float oiy, float oiz,
                                            float tmax, float d[4], int c[4]) {
    constexpr bool NX = OCT & 1, NY = OCT & 2, NZ = OCT & 4;
    const float4 *nd = nodes + 8 * node;
    float x[8], y[8], z[8], w[8];
    ldg256(nd + 0, x);
    ldg256(nd + 2, y);
    ldg256(nd + 4, z);
    ldg256(nd + 6, w);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float nx = fmaf(x[NX ? 4 + k : k], ix, -oix), fx = fmaf(x[NX ? k : 4 + k], ix, -oix);
        const float ny = fmaf(y[NY ? 4 + k : k], iy, -oiy), fy = fmaf(y[NY ? k : 4 + k], iy, -oiy);
        const float nz = fmaf(z[NZ ? 4 + k : k], iz, -oiz), fz = fmaf(z[NZ ? k : 4 + k], iz, -oiz);
        const float tn = fmaxf(fmaxf(nx, ny), fmaxf(nz, 0.0f));
        const float tf = fminf(fminf(fx, fy), fminf(fz, tmax));
        // unused slots hold lo = +inf, hi = -inf: tn = +inf, never a hit
        d[k] = tn <= tf ? tn : INFINITY;
        c[k] = __float_as_int(w[k]);
    }
    cswap(d[0], c[0], d[1], c[1]);
    cswap(d[2], c[2], d[3], c[3]);
    cswap(d[0], c[0], d[2], c[2]);
    cswap(d[1], c[1], d[3], c[3]);
    cswap(d[1], c[1], d[2], c[2]);
}

// WIDTH 6: BVH4, octant-specialised node test chosen per node (warp-uniform
// when the warp's rays share a direction); WIDTH 7: the whole traversal
// instantiated per octant (WIDTH 8 + octant) and chosen once per ray
// leaf visits, triangle tests, rays
static __device__ unsigned long long g_trav_stats[4];

template <bool ANY_HIT, int LEAFV = 0, int WIDTH = 2, int STATS = 0>
__device__ int traverse(const float4 *__restrict__ nodes, const float4 *__restrict__ tris,
                        const Ray &r, float tmax, float &t_best) {
    unsigned long long st_nodes = 0, st_leaves = 0, st_tris = 0;
    // reciprocal direction; tiny components replaced so the slabs stay finite
    const float sx = fabsf(r.dx) < 1e-12f ? copysignf(1e-12f, r.dx) : r.dx;
    const float sy = fabsf(r.dy) < 1e-12f ? copysignf(1e-12f, r.dy) : r.dy;
    const float sz = fabsf(r.dz) < 1e-12f ? copysignf(1e-12f, r.dz) : r.dz;
    const int oct = (sx < 0.0f ? 1 : 0) | (sy < 0.0f ? 2 : 0) | (sz < 0.0f ? 4 : 0);
    if constexpr (WIDTH == 7) {
        switch (oct) {
            case 0: return traverse<ANY_HIT, LEAFV, 8, STATS>(nodes, tris, r, tmax, t_best);
            case 1: return traverse<ANY_HIT, LEAFV, 9, STATS>(nodes, tris, r, tmax, t_best);
            case 2: return traverse<ANY_HIT, LEAFV, 10, STATS>(nodes, tris, r, tmax, t_best);
            case 3: return traverse<ANY_HIT, LEAFV, 11, STATS>(nodes, tris, r, tmax, t_best);
            case 4: return traverse<ANY_HIT, LEAFV, 12, STATS>(nodes, tris, r, tmax, t_best);
            case 5: return traverse<ANY_HIT, LEAFV, 13, STATS>(nodes, tris, r, tmax, t_best);
            case 6: return traverse<ANY_HIT, LEAFV, 14, STATS>(nodes, tris, r, tmax, t_best);
            default: return traverse<ANY_HIT, LEAFV, 15, STATS>(nodes, tris, r, tmax, t_best);
        }
    }
    const float ix = 1.0f / sx, iy = 1.0f / sy, iz = 1.0f / sz;
    const float oix = r.ox * ix, oiy = r.oy * iy, oiz = r.oz * iz;
    int2 stack[STACK];
    int sp = 0;
    int node = 0;
    int hit_slot = -1;
    t_best = tmax;
    while (true) {
        if (STATS) {
            if (node >= 0) ++st_nodes;
            else {
                ++st_leaves;
                st_tris += (~node) & 7;
            }
        }
        if (node >= 0 && (WIDTH == 4 || WIDTH == 5 || WIDTH == 6 || WIDTH >= 8)) {
            float d[4];
            int c[4];
            if constexpr (WIDTH == 5) {
                node4h_hits(nodes, node, ix, iy, iz, oix, oiy, oiz, t_best, d, c);
            } else if constexpr (WIDTH >= 8) {
                node4o_hits<(WIDTH - 8) & 7>(nodes, node, ix, iy, iz, oix, oiy, oiz, t_best, d, c);
            } else if constexpr (WIDTH == 6) {
#define PS_OCT_CASE(o) \
    case o: node4o_hits<o>(nodes, node, ix, iy, iz, oix, oiy, oiz, t_best, d, c); break;
                switch (oct) {
                    PS_OCT_CASE(0) PS_OCT_CASE(1) PS_OCT_CASE(2) PS_OCT_CASE(3)
                    PS_OCT_CASE(4) PS_OCT_CASE(5) PS_OCT_CASE(6)
                    default: node4o_hits<7>(nodes, node, ix, iy, iz, oix, oiy, oiz, t_best, d, c);
                }
#undef PS_OCT_CASE
            } else {
                node4_hits(nodes, node, ix, iy, iz, oix, oiy, oiz, t_best, d, c);
            }
            if (d[0] != INFINITY) {
                if (d[3] != INFINITY) stack[sp++] = make_int2(c[3], __float_as_int(d[3]));
                if (d[2] != INFINITY) stack[sp++] = make_int2(c[2], __float_as_int(d[2]));
                if (d[1] != INFINITY) stack[sp++] = make_int2(c[1], __float_as_int(d[1]));
                node = c[0];
                continue;
            }
        } else if (node >= 0) {
            bool h0, h1;
            float t0, t1;
            int c0, c1;
            node_hits(nodes, node, ix, iy, iz, oix, oiy, oiz, t_best, h0, h1, t0, t1, c0, c1);
            if (h0 && h1) {
                const bool swap = t1 < t0;
                node = swap ? c1 : c0;
                stack[sp++] = make_int2(swap ? c0 : c1, __float_as_int(swap ? t0 : t1));
                continue;
            }
            if (h0 || h1) {
                node = h0 ? c0 : c1;
                continue;
            }
        } else {
            const int ref = ~node;
            const int first = ref >> 3, cnt = ref & 7;
            if (LEAFV == 2) {  // fetch up to 4 triangles before testing
                float4 v0[4], e1[4], e2[4];
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (k < cnt) {
                        v0[k] = __ldg(tris + 3 * (first + k));
                        e1[k] = __ldg(tris + 3 * (first + k) + 1);
                        e2[k] = __ldg(tris + 3 * (first + k) + 2);
                    }
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (k < cnt) {
                        const float t = tri_hit(r, v0[k], e1[k], e2[k]);
                        if (t < t_best) {
                            t_best = t;
                            hit_slot = first + k;
                            if (ANY_HIT) return hit_slot;
                        }
                    }
            } else if (LEAFV == 1) {  // two triangles in flight
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
                    float t = tri_hit(r, a0, a1, a2);
                    if (t < t_best) {
                        t_best = t;
                        hit_slot = first + k;
                        if (ANY_HIT) return hit_slot;
                    }
                    if (two) {
                        t = tri_hit(r, b0, b1, b2);
                        if (t < t_best) {
                            t_best = t;
                            hit_slot = first + k + 1;
                            if (ANY_HIT) return hit_slot;
                        }
                    }
                }
            } else {
                for (int k = 0; k < cnt; ++k) {
                    const float t = tri_hit(r, __ldg(tris + 3 * (first + k)),
                                            __ldg(tris + 3 * (first + k) + 1),
                                            __ldg(tris + 3 * (first + k) + 2));
                    if (t < t_best) {
                        t_best = t;
                        hit_slot = first + k;
                        if (ANY_HIT) return hit_slot;
                    }
                }
            }
            if (LEAFV == 2)
                for (int k = 4; k < cnt; ++k) {  // leaves larger than 4 (leaf_size > 4)
                    const float t = tri_hit(r, __ldg(tris + 3 * (first + k)),
                                            __ldg(tris + 3 * (first + k) + 1),
                                            __ldg(tris + 3 * (first + k) + 2));
                    if (t < t_best) {
                        t_best = t;
                        hit_slot = first + k;
                        if (ANY_HIT) return hit_slot;
                    }
                }
        }
        // pop the nearest pending subtree that can still hold a closer hit
        bool found = false;
        while (sp > 0) {
            const int2 e = stack[--sp];
            if (__int_as_float(e.y) <= t_best) {
                node = e.x;
                found = true;
                break;
            }
        }
        if (!found) break;
    }
    if (STATS) {
        atomicAdd(&g_trav_stats[0], st_nodes);
        atomicAdd(&g_trav_stats[1], st_leaves);
        atomicAdd(&g_trav_stats[2], st_tris);
        atomicAdd(&g_trav_stats[3], 1ull);
    }
    return hit_slot;
}


}  // namespace trav
}  // namespace ps
