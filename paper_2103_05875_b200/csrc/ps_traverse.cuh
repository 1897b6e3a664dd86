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
// PS_TRACE_PREFETCH (tuning): prefetch a parked leaf's triangles into L1
#ifndef PS_TRACE_PREFETCH
#define PS_TRACE_PREFETCH 0
#endif
// PS_TRACE_L1_HINT (tuning): 1 = node loads L1::evict_last and triangle loads
// L1::evict_first, 2 = node loads evict_last only
#ifndef PS_TRACE_L1_HINT
#define PS_TRACE_L1_HINT 0
#endif
__device__ __forceinline__ void ldg256(const void *p, float (&v)[8]) {
#if PS_TRACE_L1_HINT >= 1
    asm("ld.global.nc.L1::evict_last.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
#else
    asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
#endif
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
          "=f"(v[7])
        : "l"(p));
}

// triangle record load (see PS_TRACE_L1_HINT)
__device__ __forceinline__ float4 ldg_tri(const float4 *p) {
#if PS_TRACE_L1_HINT == 1
    float4 v;
    asm("ld.global.nc.L1::evict_first.v4.f32 {%0, %1, %2, %3}, [%4];"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
        : "l"(p));
    return v;
#else
    return __ldg(p);
#endif
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

// fp16-box BVH4 (64-byte nodes) with the octant-specialised test: two 256-bit
// loads per node instead of four (the trace is bound by L1 wavefronts of
// divergent node fetches, one per distinct line per load instruction)
template <int OCT>
__device__ __forceinline__ void node4ho_hits(const float4 *nodes, int node, float ix, float iy,
                                             float iz, float oix, float oiy, float oiz,
                                             float tmax, float d[4], int c[4]) {
    constexpr bool NX = OCT & 1, NY = OCT & 2, NZ = OCT & 4;
    const float4 *nd = nodes + 4 * node;
    float a[8], b[8];
    ldg256(nd + 0, a);  // lo_x[4] hi_x[4] | lo_y[4] hi_y[4] (halves)
    ldg256(nd + 2, b);  // lo_z[4] hi_z[4] | child[4]
    auto h2 = [](float w) { return __half22float2(*reinterpret_cast<const __half2 *>(&w)); };
    // word k / 2 of a plane set holds children (2j, 2j+1)
    const float2 lx0 = h2(a[0]), lx1 = h2(a[1]), hx0 = h2(a[2]), hx1 = h2(a[3]);
    const float2 ly0 = h2(a[4]), ly1 = h2(a[5]), hy0 = h2(a[6]), hy1 = h2(a[7]);
    const float2 lz0 = h2(b[0]), lz1 = h2(b[1]), hz0 = h2(b[2]), hz1 = h2(b[3]);
    const float lxs[4] = {lx0.x, lx0.y, lx1.x, lx1.y}, hxs[4] = {hx0.x, hx0.y, hx1.x, hx1.y};
    const float lys[4] = {ly0.x, ly0.y, ly1.x, ly1.y}, hys[4] = {hy0.x, hy0.y, hy1.x, hy1.y};
    const float lzs[4] = {lz0.x, lz0.y, lz1.x, lz1.y}, hzs[4] = {hz0.x, hz0.y, hz1.x, hz1.y};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float nx = fmaf(NX ? hxs[k] : lxs[k], ix, -oix), fx = fmaf(NX ? lxs[k] : hxs[k], ix, -oix);
        const float ny = fmaf(NY ? hys[k] : lys[k], iy, -oiy), fy = fmaf(NY ? lys[k] : hys[k], iy, -oiy);
        const float nz = fmaf(NZ ? hzs[k] : lzs[k], iz, -oiz), fz = fmaf(NZ ? lzs[k] : hzs[k], iz, -oiz);
        const float tn = fmaxf(fmaxf(nx, ny), fmaxf(nz, 0.0f));
        const float tf = fminf(fminf(fx, fy), fminf(fz, tmax));
        d[k] = tn <= tf ? tn : INFINITY;
        c[k] = __float_as_int(b[4 + k]);
    }
    cswap(d[0], c[0], d[1], c[1]);
    cswap(d[2], c[2], d[3], c[3]);
    cswap(d[0], c[0], d[2], c[2]);
    cswap(d[1], c[1], d[3], c[3]);
    cswap(d[1], c[1], d[2], c[2]);
}

// BVH4 with origin-relative fp16 boxes and compact child references (WIDTH 17;
// layout: ps_bvh.cpp emit_bvh4r): two 256-bit loads per node, planes decoded
// as fma(rel, idir, fma(origin, idir, -o * idir)), children referenced as
// child_base + rank (inner) or a leaf's (offset, count) from tri_base.
template <int OCT>
__device__ __forceinline__ void node4r_hits(const float4 *nodes, int node, float ix, float iy,
                                            float iz, float oix, float oiy, float oiz,
                                            float tmax, float d[4], int c[4]) {
    constexpr bool NX = OCT & 1, NY = OCT & 2, NZ = OCT & 4;
    const float4 *nd = nodes + 4 * node;
    float a[8], b[8];
    ldg256(nd + 0, a);  // lo_x[4] hi_x[4] | lo_y[4] hi_y[4]
    ldg256(nd + 2, b);  // lo_z[4] hi_z[4] | origin xy, origin z | meta, child_base, tri_base
    auto h2 = [](float w) { return __half22float2(*reinterpret_cast<const __half2 *>(&w)); };
    const float2 oxy = h2(b[4]);
    const uint32_t w13 = __float_as_uint(b[5]);
    const float oz = __half2float(__ushort_as_half(uint16_t(w13 & 0xFFFFu)));
    const float Cx = fmaf(oxy.x, ix, -oix), Cy = fmaf(oxy.y, iy, -oiy), Cz = fmaf(oz, iz, -oiz);
    const float2 lx0 = h2(a[0]), lx1 = h2(a[1]), hx0 = h2(a[2]), hx1 = h2(a[3]);
    const float2 ly0 = h2(a[4]), ly1 = h2(a[5]), hy0 = h2(a[6]), hy1 = h2(a[7]);
    const float2 lz0 = h2(b[0]), lz1 = h2(b[1]), hz0 = h2(b[2]), hz1 = h2(b[3]);
    const float lxs[4] = {lx0.x, lx0.y, lx1.x, lx1.y}, hxs[4] = {hx0.x, hx0.y, hx1.x, hx1.y};
    const float lys[4] = {ly0.x, ly0.y, ly1.x, ly1.y}, hys[4] = {hy0.x, hy0.y, hy1.x, hy1.y};
    const float lzs[4] = {lz0.x, lz0.y, lz1.x, lz1.y}, hzs[4] = {hz0.x, hz0.y, hz1.x, hz1.y};
    const uint32_t meta = w13 >> 16;
    const int child_base = __float_as_int(b[6]), tri_base = __float_as_int(b[7]);
    int rank = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float nx = fmaf(NX ? hxs[k] : lxs[k], ix, Cx), fx = fmaf(NX ? lxs[k] : hxs[k], ix, Cx);
        const float ny = fmaf(NY ? hys[k] : lys[k], iy, Cy), fy = fmaf(NY ? lys[k] : hys[k], iy, Cy);
        const float nz = fmaf(NZ ? hzs[k] : lzs[k], iz, Cz), fz = fmaf(NZ ? lzs[k] : hzs[k], iz, Cz);
        const float tn = fmaxf(fmaxf(nx, ny), fmaxf(nz, 0.0f));
        const float tf = fminf(fminf(fx, fy), fminf(fz, tmax));
        d[k] = tn <= tf ? tn : INFINITY;
        const uint32_t nib = (meta >> (4 * k)) & 15u;
        const uint32_t v = nib - 1u;  // leaf: offset << 1 | (count - 1)
        const int leaf = ~int(((uint32_t(tri_base) + (v >> 1)) << 3) | ((v & 1u) + 1u));
        c[k] = nib == 15u ? child_base + rank : leaf;
        rank += nib == 15u ? 1 : 0;
    }
    cswap(d[0], c[0], d[1], c[1]);
    cswap(d[2], c[2], d[3], c[3]);
    cswap(d[0], c[0], d[2], c[2]);
    cswap(d[1], c[1], d[3], c[3]);
    cswap(d[1], c[1], d[2], c[2]);
}

// fp16-box BVH4 (64-byte nodes), entry / exit planes picked per axis by the
// ray's direction signs with word selects on the packed halves (12 SEL per
// node) instead of a per-node switch over octant-specialised tests (WIDTH 18)
__device__ __forceinline__ void node4hs_hits(const float4 *nodes, int node, float ix, float iy,
                                             float iz, float oix, float oiy, float oiz,
                                             float tmax, bool negx, bool negy, bool negz,
                                             float d[4], int c[4]) {
    const float4 *nd = nodes + 4 * node;
    float a[8], b[8];
    ldg256(nd + 0, a);  // lo_x[4] hi_x[4] | lo_y[4] hi_y[4] (halves)
    ldg256(nd + 2, b);  // lo_z[4] hi_z[4] | child[4]
    auto h2 = [](float w) { return __half22float2(*reinterpret_cast<const __half2 *>(&w)); };
    const float2 nx0 = h2(negx ? a[2] : a[0]), nx1 = h2(negx ? a[3] : a[1]);
    const float2 fx0 = h2(negx ? a[0] : a[2]), fx1 = h2(negx ? a[1] : a[3]);
    const float2 ny0 = h2(negy ? a[6] : a[4]), ny1 = h2(negy ? a[7] : a[5]);
    const float2 fy0 = h2(negy ? a[4] : a[6]), fy1 = h2(negy ? a[5] : a[7]);
    const float2 nz0 = h2(negz ? b[2] : b[0]), nz1 = h2(negz ? b[3] : b[1]);
    const float2 fz0 = h2(negz ? b[0] : b[2]), fz1 = h2(negz ? b[1] : b[3]);
    const float nxs[4] = {nx0.x, nx0.y, nx1.x, nx1.y}, fxs[4] = {fx0.x, fx0.y, fx1.x, fx1.y};
    const float nys[4] = {ny0.x, ny0.y, ny1.x, ny1.y}, fys[4] = {fy0.x, fy0.y, fy1.x, fy1.y};
    const float nzs[4] = {nz0.x, nz0.y, nz1.x, nz1.y}, fzs[4] = {fz0.x, fz0.y, fz1.x, fz1.y};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float nx = fmaf(nxs[k], ix, -oix), fx = fmaf(fxs[k], ix, -oix);
        const float ny = fmaf(nys[k], iy, -oiy), fy = fmaf(fys[k], iy, -oiy);
        const float nz = fmaf(nzs[k], iz, -oiz), fz = fmaf(fzs[k], iz, -oiz);
        const float tn = fmaxf(fmaxf(nx, ny), fmaxf(nz, 0.0f));
        const float tf = fminf(fminf(fx, fy), fminf(fz, tmax));
        d[k] = tn <= tf ? tn : INFINITY;
        c[k] = __float_as_int(b[4 + k]);
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

// ---- BVH8 with 8-bit quantised child boxes (WIDTH 16; node layout: ps_bvh.cpp
// emit_bvh8).  Per node three 256-bit loads cover eight children; hit inner
// children are visited in ascending (slot ^ ray octant), an approximate
// front-to-back order fixed at build time, so there is no sort and at most one
// stack push per visited node: the stack holds node groups (first child index,
// remaining hit slots in order space << 24 | the inner-slot mask).  A popped
// child is culled by its own children's tests against the current t_best.
constexpr int STACK8 = 32;

__device__ __forceinline__ float q2f(uint32_t word, int byte) {
    // 2^23 + q as a float: one byte permute, the 2^23 is folded into the offset
    return __uint_as_float(__byte_perm(word, 0x4B000000u, 0x7440u + byte));
}

__device__ __forceinline__ uint32_t oct_permute8(uint32_t m, uint32_t oct) {
    // bit s -> bit s ^ oct
    if (oct & 1) m = ((m & 0x55u) << 1) | ((m >> 1) & 0x55u);
    if (oct & 2) m = ((m & 0x33u) << 2) | ((m >> 2) & 0x33u);
    if (oct & 4) m = ((m & 0x0Fu) << 4) | ((m >> 4) & 0x0Fu);
    return m;
}

template <bool ANY_HIT, int STATS = 0>
__device__ int traverse8(const float4 *__restrict__ nodes, const float4 *__restrict__ tris,
                         const Ray &r, float tmax, float &t_best) {
    unsigned long long st_nodes = 0, st_tris = 0;
    const float sx = fabsf(r.dx) < 1e-12f ? copysignf(1e-12f, r.dx) : r.dx;
    const float sy = fabsf(r.dy) < 1e-12f ? copysignf(1e-12f, r.dy) : r.dy;
    const float sz = fabsf(r.dz) < 1e-12f ? copysignf(1e-12f, r.dz) : r.dz;
    const bool negx = sx < 0.0f, negy = sy < 0.0f, negz = sz < 0.0f;
    const uint32_t oct = (negx ? 1u : 0u) | (negy ? 2u : 0u) | (negz ? 4u : 0u);
    const float ix = 1.0f / sx, iy = 1.0f / sy, iz = 1.0f / sz;
    const float oix = r.ox * ix, oiy = r.oy * iy, oiz = r.oz * iz;
    uint2 stack[STACK8];
    int sp = 0;
    uint32_t g_base = 0, g_hits = 0;  // current group: order-space hits << 24 | imask
    int node = 0;
    int hit_slot = -1;
    t_best = tmax;
    while (true) {
        if (STATS) ++st_nodes;
        // ---- visit `node`: test its eight children ------------------------------------------
        const float4 *nd = nodes + 6 * node;
        float a[8], b[8], c[8];
        ldg256(nd + 0, a);
        ldg256(nd + 2, b);
        ldg256(nd + 4, c);
        const uint32_t ew = __float_as_uint(a[3]);
        const uint32_t child_base = __float_as_uint(a[4]), tri_base = __float_as_uint(a[5]);
        const uint32_t meta0 = __float_as_uint(a[6]), meta1 = __float_as_uint(a[7]);
        const uint32_t imask = ew >> 24;
        // per axis: A = scale * idir, C = (p - o) * idir - 2^23 * A
        const float sxa = __uint_as_float((ew & 0xFFu) << 23);
        const float sya = __uint_as_float(((ew >> 8) & 0xFFu) << 23);
        const float sza = __uint_as_float(((ew >> 16) & 0xFFu) << 23);
        const float Ax = sxa * ix, Ay = sya * iy, Az = sza * iz;
        const float Cx = fmaf(-8388608.0f, Ax, fmaf(a[0], ix, -oix));
        const float Cy = fmaf(-8388608.0f, Ay, fmaf(a[1], iy, -oiy));
        const float Cz = fmaf(-8388608.0f, Az, fmaf(a[2], iz, -oiz));
        // entry / exit planes by direction sign (4 children per word)
        const uint32_t lx0 = __float_as_uint(b[0]), lx1 = __float_as_uint(b[1]);
        const uint32_t ly0 = __float_as_uint(b[2]), ly1 = __float_as_uint(b[3]);
        const uint32_t lz0 = __float_as_uint(b[4]), lz1 = __float_as_uint(b[5]);
        const uint32_t hx0 = __float_as_uint(b[6]), hx1 = __float_as_uint(b[7]);
        const uint32_t hy0 = __float_as_uint(c[0]), hy1 = __float_as_uint(c[1]);
        const uint32_t hz0 = __float_as_uint(c[2]), hz1 = __float_as_uint(c[3]);
        const uint32_t nx0 = negx ? hx0 : lx0, nx1 = negx ? hx1 : lx1;
        const uint32_t fx0 = negx ? lx0 : hx0, fx1 = negx ? lx1 : hx1;
        const uint32_t ny0 = negy ? hy0 : ly0, ny1 = negy ? hy1 : ly1;
        const uint32_t fy0 = negy ? ly0 : hy0, fy1 = negy ? ly1 : hy1;
        const uint32_t nz0 = negz ? hz0 : lz0, nz1 = negz ? hz1 : lz1;
        const uint32_t fz0 = negz ? lz0 : hz0, fz1 = negz ? lz1 : hz1;
        uint32_t hit8 = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int w = k & 3;
            const float tnx = fmaf(q2f(k < 4 ? nx0 : nx1, w), Ax, Cx);
            const float tny = fmaf(q2f(k < 4 ? ny0 : ny1, w), Ay, Cy);
            const float tnz = fmaf(q2f(k < 4 ? nz0 : nz1, w), Az, Cz);
            const float tfx = fmaf(q2f(k < 4 ? fx0 : fx1, w), Ax, Cx);
            const float tfy = fmaf(q2f(k < 4 ? fy0 : fy1, w), Ay, Cy);
            const float tfz = fmaf(q2f(k < 4 ? fz0 : fz1, w), Az, Cz);
            const float tn = fmaxf(fmaxf(tnx, tny), fmaxf(tnz, 0.0f));
            const float tf = fminf(fminf(tfx, tfy), fminf(tfz, t_best));
            hit8 |= tn <= tf ? (1u << k) : 0u;
        }
        // ---- leaf children: their triangles now -------------------------------------------
        uint32_t leaves = hit8 & ~imask;
        while (leaves) {
            const int sl = __ffs(leaves) - 1;
            leaves &= leaves - 1;
            const uint32_t meta = ((sl < 4 ? meta0 : meta1) >> (8 * (sl & 3))) & 0xFFu;
            const int first = int(tri_base + (meta & 31u)), cnt = int(meta >> 5);
            for (int k = 0; k < cnt; ++k) {
                if (STATS) ++st_tris;
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
        // ---- inner children: a new group --------------------------------------------------
        const uint32_t inner = oct_permute8(hit8 & imask, oct);
        if (inner) {
            if (g_hits & 0xFF000000u) stack[sp++] = make_uint2(g_base, g_hits);
            g_base = child_base;
            g_hits = (inner << 24) | imask;
        }
        // ---- next child: this group's, else a popped one ---------------------------------
        while (!(g_hits & 0xFF000000u)) {
            if (sp == 0) {
                if (STATS) {
                    atomicAdd(&g_trav_stats[0], st_nodes);
                    atomicAdd(&g_trav_stats[2], st_tris);
                    atomicAdd(&g_trav_stats[3], 1ull);
                }
                return hit_slot;
            }
            const uint2 e = stack[--sp];
            g_base = e.x;
            g_hits = e.y;
        }
        const uint32_t bit = __ffs(g_hits >> 24) - 1;
        g_hits &= ~(1u << (bit + 24));
        const uint32_t slot = bit ^ oct;
        node = int(g_base + __popc(g_hits & ((1u << slot) - 1u) & 0xFFu));
    }
}

// fp16-box BVH4 node test (node4ho_hits) dispatched on the ray octant
__device__ __forceinline__ void node4ho_switch(const float4 *nodes, int node, int oct, float ix,
                                               float iy, float iz, float oix, float oiy, float oiz,
                                               float tmax, float d[4], int c[4]) {
#define PS_OCTS_CASE(o) \
    case o: node4ho_hits<o>(nodes, node, ix, iy, iz, oix, oiy, oiz, tmax, d, c); break;
    switch (oct) {
        PS_OCTS_CASE(0) PS_OCTS_CASE(1) PS_OCTS_CASE(2) PS_OCTS_CASE(3)
        PS_OCTS_CASE(4) PS_OCTS_CASE(5) PS_OCTS_CASE(6)
        default: node4ho_hits<7>(nodes, node, ix, iy, iz, oix, oiy, oiz, tmax, d, c);
    }
#undef PS_OCTS_CASE
}

// ---- fp16 slab arithmetic (WIDTH 23) ----------------------------------------------
// The node test of node4ho_hits in packed half2 arithmetic: one HFMA2 computes
// a plane's t for two children at once straight from the node's fp16 words
// (no fp16 -> fp32 conversions), HMNMX2 reduces the slabs.  The result is
// conservative -- a child the exact slab test accepts is never rejected --
// so the set of tested triangles only grows and the nearest hit (an fp32
// triangle test) is unchanged:
//   t' = rn(b * I + C) with, per axis, near-plane  I_n = rd(|1/d| (1 - s)),
//   C_n = rd(-o I_n) and far-plane I_f = ru(|1/d| (1 + s)), C_f = ru(-o I_f)
//   (magnitudes; sign of d applied).  For t >= 0 the slack s (PS_HALF_SLACK)
//   covers the final rounding (<= 2^-11 relative), so near t' <= t and far
//   t' >= t.
// A ray with an axis whose constants would leave the fp16 range (|o / d|
// >~ 6e4) takes the fp32 test (traverse_spec); dropping the axis (I = 0,
// C = -inf / +inf) would be conservative too, but such rays then visit most
// of the BVH.
struct HalfSlabs {
    __half2 i[3];  // (I_near, I_far) per axis
    __half2 c[3];  // (C_near, C_far)
};

// relative slack s of the reciprocals: the final rn rounding of an HFMA2 is
// within 2^-11 of its result, so (1 - s)(1 + 2^-11) <= 1 <= (1 + s)(1 - 2^-11)
// needs s >= 2^-11 / (1 - 2^-11); 2^-11 (1 + 2^-8) also covers the fp32
// rounding of 1/d and of |1/d| (1 -+ s) (2^-24 each)
#ifndef PS_HALF_SLACK
#define PS_HALF_SLACK (1.00390625f / 2048.0f)
#endif
__device__ __forceinline__ bool half_axis(float o, float s, __half2 &I, __half2 &C) {
    const float mag = fabsf(1.0f / s);
    const float mn = mag * (1.0f - PS_HALF_SLACK), mf = mag * (1.0f + PS_HALF_SLACK);
    if (mf < 60000.0f && mf * fabsf(o) < 60000.0f) {
        const float in_ = copysignf(__half2float(__float2half_rd(mn)), s);
        const float if_ = copysignf(__half2float(__float2half_ru(mf)), s);
        I = __halves2half2(__float2half_rn(in_), __float2half_rn(if_));  // exact
#ifdef PS_HALF_C_RN  // tuning only: not conservative
        C = __halves2half2(__float2half_rn(-o * in_), __float2half_rn(-o * if_));
#else
        C = __halves2half2(__float2half_rd(__fmul_rd(-o, in_)), __float2half_ru(__fmul_ru(-o, if_)));
#endif
        return true;
    }
    I = __floats2half2_rn(0.0f, 0.0f);
    C = __floats2half2_rn(-INFINITY, INFINITY);
    return false;
}

template <int OCT>
__device__ __forceinline__ void node4hh_hits(const float4 *nodes, int node, const HalfSlabs &h,
                                             __half tbh, float d[4], int c[4]) {
    constexpr bool NX = OCT & 1, NY = OCT & 2, NZ = OCT & 4;
    const float4 *nd = nodes + 4 * node;
    float a[8], b[8];
    ldg256(nd + 0, a);  // lo_x[4] hi_x[4] | lo_y[4] hi_y[4] (halves)
    ldg256(nd + 2, b);  // lo_z[4] hi_z[4] | child[4]
    auto hw = [](float w) { return *reinterpret_cast<const __half2 *>(&w); };
    const __half2 tb2 = __half2half2(tbh);
#pragma unroll
    for (int j = 0; j < 2; ++j) {  // children (2j, 2j+1)
        const __half2 nx = __hfma2(hw(NX ? a[2 + j] : a[j]), __low2half2(h.i[0]), __low2half2(h.c[0]));
        const __half2 fx = __hfma2(hw(NX ? a[j] : a[2 + j]), __high2half2(h.i[0]), __high2half2(h.c[0]));
        const __half2 ny = __hfma2(hw(NY ? a[6 + j] : a[4 + j]), __low2half2(h.i[1]), __low2half2(h.c[1]));
        const __half2 fy = __hfma2(hw(NY ? a[4 + j] : a[6 + j]), __high2half2(h.i[1]), __high2half2(h.c[1]));
        const __half2 nz = __hfma2_relu(hw(NZ ? b[2 + j] : b[j]), __low2half2(h.i[2]), __low2half2(h.c[2]));
        const __half2 fz = __hfma2(hw(NZ ? b[j] : b[2 + j]), __high2half2(h.i[2]), __high2half2(h.c[2]));
        const __half2 tn = __hmax2(__hmax2(nx, ny), nz);
        const __half2 tf = __hmin2(__hmin2(fx, fy), __hmin2(fz, tb2));
        const uint32_t m = __hle2_mask(tn, tf);
        const uint32_t sel = (*reinterpret_cast<const uint32_t *>(&tn) & m) | (0x7C007C00u & ~m);
        const float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&sel));
        d[2 * j] = f.x;
        d[2 * j + 1] = f.y;
        c[2 * j] = __float_as_int(b[4 + 2 * j]);
        c[2 * j + 1] = __float_as_int(b[5 + 2 * j]);
    }
    cswap(d[0], c[0], d[1], c[1]);
    cswap(d[2], c[2], d[3], c[3]);
    cswap(d[0], c[0], d[2], c[2]);
    cswap(d[1], c[1], d[3], c[3]);
    cswap(d[1], c[1], d[2], c[2]);
}

__device__ __forceinline__ void node4hh_switch(const float4 *nodes, int node, int oct,
                                               const HalfSlabs &h, __half tbh, float d[4],
                                               int c[4]) {
#define PS_OCTH_CASE(o) \
    case o: node4hh_hits<o>(nodes, node, h, tbh, d, c); break;
    switch (oct) {
        PS_OCTH_CASE(0) PS_OCTH_CASE(1) PS_OCTH_CASE(2) PS_OCTH_CASE(3)
        PS_OCTH_CASE(4) PS_OCTH_CASE(5) PS_OCTH_CASE(6)
        default: node4hh_hits<7>(nodes, node, h, tbh, d, c);
    }
#undef PS_OCTH_CASE
}

// Speculative while-while traversal (Aila & Laine 2009) over the fp16-box
// BVH4: a lane that reaches a leaf parks it and keeps walking inner nodes
// until every lane still in the loop holds a leaf (warp vote), then the
// warp tests the parked leaves together -- node tests and triangle tests
// run in converged phases instead of interleaving partial warps.  Same
// nearest hit as traverse<..., 3>: a parked leaf is tested later than in the
// plain loop, so pops cull against a t_best that can only be larger (stale),
// never smaller -- no subtree holding the nearest hit is skipped.
constexpr int TRAV_DONE = -1;  // leaf refs are ~(first << 3 | count), count >= 1: <= -2

// SEL: node test with per-axis word selects (node4hs_hits) instead of the
// octant switch; VOTE: leave the node phase when all (0), >= 3/4 (1) or >= 1/2
// (2) of the lanes still walking hold a parked leaf
template <bool ANY_HIT, int SEL = 0, int VOTE = 0, int HALF = 0, int STATS = 0>
__device__ int traverse_spec(const float4 *__restrict__ nodes, const float4 *__restrict__ tris,
                             const Ray &r, float tmax, float &t_best) {
    const float sx = fabsf(r.dx) < 1e-12f ? copysignf(1e-12f, r.dx) : r.dx;
    const float sy = fabsf(r.dy) < 1e-12f ? copysignf(1e-12f, r.dy) : r.dy;
    const float sz = fabsf(r.dz) < 1e-12f ? copysignf(1e-12f, r.dz) : r.dz;
    const int oct = (sx < 0.0f ? 1 : 0) | (sy < 0.0f ? 2 : 0) | (sz < 0.0f ? 4 : 0);
    const float ix = 1.0f / sx, iy = 1.0f / sy, iz = 1.0f / sz;
    const float oix = r.ox * ix, oiy = r.oy * iy, oiz = r.oz * iz;
    HalfSlabs hs;
    // a ray nearly parallel to an axis (|d| < ~2.7e-4 at |o| = 16) cannot use
    // the fp16 constants for that axis: it takes the fp32 node test instead
    // (warp-uniform in the probe trace, whose warps share one direction)
    bool half_ok = false;
    if (HALF) {
        half_ok = half_axis(r.ox, sx, hs.i[0], hs.c[0]);
        half_ok &= half_axis(r.oy, sy, hs.i[1], hs.c[1]);
        half_ok &= half_axis(r.oz, sz, hs.i[2], hs.c[2]);
    }
    __half tbh = __float2half_ru(tmax);
    unsigned long long st_nodes = 0, st_leaves = 0, st_tris = 0;
    int2 stack[STACK];
    int sp = 0;
    int node = 0, leaf = 0;  // leaf: parked leaf ref (0 = none)
    int hit_slot = -1;
    t_best = tmax;
    auto pop = [&]() -> int {
        while (sp > 0) {
            const int2 e = stack[--sp];
            if (__int_as_float(e.y) <= t_best) return e.x;
        }
        return TRAV_DONE;
    };
    while (node != TRAV_DONE || leaf != 0) {
        // ---- inner nodes until every lane holds a leaf (or is done) -------------------
        while (node >= 0) {
            float d[4];
            int c[4];
            if (STATS) ++st_nodes;
            if (HALF && half_ok)
                node4hh_switch(nodes, node, oct, hs, tbh, d, c);
            else if (SEL)
                node4hs_hits(nodes, node, ix, iy, iz, oix, oiy, oiz, t_best, oct & 1, oct & 2,
                             oct & 4, d, c);
            else
                node4ho_switch(nodes, node, oct, ix, iy, iz, oix, oiy, oiz, t_best, d, c);
            if (d[0] != INFINITY) {
                if (d[3] != INFINITY) stack[sp++] = make_int2(c[3], __float_as_int(d[3]));
                if (d[2] != INFINITY) stack[sp++] = make_int2(c[2], __float_as_int(d[2]));
                if (d[1] != INFINITY) stack[sp++] = make_int2(c[1], __float_as_int(d[1]));
                node = c[0];
            } else {
                node = pop();
            }
            if (node < TRAV_DONE && leaf == 0) {  // park the leaf, keep walking
                leaf = node;
#if PS_TRACE_PREFETCH
                {  // its triangle records (48 B each) are fetched into L1 meanwhile
                    const float4 *tp = tris + 3 * ((~leaf) >> 3);
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(tp));
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(tp + 5));
                }
#endif
                node = pop();
            }
            if (VOTE == 0) {
                if (__all_sync(__activemask(), leaf != 0)) break;
            } else {
                const unsigned m = __activemask();
                const int parked = __popc(__ballot_sync(m, leaf != 0));
                if (parked * (VOTE == 1 ? 4 : 2) >= __popc(m) * (VOTE == 1 ? 3 : 1)) break;
            }
        }
        // ---- parked (and directly reached) leaves ----------------------------------------
        while (leaf != 0) {
            const int ref = ~leaf;
            const int first = ref >> 3, cnt = ref & 7;
            if (STATS) {
                ++st_leaves;
                st_tris += cnt;
            }
            for (int k = 0; k < cnt; ++k) {
                const float t = tri_hit(r, ldg_tri(tris + 3 * (first + k)),
                                        ldg_tri(tris + 3 * (first + k) + 1),
                                        ldg_tri(tris + 3 * (first + k) + 2));
                if (t < t_best) {
                    t_best = t;
                    hit_slot = first + k;
                    if (ANY_HIT) return hit_slot;
                }
            }
            if (HALF) tbh = __float2half_ru(t_best);
            leaf = 0;
            if (node < TRAV_DONE) {  // the walk stopped on another leaf
                leaf = node;
                node = pop();
            }
        }
    }
    if (STATS) {
        atomicAdd(&g_trav_stats[0], st_nodes);
        atomicAdd(&g_trav_stats[1], st_leaves);
        atomicAdd(&g_trav_stats[2], st_tris);
        atomicAdd(&g_trav_stats[3], 1ull);
    }
    return hit_slot;
}

template <bool ANY_HIT, int LEAFV = 0, int WIDTH = 2, int STATS = 0>
__device__ int traverse_impl(const float4 *__restrict__ nodes, const float4 *__restrict__ tris,
                             const Ray &r, float tmax, float &t_best) {
    if constexpr (WIDTH == 16) return traverse8<ANY_HIT, STATS>(nodes, tris, r, tmax, t_best);
    if constexpr (WIDTH == 19) return traverse_spec<ANY_HIT>(nodes, tris, r, tmax, t_best);
    if constexpr (WIDTH == 20) return traverse_spec<ANY_HIT, 1>(nodes, tris, r, tmax, t_best);
    if constexpr (WIDTH == 21) return traverse_spec<ANY_HIT, 0, 1>(nodes, tris, r, tmax, t_best);
    if constexpr (WIDTH == 22) return traverse_spec<ANY_HIT, 0, 2>(nodes, tris, r, tmax, t_best);
    if constexpr (WIDTH == 23) return traverse_spec<ANY_HIT, 0, 0, 1>(nodes, tris, r, tmax, t_best);
    if constexpr (WIDTH == 24) return traverse_spec<ANY_HIT, 0, 0, 0, 1>(nodes, tris, r, tmax, t_best);
    if constexpr (WIDTH == 25) return traverse_spec<ANY_HIT, 0, 0, 1, 1>(nodes, tris, r, tmax, t_best);
    unsigned long long st_nodes = 0, st_leaves = 0, st_tris = 0;
    // reciprocal direction; tiny components replaced so the slabs stay finite
    const float sx = fabsf(r.dx) < 1e-12f ? copysignf(1e-12f, r.dx) : r.dx;
    const float sy = fabsf(r.dy) < 1e-12f ? copysignf(1e-12f, r.dy) : r.dy;
    const float sz = fabsf(r.dz) < 1e-12f ? copysignf(1e-12f, r.dz) : r.dz;
    const int oct = (sx < 0.0f ? 1 : 0) | (sy < 0.0f ? 2 : 0) | (sz < 0.0f ? 4 : 0);
    if constexpr (WIDTH == 7) {
        switch (oct) {
            case 0: return traverse_impl<ANY_HIT, LEAFV, 8, STATS>(nodes, tris, r, tmax, t_best);
            case 1: return traverse_impl<ANY_HIT, LEAFV, 9, STATS>(nodes, tris, r, tmax, t_best);
            case 2: return traverse_impl<ANY_HIT, LEAFV, 10, STATS>(nodes, tris, r, tmax, t_best);
            case 3: return traverse_impl<ANY_HIT, LEAFV, 11, STATS>(nodes, tris, r, tmax, t_best);
            case 4: return traverse_impl<ANY_HIT, LEAFV, 12, STATS>(nodes, tris, r, tmax, t_best);
            case 5: return traverse_impl<ANY_HIT, LEAFV, 13, STATS>(nodes, tris, r, tmax, t_best);
            case 6: return traverse_impl<ANY_HIT, LEAFV, 14, STATS>(nodes, tris, r, tmax, t_best);
            default: return traverse_impl<ANY_HIT, LEAFV, 15, STATS>(nodes, tris, r, tmax, t_best);
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
        if (node >= 0 && (WIDTH == 3 || WIDTH == 4 || WIDTH == 5 || WIDTH == 6 || WIDTH >= 8)) {
            float d[4];
            int c[4];
            if constexpr (WIDTH == 5) {
                node4h_hits(nodes, node, ix, iy, iz, oix, oiy, oiz, t_best, d, c);
            } else if constexpr (WIDTH >= 8 && WIDTH < 16) {
                node4o_hits<(WIDTH - 8) & 7>(nodes, node, ix, iy, iz, oix, oiy, oiz, t_best, d, c);
            } else if constexpr (WIDTH == 18) {
                node4hs_hits(nodes, node, ix, iy, iz, oix, oiy, oiz, t_best, oct & 1, oct & 2,
                             oct & 4, d, c);
            } else if constexpr (WIDTH == 17) {
#define PS_OCTR_CASE(o) \
    case o: node4r_hits<o>(nodes, node, ix, iy, iz, oix, oiy, oiz, t_best, d, c); break;
                switch (oct) {
                    PS_OCTR_CASE(0) PS_OCTR_CASE(1) PS_OCTR_CASE(2) PS_OCTR_CASE(3)
                    PS_OCTR_CASE(4) PS_OCTR_CASE(5) PS_OCTR_CASE(6)
                    default: node4r_hits<7>(nodes, node, ix, iy, iz, oix, oiy, oiz, t_best, d, c);
                }
#undef PS_OCTR_CASE
            } else if constexpr (WIDTH == 3) {
#define PS_OCTH_CASE(o) \
    case o: node4ho_hits<o>(nodes, node, ix, iy, iz, oix, oiy, oiz, t_best, d, c); break;
                switch (oct) {
                    PS_OCTH_CASE(0) PS_OCTH_CASE(1) PS_OCTH_CASE(2) PS_OCTH_CASE(3)
                    PS_OCTH_CASE(4) PS_OCTH_CASE(5) PS_OCTH_CASE(6)
                    default: node4ho_hits<7>(nodes, node, ix, iy, iz, oix, oiy, oiz, t_best, d, c);
                }
#undef PS_OCTH_CASE
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


// BVH frame: the node buffer is preceded by a 64-byte header whose first three
// floats are the origin the BVH (boxes and triangle records) was built
// around (scene.py DeviceScene: the scene's centre, so fp16 boxes round
// outward at half the magnitude); rays are translated into that frame for
// the traversal only -- hit distances are unchanged, shading stays in world
// coordinates.
__device__ __forceinline__ Ray to_bvh_frame(const float4 *nodes, const Ray &r) {
    const float4 org = __ldg(nodes - 4);
    return Ray{r.ox - org.x, r.oy - org.y, r.oz - org.z, r.dx, r.dy, r.dz};
}

template <bool ANY_HIT, int LEAFV = 0, int WIDTH = 2, int STATS = 0>
__device__ __forceinline__ int traverse(const float4 *__restrict__ nodes,
                                        const float4 *__restrict__ tris, const Ray &r, float tmax,
                                        float &t_best) {
    return traverse_impl<ANY_HIT, LEAFV, WIDTH, STATS>(nodes, tris, to_bvh_frame(nodes, r), tmax,
                                                       t_best);
}

}  // namespace trav
}  // namespace ps
