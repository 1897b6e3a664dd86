// §8(f) row 2: potentially visible probe set on the GPU (selection.py:329-407).
//
// One thread per PVS ray (frustum grid + fibonacci sphere, built on the host
// exactly as pvs_rays does, selection.py:375-381) plus one for the camera's
// own cell.  The nearest hit is found with the float32 BVH traversal of the
// probe tracer, then its distance is recomputed in double precision with the
// reference's Moller-Trumbore arithmetic (selection.py:123-139) on the
// original float64 vertices, so hit points -- and the probe cages they select
// (cage_probes, selection.py:329-351) -- are the reference's bit for bit
// whenever the same triangle is found.  Rays that escape contribute the cage
// of the point where they leave the volume's box (_volume_exit_points,
// selection.py:359-372).  Cages are ORed into a bitmap, ANDed with the active
// flags and compacted (np.flatnonzero).
#include <cuda_runtime.h>

#include <cmath>

#include "ps_common.cuh"
#include "ps_traverse.cuh"

namespace ps {

size_t compact_workspace_bytes(int64_t n);
void compact_bits(const uint32_t *bits, int64_t n, int64_t *out, const int32_t *aux_pairs,
                  int64_t *out_count, void *ws, size_t ws_bytes, cudaStream_t s);

namespace {

struct PvsArgs {
    const float *nodes;
    int width;
    const float *tris;
    const double *verts;  // (T, 3, 3) float64
    const double *dirs;   // (n, 3)
    int64_t n;
    double o[3];
    int nx, ny, nz;
    double vo[3], vs[3];  // volume origin / spacing
    uint32_t *bits;
};

__device__ __forceinline__ double dot3d(const double *a, const double *b) {
    return __dadd_rn(__dadd_rn(__dmul_rn(a[0], b[0]), __dmul_rn(a[1], b[1])), __dmul_rn(a[2], b[2]));
}

__device__ __forceinline__ void cross3d(const double *a, const double *b, double *c) {
    c[0] = __dsub_rn(__dmul_rn(a[1], b[2]), __dmul_rn(a[2], b[1]));
    c[1] = __dsub_rn(__dmul_rn(a[2], b[0]), __dmul_rn(a[0], b[2]));
    c[2] = __dsub_rn(__dmul_rn(a[0], b[1]), __dmul_rn(a[1], b[0]));
}

// reference Moller-Trumbore in float64, no FMA contraction; inf if rejected
__device__ double mt_double(const double *tri, const double *o, const double *d) {
    double e1[3], e2[3], p[3], s[3], q[3];
    for (int k = 0; k < 3; ++k) {
        e1[k] = __dsub_rn(tri[3 + k], tri[k]);
        e2[k] = __dsub_rn(tri[6 + k], tri[k]);
        s[k] = __dsub_rn(o[k], tri[k]);
    }
    cross3d(d, e2, p);
    const double det = dot3d(e1, p);
    if (!(fabs(det) > 1e-6)) return INFINITY;
    const double inv = __ddiv_rn(1.0, det);
    const double u = __dmul_rn(dot3d(s, p), inv);
    cross3d(s, e1, q);
    const double v = __dmul_rn(dot3d(d, q), inv);
    const double t = __dmul_rn(dot3d(e2, q), inv);
    if (u >= -1e-6 && v >= -1e-6 && __dadd_rn(u, v) <= 1.0 + 1e-6 && t > 1e-6) return t;
    return INFINITY;
}

__device__ void set_cage(const PvsArgs &a, const double *pt) {
    const int dims[3] = {a.nx, a.ny, a.nz};
    int64_t low[3];
    for (int k = 0; k < 3; ++k) {
        const double rel = __ddiv_rn(__dsub_rn(pt[k], a.vo[k]), a.vs[k]);
        int64_t l = int64_t(floor(rel));
        const int64_t hi = dims[k] - 2 > 0 ? dims[k] - 2 : 0;
        l = l < 0 ? 0 : (l > hi ? hi : l);
        low[k] = l;
    }
    for (int dk = 0; dk < 2; ++dk)
        for (int dj = 0; dj < 2; ++dj)
            for (int di = 0; di < 2; ++di) {
                const int64_t i = low[0] + di < a.nx - 1 ? low[0] + di : a.nx - 1;
                const int64_t j = low[1] + dj < a.ny - 1 ? low[1] + dj : a.ny - 1;
                const int64_t k = low[2] + dk < a.nz - 1 ? low[2] + dk : a.nz - 1;
                const int64_t p = i + int64_t(a.nx) * (j + int64_t(a.ny) * k);
                atomicOr(a.bits + (p >> 5), 1u << (p & 31));
            }
}

__global__ void __launch_bounds__(128) pvs_kernel(PvsArgs a) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i <= a.n;
         i += int64_t(gridDim.x) * blockDim.x) {
        if (i == a.n) {  // the camera's own cell (selection.py:404-405)
            set_cage(a, a.o);
            continue;
        }
        const double *d = a.dirs + 3 * i;
        float tf;
        const trav::Ray ray{float(a.o[0]), float(a.o[1]), float(a.o[2]),
                            float(d[0]), float(d[1]), float(d[2])};
        const float4 *nd = reinterpret_cast<const float4 *>(a.nodes);
        const float4 *tr = reinterpret_cast<const float4 *>(a.tris);
        const int slot = a.width == 3   ? trav::traverse<false, 1, 17>(nd, tr, ray, INFINITY, tf)
                         : a.width == 8 ? trav::traverse<false, 1, 16>(nd, tr, ray, INFINITY, tf)
                         : a.width == 5 ? trav::traverse<false, 1, 5>(nd, tr, ray, INFINITY, tf)
                         : a.width == 4 ? trav::traverse<false, 1, 4>(nd, tr, ray, INFINITY, tf)
                                        : trav::traverse<false, 1, 2>(nd, tr, ray, INFINITY, tf);
        double pt[3];
        if (slot >= 0) {
            const int prim = __float_as_int(a.tris[12 * slot + 3]);
            double t = mt_double(a.verts + 9 * int64_t(prim), a.o, d);
            if (!isfinite(t)) t = double(tf);
            for (int k = 0; k < 3; ++k) pt[k] = __dadd_rn(a.o[k], __dmul_rn(d[k], t));
            set_cage(a, pt);
            continue;
        }
        // miss: exit point of the volume box
        double tnear = -INFINITY, tfar = INFINITY;
        const int dims[3] = {a.nx, a.ny, a.nz};
        for (int k = 0; k < 3; ++k) {
            const double sd = fabs(d[k]) < 1e-6 ? 1e-6 : d[k];
            const double inv = __ddiv_rn(1.0, sd);
            const double lo = a.vo[k];
            const double hi = __dadd_rn(a.vo[k], __dmul_rn(a.vs[k], double(dims[k] - 1)));
            const double t1 = __dmul_rn(__dsub_rn(lo, a.o[k]), inv);
            const double t2 = __dmul_rn(__dsub_rn(hi, a.o[k]), inv);
            tnear = fmax(tnear, fmin(t1, t2));
            tfar = fmin(tfar, fmax(t1, t2));
        }
        if (tnear <= tfar && tfar > 0.0) {
            for (int k = 0; k < 3; ++k) pt[k] = __dadd_rn(a.o[k], __dmul_rn(d[k], tfar));
            set_cage(a, pt);
        }
    }
}

__global__ void and_active_kernel(uint32_t *bits, const uint8_t *active, int64_t n) {
    const int64_t words = (n + 31) / 32;
    for (int64_t w = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; w < words;
         w += int64_t(gridDim.x) * blockDim.x) {
        uint32_t act = 0;
        for (int b = 0; b < 32; ++b) {
            const int64_t p = w * 32 + b;
            if (p < n && (!active || active[p])) act |= 1u << b;
        }
        bits[w] &= act;
    }
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" {

size_t ps_pvs_workspace_bytes(int64_t probe_count) {
    return compact_workspace_bytes(std::max<int64_t>(probe_count, 1));
}

int ps_pvs(const float *nodes, int32_t bvh_width, const float *tris, const double *vertices,
           const double *ray_dirs, int64_t ray_count, const double *camera, int32_t nx, int32_t ny,
           int32_t nz, const double *volume_origin, const double *volume_spacing,
           const uint8_t *active, uint32_t *mask_bits, int64_t *out_ids, int64_t *out_count,
           void *workspace, size_t workspace_bytes, void *stream) {
    PS_ABI_BEGIN
    if (nx < 1 || ny < 1 || nz < 1) fail(PS_ERR_VALUE, "volume dims must be >= 1");
    if (bvh_width != 2 && bvh_width != 3 && bvh_width != 4 && bvh_width != 5 && bvh_width != 8)
        fail(PS_ERR_VALUE, "bad bvh_width");
    if (ray_count < 0) fail(PS_ERR_VALUE, "negative ray count");
    auto s = as_stream(stream);
    const int64_t n = int64_t(nx) * ny * nz;
    check_cuda(cudaMemsetAsync(mask_bits, 0, size_t(ceil_div(n, 32)) * 4, s), "memset pvs bits");
    PvsArgs a;
    a.nodes = nodes;
    a.width = bvh_width;
    a.tris = tris;
    a.verts = vertices;
    a.dirs = ray_dirs;
    a.n = ray_count;
    for (int k = 0; k < 3; ++k) {
        a.o[k] = camera[k];
        a.vo[k] = volume_origin[k];
        a.vs[k] = volume_spacing[k];
    }
    a.nx = nx;
    a.ny = ny;
    a.nz = nz;
    a.bits = mask_bits;
    const unsigned blocks = unsigned(std::max<int64_t>(1, ceil_div(ray_count + 1, 128)));
    pvs_kernel<<<blocks, 128, 0, s>>>(a);
    check_launch("pvs_kernel");
    and_active_kernel<<<unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(ceil_div(n, 32), 256), 1024))),
                        256, 0, s>>>(mask_bits, active, n);
    check_launch("and_active_kernel");
    if (out_ids || out_count) compact_bits(mask_bits, n, out_ids, nullptr, out_count, workspace, workspace_bytes, s);
    PS_ABI_END
}

}  // extern "C"
