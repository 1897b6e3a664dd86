/*
 * C restatement of the reference's ray query, SceneGeometry.raycast for
 * triangles (/root/reference/pkg/src/probestream/selection.py:66-93 and
 * :123-149): double precision, brute force over every triangle, nearest hit
 * with the first minimal index winning (np.argmin).  TEST INFRASTRUCTURE
 * ONLY -- the traversal oracle for the GPU BVH tracer and the CPU baseline of
 * stage (1).  Compiled with -ffp-contract=off so every product and sum
 * rounds exactly as numpy's does.
 *
 * Per triangle (selection.py:124-139):
 *   e1 = v1 - v0, e2 = v2 - v0, p = d x e2, det = e1 . p
 *   ok = |det| > 1e-6;  s = o - v0;  u = (s . p) / det;  q = s x e1
 *   v = (d . q) / det;  t = (e2 . q) / det
 *   ok &= u >= -1e-6 && v >= -1e-6 && u + v <= 1 + 1e-6 && t > 1e-6
 * Dot products sum left to right ((a0 b0 + a1 b1) + a2 b2), as numpy's
 * three-element reduction does.
 */
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <stdint.h>

#define EPS 1e-6

static inline double dot3(const double *a, const double *b) {
    return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}

static inline void cross3(const double *a, const double *b, double *out) {
    out[0] = a[1] * b[2] - a[2] * b[1];
    out[1] = a[2] * b[0] - a[0] * b[2];
    out[2] = a[0] * b[1] - a[1] * b[0];
}

/* t of the hit or +inf (the reference's np.where(ok, t, inf)) */
static inline double tri_t(const double *tri, const double *o, const double *d) {
    double e1[3], e2[3], p[3], s[3], q[3];
    for (int k = 0; k < 3; ++k) {
        e1[k] = tri[3 + k] - tri[k];
        e2[k] = tri[6 + k] - tri[k];
        s[k] = o[k] - tri[k];
    }
    cross3(d, e2, p);
    const double det = dot3(e1, p);
    if (!(fabs(det) > EPS)) return INFINITY;
    const double inv = 1.0 / det;
    const double u = dot3(s, p) * inv;
    cross3(s, e1, q);
    const double v = dot3(d, q) * inv;
    const double t = dot3(e2, q) * inv;
    if (u >= -EPS && v >= -EPS && u + v <= 1.0 + EPS && t > EPS) return t;
    return INFINITY;
}

/* OpenMP team size (torchrun exports OMP_NUM_THREADS=1 to every rank; the
 * CPU baseline wants every host thread) */
void oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* nearest hit per ray; prim = -1 on a miss */
int oracle_raycast(const double *tris, int64_t ntri, const double *origins,
                   const double *dirs, int64_t nray, double *t_out, int64_t *prim_out) {
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t r = 0; r < nray; ++r) {
        const double *o = origins + 3 * r, *d = dirs + 3 * r;
        double best = INFINITY;
        int64_t arg = -1;
        for (int64_t i = 0; i < ntri; ++i) {
            const double t = tri_t(tris + 9 * i, o, d);
            if (t < best) {
                best = t;
                arg = i;
            }
        }
        t_out[r] = best;
        prim_out[r] = arg;
    }
    return 0;
}

/* occlusion: any triangle with 1e-6 < t < tmax[r] */
int oracle_occluded(const double *tris, int64_t ntri, const double *origins, const double *dirs,
                    const double *tmax, int64_t nray, uint8_t *out) {
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t r = 0; r < nray; ++r) {
        const double *o = origins + 3 * r, *d = dirs + 3 * r;
        uint8_t hit = 0;
        for (int64_t i = 0; i < ntri && !hit; ++i)
            if (tri_t(tris + 9 * i, o, d) < tmax[r]) hit = 1;
        out[r] = hit;
    }
    return 0;
}
