// Host BVH2 builder (binned SAH) for the probe ray tracer.
//
// The reference has no acceleration structure: SceneGeometry.raycast
// (selection.py:66-149) tests every ray against every primitive.  B200 has no
// RT cores, so stage (1) traverses a BVH in SIMT code (csrc/ps_trace.cu);
// this file builds it once per scene on the host.
//
// GPU layout (all little-endian float words):
//   node  = 16 floats: [c0.lo.x c0.hi.x c0.lo.y c0.hi.y]
//                      [c1.lo.x c1.hi.x c1.lo.y c1.hi.y]
//                      [c0.lo.z c0.hi.z c1.lo.z c1.hi.z]
//                      [child0  child1  0       0      ]  (int bits)
//           child >= 0: inner node index; child < 0: leaf with
//           ~child = first_triangle_record << 3 | count (count <= 7)
//   tri   = 12 floats: [v0.xyz prim] [e1.xyz 0] [e2.xyz 0], leaves contiguous
// Edges are formed in double (v1 - v0, v2 - v0) and rounded once to float,
// the same construction the Moller-Trumbore test of the reference uses
// (selection.py:124-126).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "probestream.h"

namespace ps {
void set_last_error(const std::string &msg);
}

namespace {

struct Aabb {
    double lo[3] = {std::numeric_limits<double>::infinity(), std::numeric_limits<double>::infinity(),
                    std::numeric_limits<double>::infinity()};
    double hi[3] = {-std::numeric_limits<double>::infinity(), -std::numeric_limits<double>::infinity(),
                    -std::numeric_limits<double>::infinity()};
    void grow(const Aabb &b) {
        for (int k = 0; k < 3; ++k) {
            lo[k] = std::min(lo[k], b.lo[k]);
            hi[k] = std::max(hi[k], b.hi[k]);
        }
    }
    void grow(const double *p) {
        for (int k = 0; k < 3; ++k) {
            lo[k] = std::min(lo[k], p[k]);
            hi[k] = std::max(hi[k], p[k]);
        }
    }
    double area() const {
        double d[3];
        for (int k = 0; k < 3; ++k) d[k] = std::max(0.0, hi[k] - lo[k]);
        return 2.0 * (d[0] * d[1] + d[1] * d[2] + d[2] * d[0]);
    }
};

struct BuildNode {
    Aabb box;
    int left = -1, right = -1;  // children (inner)
    int first = 0, count = 0;   // primitive range (leaf)
};

// Early split clipping (Ernst & Greiner 2007): a triangle whose box is large
// next to the scene is referenced by the tight boxes of its pieces clipped at
// the box midplanes, so a few huge triangles (the hall's gallery slabs span
// the whole nave) no longer inflate every node above them.  The pieces keep
// the whole triangle's record (a duplicate in each leaf): hits are tested
// against the full triangle, so any piece box the ray enters finds it.
using Poly = std::vector<std::array<double, 3>>;

Poly clip_half(const Poly &in, int axis, double plane, bool keep_below) {
    Poly out;
    const size_t n = in.size();
    for (size_t i = 0; i < n; ++i) {
        const auto &a = in[i], &b = in[(i + 1) % n];
        const double da = keep_below ? plane - a[axis] : a[axis] - plane;
        const double db = keep_below ? plane - b[axis] : b[axis] - plane;
        if (da >= 0) out.push_back(a);
        if ((da >= 0) != (db >= 0)) {
            const double t = da / (da - db);
            std::array<double, 3> p;
            for (int k = 0; k < 3; ++k) p[k] = a[k] + t * (b[k] - a[k]);
            p[axis] = plane;
            out.push_back(p);
        }
    }
    return out;
}

void split_refs(int tri, const Poly &poly, const Aabb &box, double limit, int depth,
                std::vector<Aabb> &boxes, std::vector<int> &tris) {
    int axis = 0;
    for (int k = 1; k < 3; ++k)
        if (box.hi[k] - box.lo[k] > box.hi[axis] - box.lo[axis]) axis = k;
    if (box.hi[axis] - box.lo[axis] <= limit || depth == 0 || poly.size() < 3) {
        boxes.push_back(box);
        tris.push_back(tri);
        return;
    }
    const double mid = 0.5 * (box.lo[axis] + box.hi[axis]);
    for (int side = 0; side < 2; ++side) {
        const Poly part = clip_half(poly, axis, mid, side == 0);
        if (part.size() < 3) continue;
        Aabb pb;
        for (const auto &q : part) pb.grow(q.data());
        for (int k = 0; k < 3; ++k) {  // never outside the parent box
            pb.lo[k] = std::max(pb.lo[k], box.lo[k]);
            pb.hi[k] = std::min(pb.hi[k], box.hi[k]);
        }
        split_refs(tri, part, pb, limit, depth - 1, boxes, tris);
    }
}

struct Builder {
    const double *v;
    std::vector<Aabb> tri_box;    // per reference
    std::vector<double> centroid; // per reference
    std::vector<int> ref_tri;     // reference -> triangle
    std::vector<int> order;
    std::vector<BuildNode> nodes;
    int leaf_size;
    double traversal_cost = 1.2;  // SAH: one node visit vs one triangle test
    static constexpr int BINS = 32;

    int build(int first, int count) {
        BuildNode node;
        for (int i = first; i < first + count; ++i) node.box.grow(tri_box[order[i]]);
        node.first = first;
        node.count = count;
        const int id = int(nodes.size());
        nodes.push_back(node);
        if (count <= 1) return id;
        // centroid bounds
        Aabb cb;
        for (int i = first; i < first + count; ++i) cb.grow(&centroid[3 * order[i]]);
        double best_cost = std::numeric_limits<double>::infinity();
        int best_axis = -1, best_split = -1;
        for (int axis = 0; axis < 3; ++axis) {
            const double lo = cb.lo[axis], ext = cb.hi[axis] - cb.lo[axis];
            if (!(ext > 0.0)) continue;
            Aabb bin_box[BINS];
            int bin_cnt[BINS] = {0};
            const double scale = BINS / ext;
            for (int i = first; i < first + count; ++i) {
                int b = int((centroid[3 * order[i] + axis] - lo) * scale);
                b = std::min(std::max(b, 0), BINS - 1);
                bin_cnt[b]++;
                bin_box[b].grow(tri_box[order[i]]);
            }
            double left_area[BINS];
            int left_cnt[BINS];
            Aabb acc;
            int cnt = 0;
            for (int b = 0; b < BINS - 1; ++b) {
                acc.grow(bin_box[b]);
                cnt += bin_cnt[b];
                left_area[b] = cnt ? acc.area() : 0.0;
                left_cnt[b] = cnt;
            }
            Aabb racc;
            int rcnt = 0;
            for (int b = BINS - 1; b > 0; --b) {
                racc.grow(bin_box[b]);
                rcnt += bin_cnt[b];
                const int lc = left_cnt[b - 1];
                if (lc == 0 || rcnt == 0) continue;
                const double cost = left_area[b - 1] * lc + racc.area() * rcnt;
                if (cost < best_cost) {
                    best_cost = cost;
                    best_axis = axis;
                    best_split = b;
                }
            }
        }
        const double parent_area = nodes[id].box.area();
        const double leaf_cost = parent_area * count;
        // traversal cost ~ 1 box pair per node vs 1 triangle per primitive
        const double split_cost = traversal_cost * parent_area + best_cost;
        if (best_axis < 0) {
            if (count <= leaf_size) return id;
            // coincident centroids: split the range in half by index
            const int half = count / 2;
            const int l = build(first, half);
            const int r = build(first + half, count - half);
            nodes[id].left = l;
            nodes[id].right = r;
            return id;
        }
        if (count <= leaf_size && leaf_cost <= split_cost) return id;
        const double lo = cb.lo[best_axis];
        const double scale = BINS / (cb.hi[best_axis] - cb.lo[best_axis]);
        auto mid_it = std::partition(order.begin() + first, order.begin() + first + count, [&](int t) {
            int b = int((centroid[3 * t + best_axis] - lo) * scale);
            b = std::min(std::max(b, 0), BINS - 1);
            return b < best_split;
        });
        int mid = int(mid_it - order.begin());
        if (mid == first || mid == first + count) mid = first + count / 2;
        int l = build(first, mid - first);
        int r = build(mid, first + count - mid);
        nodes[id].left = l;
        nodes[id].right = r;
        return id;
    }
};

}  // namespace

namespace {

constexpr int32_t EMPTY_CHILD = 0x7fffffff;

// round outward so the float box contains the double box
float round_down(double x) {
    float f = float(x);
    return double(f) > x ? std::nextafter(f, -INFINITY) : f;
}
float round_up(double x) {
    float f = float(x);
    return double(f) < x ? std::nextafter(f, INFINITY) : f;
}
void set_int(float *f, int32_t v) { std::memcpy(f, &v, 4); }

struct Wide {
    int kids[4];
    int n;
};

// IEEE binary16 helpers for the fp16-box BVH4 (round to nearest even, then
// nudged outward so the half box contains the double box)
uint16_t f2h_rne(float f) {
    uint32_t x;
    std::memcpy(&x, &f, 4);
    const uint32_t sign = (x >> 16) & 0x8000u;
    x &= 0x7FFFFFFFu;
    if (x >= 0x47800000u) return uint16_t(sign | 0x7C00u);  // overflow -> inf
    if (x < 0x38800000u) {  // subnormal half
        const float a = std::fabs(f) * 16777216.0f;  // / 2^-24
        return uint16_t(sign | uint16_t(std::nearbyint(a)));
    }
    uint32_t m = x + 0xFFFu + ((x >> 13) & 1u);  // round mantissa to 10 bits, ties to even
    return uint16_t(sign | ((m - 0x38000000u) >> 13));
}
double h2d(uint16_t h) {
    const int e = (h >> 10) & 0x1F, m = h & 0x3FF;
    const double s = (h & 0x8000) ? -1.0 : 1.0;
    if (e == 0) return s * std::ldexp(double(m), -24);
    if (e == 31) return m ? NAN : s * INFINITY;
    return s * std::ldexp(double(m | 0x400), e - 25);
}
uint16_t h_up(uint16_t h) { return h == 0x8000u ? 1 : ((h & 0x8000u) ? h - 1 : h + 1); }
uint16_t h_down(uint16_t h) { return h == 0 ? 0x8001u : ((h & 0x8000u) ? h + 1 : h - 1); }
uint16_t half_down(double x) {
    uint16_t h = f2h_rne(float(x));
    while (h2d(h) > x) h = h_down(h);
    return h;
}
uint16_t half_up(double x) {
    uint16_t h = f2h_rne(float(x));
    while (h2d(h) < x) h = h_up(h);
    return h;
}

}  // namespace

// ---- BVH8 with quantised child boxes --------------------------------------------------
// Node = 96 bytes (24 words), three 32-byte sectors, 32-byte aligned:
//   w0-2   p.x p.y p.z          float quantisation origin (node box lo - one step)
//   w3     e_x | e_y << 8 | e_z << 16 | imask << 24
//                               biased exponents (scale_a = 2^(e_a - 127)) and the
//                               inner-child slot mask
//   w4     child_base           node index of the first inner child; a node's inner
//                               children are contiguous, in slot order
//   w5     tri_base             first triangle record of the node's leaf children
//                               (contiguous, in slot order)
//   w6-7   meta[8]              leaf slot: offset (bits 0-4) from tri_base | count << 5
//   w8-9   qlo_x[8]  w10-11 qlo_y[8]  w12-13 qlo_z[8]  w14-15 qhi_x[8]
//   w16-17 qhi_y[8]  w18-19 qhi_z[8]  w20-23 zero
// Child box along axis a = p_a + scale_a * [qlo, qhi], rounded outward by one
// extra step: the device evaluates the slab distance as
// fma(float(0x4B000000 | q), scale * idir, fma(p, idir, -o * idir) - 2^23 * scale * idir),
// whose rounding error is at most half a step (plus the fp32 rounding the float
// box test has too), so the decoded box still contains the child.  Empty slots:
// qlo = 255, qhi = 0 (entry beyond exit for either direction sign: never hit).
// Slots: child c goes to the slot s minimising dot(centroid_c - centroid, d_s),
// d_s = the diagonal of octant s (bit a set: axis a negative), greedily; a ray of
// octant o then visits hit inner slots in ascending s ^ o, which approximates
// front-to-back order without sorting (Ylitie et al. 2017, simplified).
constexpr int N8_WORDS = 24;

struct Quant {
    float p;
    int e;  // biased exponent byte
    double scale;
};

Quant quantise_axis(double lo, double hi) {
    const double ext = std::max(0.0, hi - lo);
    int e = ext > 0 ? int(std::ceil(std::log2(ext / 252.0))) : -126;
    e = std::max(e, -126);
    for (;; ++e) {
        if (e > 127) throw std::invalid_argument("scene extent too large for the BVH8 quantisation");
        const double s = std::ldexp(1.0, e);
        const float p = round_down(lo - s);
        // every child plane maps into [1, 254] before the one-step margin
        if ((hi - double(p)) / s + 1.0 <= 254.0 && (lo - double(p)) / s >= 1.0) return {p, e + 127, s};
    }
}

int emit_bvh8(const Builder &b, const double *vertices, int64_t tri_count, ps_bvh_sizes *sizes,
              float *nodes_out, float *tris_out) {
    const auto &bn = b.nodes;
    auto is_leaf = [&](int id) { return bn[id].left < 0; };
    auto collapse = [&](int id) {
        std::vector<int> kids;
        if (is_leaf(id)) {
            kids.push_back(id);  // the whole scene is one leaf
            return kids;
        }
        kids = {bn[id].left, bn[id].right};
        while (kids.size() < 8) {
            int best = -1;
            double area = -1.0;
            for (int k = 0; k < int(kids.size()); ++k)
                if (!is_leaf(kids[k]) && bn[kids[k]].box.area() > area) {
                    area = bn[kids[k]].box.area();
                    best = k;
                }
            if (best < 0) break;
            const int c = kids[best];
            kids[best] = bn[c].left;
            kids.insert(kids.begin() + best + 1, bn[c].right);
        }
        return kids;
    };
    struct Out {
        int build_id;
        std::vector<int> slot_kid;  // 8 entries, -1 = empty
        int child_base = 0, tri_base = 0;
        std::vector<int> leaf_off;  // per slot
        int depth = 1;
    };
    std::vector<Out> out;
    std::vector<int> leaf_order;  // build leaves in record order
    int64_t slots = 0, max_depth = 1;
    out.push_back(Out{0, {}, 0, 0, {}, 1});
    for (size_t i = 0; i < out.size(); ++i) {  // BFS: children get consecutive indices
        const std::vector<int> kids = collapse(out[i].build_id);
        const Aabb &pb = bn[out[i].build_id].box;
        double pc[3];
        for (int a = 0; a < 3; ++a) pc[a] = 0.5 * (pb.lo[a] + pb.hi[a]);
        // greedy slot assignment by the lowest dot(centroid - parent centroid, d_s)
        std::vector<int> slot_kid(8, -1);
        std::vector<char> used(kids.size(), 0);
        for (size_t round = 0; round < kids.size(); ++round) {
            double best = std::numeric_limits<double>::infinity();
            int bk = -1, bs = -1;
            for (size_t k = 0; k < kids.size(); ++k) {
                if (used[k]) continue;
                const Aabb &cb = bn[kids[k]].box;
                for (int sl = 0; sl < 8; ++sl) {
                    if (slot_kid[sl] >= 0) continue;
                    double d = 0.0;
                    for (int a = 0; a < 3; ++a)
                        d += (0.5 * (cb.lo[a] + cb.hi[a]) - pc[a]) * ((sl >> a) & 1 ? -1.0 : 1.0);
                    if (d < best) {
                        best = d;
                        bk = int(k);
                        bs = sl;
                    }
                }
            }
            slot_kid[bs] = kids[bk];
            used[bk] = 1;
        }
        Out &o = out[i];
        o.slot_kid = slot_kid;
        o.leaf_off.assign(8, 0);
        o.child_base = int(out.size());
        o.tri_base = int(slots);
        int off = 0;
        for (int sl = 0; sl < 8; ++sl) {
            const int c = slot_kid[sl];
            if (c < 0 || !is_leaf(c)) continue;
            if (bn[c].count > 7) throw std::invalid_argument("BVH8 leaf with more than 7 triangles");
            o.leaf_off[sl] = off;
            off += bn[c].count;
            leaf_order.push_back(c);
        }
        if (off > 31) throw std::invalid_argument("BVH8 node with more than 31 leaf triangles");
        slots += off;
        const int depth = o.depth;
        for (int sl = 0; sl < 8; ++sl) {
            const int c = out[i].slot_kid[sl];
            if (c >= 0 && !is_leaf(c)) {
                out.push_back(Out{c, {}, 0, 0, {}, depth + 1});
                max_depth = std::max<int64_t>(max_depth, depth + 1);
            }
        }
    }
    sizes->node_count = int64_t(out.size());
    sizes->tri_count = tri_count;
    sizes->tri_slots = slots;
    sizes->max_depth = max_depth;
    if (!nodes_out || !tris_out) return PS_OK;
    for (size_t i = 0; i < out.size(); ++i) {
        const Out &o = out[i];
        float *nd = nodes_out + N8_WORDS * i;
        std::memset(nd, 0, N8_WORDS * 4);
        uint8_t *bytes = reinterpret_cast<uint8_t *>(nd);
        Aabb box;  // union of the children
        for (int sl = 0; sl < 8; ++sl)
            if (o.slot_kid[sl] >= 0) box.grow(bn[o.slot_kid[sl]].box);
        Quant q[3];
        for (int a = 0; a < 3; ++a) {
            q[a] = quantise_axis(box.lo[a], box.hi[a]);
            nd[a] = q[a].p;
            bytes[12 + a] = uint8_t(q[a].e);
        }
        uint8_t imask = 0;
        int inner_rank = 0;
        for (int sl = 0; sl < 8; ++sl) {
            const int c = o.slot_kid[sl];
            uint8_t *qlo = bytes + 32, *qhi = bytes + 56;  // qlo x/y/z at 32/40/48, qhi at 56/64/72
            if (c < 0) {
                for (int a = 0; a < 3; ++a) {
                    qlo[8 * a + sl] = 255;
                    qhi[8 * a + sl] = 0;
                }
                continue;
            }
            const Aabb &cb = bn[c].box;
            for (int a = 0; a < 3; ++a) {
                const double lo = std::floor((cb.lo[a] - double(q[a].p)) / q[a].scale) - 1.0;
                const double hi = std::ceil((cb.hi[a] - double(q[a].p)) / q[a].scale) + 1.0;
                if (lo < 0.0 || hi > 255.0) throw std::logic_error("BVH8 quantisation out of range");
                qlo[8 * a + sl] = uint8_t(lo);
                qhi[8 * a + sl] = uint8_t(hi);
            }
            if (is_leaf(c)) {
                bytes[24 + sl] = uint8_t(o.leaf_off[sl] | (bn[c].count << 5));
            } else {
                imask |= uint8_t(1u << sl);
                ++inner_rank;
            }
        }
        bytes[15] = imask;
        set_int(nd + 4, o.child_base);
        set_int(nd + 5, o.tri_base);
        (void)inner_rank;
    }
    int64_t s = 0;
    for (int id : leaf_order) {
        const BuildNode &l = bn[id];
        for (int i = l.first; i < l.first + l.count; ++i) {
            const int t = b.ref_tri[b.order[i]];
            const double *p = vertices + 9 * size_t(t);
            float *r = tris_out + 12 * s;
            r[0] = float(p[0]); r[1] = float(p[1]); r[2] = float(p[2]);
            set_int(r + 3, t);
            r[4] = float(p[3] - p[0]); r[5] = float(p[4] - p[1]); r[6] = float(p[5] - p[2]);
            r[7] = 0.f;
            r[8] = float(p[6] - p[0]); r[9] = float(p[7] - p[1]); r[10] = float(p[8] - p[2]);
            r[11] = 0.f;
            ++s;
        }
    }
    return PS_OK;
}

// ---- BVH4 with origin-relative fp16 boxes (width 3) ------------------------------------
// Node = 64 bytes (16 words), two 32-byte sectors -> two 256-bit loads:
//   w0-3   lo_x[4] hi_x[4]   halves, relative to the node origin
//   w4-7   lo_y[4] hi_y[4]
//   w8-11  lo_z[4] hi_z[4]
//   w12    origin_x | origin_y << 16   (halves: the node box lo rounded down)
//   w13    origin_z | meta << 16       meta nibble per slot: 0 empty, 15 inner
//                                      child, else leaf 1 + 2 * offset + (count - 1)
//   w14    child_base                  node index of the first inner child (a
//                                      node's inner children are contiguous)
//   w15    tri_base                    first triangle record of its leaves
// Relative boxes keep fp16's 11 bits for the node's own extent (a leaf box of a
// 0.1-unit triangle is inflated by ~1e-4, where absolute fp16 boxes at
// coordinate 30 would add 0.016 per side); lo rounded down, hi up, so the
// decoded box contains the child.  Empty slots: lo = +inf, hi = -inf.
void emit_halfbox(double lo, double hi, double origin, uint16_t &qlo, uint16_t &qhi) {
    qlo = half_down(lo - origin);
    qhi = half_up(hi - origin);
    if (!(origin + h2d(qlo) <= lo) || !(origin + h2d(qhi) >= hi))
        throw std::logic_error("relative fp16 box not conservative");
}

int emit_bvh4r(const Builder &b, const double *vertices, int64_t tri_count, ps_bvh_sizes *sizes,
               float *nodes_out, float *tris_out) {
    const auto &bn = b.nodes;
    auto is_leaf = [&](int id) { return bn[id].left < 0; };
    struct Out {
        int build_id, depth;
        std::vector<int> kids;
        int child_base = 0, tri_base = 0;
    };
    std::vector<Out> out{{0, 1, {}, 0, 0}};
    std::vector<int> leaf_order;
    int64_t slots = 0, max_depth = 1;
    for (size_t i = 0; i < out.size(); ++i) {
        std::vector<int> kids;
        const int id = out[i].build_id;
        if (is_leaf(id)) {
            kids.push_back(id);
        } else {
            kids = {bn[id].left, bn[id].right};
            while (kids.size() < 4) {
                int best = -1;
                double area = -1.0;
                for (int k = 0; k < int(kids.size()); ++k)
                    if (!is_leaf(kids[k]) && bn[kids[k]].box.area() > area) {
                        area = bn[kids[k]].box.area();
                        best = k;
                    }
                if (best < 0) break;
                const int c = kids[best];
                kids[best] = bn[c].left;
                kids.insert(kids.begin() + best + 1, bn[c].right);
            }
        }
        out[i].kids = kids;
        out[i].child_base = int(out.size());
        out[i].tri_base = int(slots);
        int off = 0;
        for (int c : kids)
            if (is_leaf(c)) {
                if (bn[c].count > 2) throw std::invalid_argument("width-3 leaf with > 2 triangles");
                leaf_order.push_back(c);
                off += bn[c].count;
            }
        slots += off;
        const int depth = out[i].depth;
        for (int c : kids)
            if (!is_leaf(c)) {
                out.push_back(Out{c, depth + 1, {}, 0, 0});
                max_depth = std::max<int64_t>(max_depth, depth + 1);
            }
    }
    sizes->node_count = int64_t(out.size());
    sizes->tri_count = tri_count;
    sizes->tri_slots = slots;
    sizes->max_depth = max_depth;
    if (!nodes_out || !tris_out) return PS_OK;
    for (size_t i = 0; i < out.size(); ++i) {
        const Out &o = out[i];
        float *nd = nodes_out + 16 * i;
        std::memset(nd, 0, 64);
        uint16_t *hb = reinterpret_cast<uint16_t *>(nd);
        Aabb box;
        for (int c : o.kids) box.grow(bn[c].box);
        double org[3];
        uint16_t org_h[3];
        for (int a = 0; a < 3; ++a) {
            org_h[a] = half_down(box.lo[a]);
            org[a] = h2d(org_h[a]);
        }
        uint32_t meta = 0;
        int off = 0;
        for (int k = 0; k < 4; ++k) {
            if (k >= int(o.kids.size())) {
                for (int a = 0; a < 3; ++a) {
                    hb[8 * a + k] = 0x7C00u;
                    hb[8 * a + 4 + k] = 0xFC00u;
                }
                continue;
            }
            const int c = o.kids[k];
            const Aabb &cb = bn[c].box;
            for (int a = 0; a < 3; ++a) emit_halfbox(cb.lo[a], cb.hi[a], org[a], hb[8 * a + k], hb[8 * a + 4 + k]);
            uint32_t nib;
            if (is_leaf(c)) {
                nib = 1u + 2u * uint32_t(off) + uint32_t(bn[c].count - 1);
                off += bn[c].count;
            } else {
                nib = 15u;
            }
            meta |= nib << (4 * k);
        }
        hb[24] = org_h[0];
        hb[25] = org_h[1];
        hb[26] = org_h[2];
        hb[27] = uint16_t(meta);
        set_int(nd + 14, o.child_base);
        set_int(nd + 15, o.tri_base);
    }
    int64_t s = 0;
    for (int id : leaf_order) {
        const BuildNode &l = bn[id];
        for (int i = l.first; i < l.first + l.count; ++i) {
            const int t = b.ref_tri[b.order[i]];
            const double *p = vertices + 9 * size_t(t);
            float *r = tris_out + 12 * s;
            r[0] = float(p[0]); r[1] = float(p[1]); r[2] = float(p[2]);
            set_int(r + 3, t);
            r[4] = float(p[3] - p[0]); r[5] = float(p[4] - p[1]); r[6] = float(p[5] - p[2]);
            r[7] = 0.f;
            r[8] = float(p[6] - p[0]); r[9] = float(p[7] - p[1]); r[10] = float(p[8] - p[2]);
            r[11] = 0.f;
            ++s;
        }
    }
    return PS_OK;
}

// Shared implementation: binned-SAH binary build, then emission as BVH2
// (16-float nodes, see the header comment) or BVH4 (32-float nodes: lo.x[4]
// hi.x[4] lo.y[4] hi.y[4] lo.z[4] hi.z[4] child[4] pad[4]; a BVH2 node's
// grandchildren are pulled up, largest surface area first, until four
// children; unused slots hold child = 0x7fffffff).
static int bvh_build_impl(const double *vertices, int64_t tri_count, int leaf_size, int width,
                          ps_bvh_sizes *sizes, float *nodes_out, float *tris_out) {
    try {
        if (!sizes) throw std::invalid_argument("sizes must not be NULL");
        if (tri_count < 1) throw std::invalid_argument("scene needs at least one triangle");
        if (tri_count > (int64_t(1) << 27)) throw std::invalid_argument("too many triangles");
        if (leaf_size < 1 || leaf_size > 7) throw std::invalid_argument("leaf_size in [1, 7]");
        // width 5 = BVH4 with fp16 child boxes (64-byte nodes); width 8 = BVH8 with
        // 8-bit quantised child boxes (96-byte nodes, see emit_bvh8)
        // width 3 = BVH4 with fp16 boxes relative to an fp16 node origin and
        // compact child references (64-byte nodes, see emit_bvh4r)
        if (width != 2 && width != 3 && width != 4 && width != 5 && width != 8)
            throw std::invalid_argument("width must be 2, 3, 4, 5 or 8");
        if (width == 8 && leaf_size > 3) throw std::invalid_argument("BVH8 leaves hold <= 3 triangles");
        if (width == 3 && leaf_size > 2) throw std::invalid_argument("width-3 leaves hold <= 2 triangles");
        const bool half_boxes = width == 5;
        if (half_boxes) width = 4;
        Builder b;
        b.v = vertices;
        b.leaf_size = leaf_size;
        if (const char *ct = std::getenv("PS_BVH_CT")) b.traversal_cost = std::atof(ct);  // tuning knob
        const int ntri = int(tri_count);
        Aabb scene_box;
        for (int t = 0; t < ntri; ++t)
            for (int k = 0; k < 3; ++k) scene_box.grow(vertices + 9 * size_t(t) + 3 * k);
        double diag = 0.0;
        for (int k = 0; k < 3; ++k) diag += (scene_box.hi[k] - scene_box.lo[k]) * (scene_box.hi[k] - scene_box.lo[k]);
        // split references longer than diag / PS_BVH_SPLIT (tuning knob; default 0 = off:
        // on the C4 hall 24 / 48 / 96 / 192 traced in 7.95 / 8.00 / 8.15 / 8.36 ms vs 7.90
        // unsplit -- its few long triangles are thin slabs the binned SAH already isolates)
        const char *env = std::getenv("PS_BVH_SPLIT");
        const double div = env ? std::atof(env) : 0.0;
        const double limit = div > 0 ? std::sqrt(diag) / div : std::numeric_limits<double>::infinity();
        for (int t = 0; t < ntri; ++t) {
            const double *p = vertices + 9 * size_t(t);
            Aabb tb;
            for (int k = 0; k < 3; ++k) tb.grow(p + 3 * k);
            Poly poly{{p[0], p[1], p[2]}, {p[3], p[4], p[5]}, {p[6], p[7], p[8]}};
            split_refs(t, poly, tb, limit, 8, b.tri_box, b.ref_tri);
        }
        const int n = int(b.ref_tri.size());
        b.centroid.resize(3 * size_t(n));
        b.order.resize(n);
        for (int r = 0; r < n; ++r) {
            for (int a = 0; a < 3; ++a) b.centroid[3 * r + a] = 0.5 * (b.tri_box[r].lo[a] + b.tri_box[r].hi[a]);
            b.order[r] = r;
        }
        b.nodes.reserve(2 * size_t(n));
        b.build(0, n);
        if (width == 8) return emit_bvh8(b, vertices, tri_count, sizes, nodes_out, tris_out);
        if (width == 3) return emit_bvh4r(b, vertices, tri_count, sizes, nodes_out, tris_out);

        // collapse into width-ary nodes (preorder), leaves numbered in DFS order
        std::vector<Wide> wide;
        std::vector<int> wide_of(b.nodes.size(), -1);
        std::vector<int> leaf_slot(b.nodes.size(), -1);
        std::vector<int> leaves;
        int64_t slots = 0, max_depth = 0;
        std::vector<std::pair<int, int>> st{{0, 1}};  // (build node, depth)
        while (!st.empty()) {
            auto [id, depth] = st.back();
            st.pop_back();
            Wide w{{0, 0, 0, 0}, 0};
            if (b.nodes[id].left < 0) {
                w.kids[0] = id;  // the whole scene is one leaf
                w.n = 1;
            } else {
                std::vector<int> kids{b.nodes[id].left, b.nodes[id].right};
                while (int(kids.size()) < width) {
                    int best = -1;
                    double area = -1.0;
                    for (int k = 0; k < int(kids.size()); ++k)
                        if (b.nodes[kids[k]].left >= 0 && b.nodes[kids[k]].box.area() > area) {
                            area = b.nodes[kids[k]].box.area();
                            best = k;
                        }
                    if (best < 0) break;
                    const int c = kids[best];
                    kids[best] = b.nodes[c].left;
                    kids.insert(kids.begin() + best + 1, b.nodes[c].right);
                }
                for (int k = 0; k < int(kids.size()); ++k) w.kids[k] = kids[k];
                w.n = int(kids.size());
            }
            wide_of[id] = int(wide.size());
            wide.push_back(w);
            max_depth = std::max<int64_t>(max_depth, depth);
            // children: leaves get slots now (DFS order), inner ones are visited next
            for (int k = w.n - 1; k >= 0; --k)
                if (b.nodes[w.kids[k]].left >= 0) st.push_back({w.kids[k], depth + 1});
            for (int k = 0; k < w.n; ++k) {
                const int c = w.kids[k];
                if (b.nodes[c].left < 0 && leaf_slot[c] < 0) {
                    leaf_slot[c] = int(slots);
                    leaves.push_back(c);
                    slots += b.nodes[c].count;
                }
            }
        }
        sizes->node_count = int64_t(wide.size());
        sizes->tri_count = tri_count;
        sizes->tri_slots = slots;
        sizes->max_depth = std::max<int64_t>(max_depth, 1);
        if (!nodes_out || !tris_out) return PS_OK;

        auto child_ref = [&](int id) -> int32_t {
            if (b.nodes[id].left >= 0) return wide_of[id];
            return ~int32_t((leaf_slot[id] << 3) | b.nodes[id].count);
        };
        const int nf = (width == 2 || half_boxes) ? 16 : 32;
        if (half_boxes) {
            // node: [lo_x[4] hi_x[4]] [lo_y[4] hi_y[4]] [lo_z[4] hi_z[4]] as halves, child[4]
            for (size_t g = 0; g < wide.size(); ++g) {
                const Wide &w = wide[g];
                float *nd = nodes_out + 16 * g;
                std::memset(nd, 0, 64);
                uint16_t *hb = reinterpret_cast<uint16_t *>(nd);
                for (int k = 0; k < 4; ++k) {
                    if (k >= w.n) {  // inverted infinite box: the octant test never hits it
                        set_int(nd + 12 + k, EMPTY_CHILD);
                        for (int a = 0; a < 3; ++a) {
                            hb[8 * a + k] = 0x7C00u;
                            hb[8 * a + 4 + k] = 0xFC00u;
                        }
                        continue;
                    }
                    const Aabb &bx = b.nodes[w.kids[k]].box;
                    for (int a = 0; a < 3; ++a) {
                        hb[8 * a + k] = half_down(bx.lo[a]);
                        hb[8 * a + 4 + k] = half_up(bx.hi[a]);
                    }
                    set_int(nd + 12 + k, child_ref(w.kids[k]));
                }
            }
        } else
        for (size_t g = 0; g < wide.size(); ++g) {
            const Wide &w = wide[g];
            float *nd = nodes_out + nf * g;  // fp32 boxes
            std::memset(nd, 0, nf * 4);
            for (int k = 0; k < width; ++k) {
                if (k >= w.n) {  // unused slot
                    set_int(nd + (width == 2 ? 12 : 24) + k, width == 2 ? ~int32_t(0) : EMPTY_CHILD);
                    if (width == 2) {  // inverted box never hit by the BVH2 test
                        nd[4 * k + 0] = 1.f; nd[4 * k + 1] = -1.f;
                        nd[4 * k + 2] = 1.f; nd[4 * k + 3] = -1.f;
                        nd[8 + 2 * k] = 1.f; nd[8 + 2 * k + 1] = -1.f;
                    } else {  // lo = +inf, hi = -inf: the octant test's entry plane is
                              // +inf for either sign, so it never hits (no child check)
                        for (int a = 0; a < 3; ++a) {
                            nd[8 * a + k] = INFINITY;
                            nd[8 * a + 4 + k] = -INFINITY;
                        }
                    }
                    continue;
                }
                const Aabb &bx = b.nodes[w.kids[k]].box;
                if (width == 2) {
                    nd[4 * k + 0] = round_down(bx.lo[0]);
                    nd[4 * k + 1] = round_up(bx.hi[0]);
                    nd[4 * k + 2] = round_down(bx.lo[1]);
                    nd[4 * k + 3] = round_up(bx.hi[1]);
                    nd[8 + 2 * k] = round_down(bx.lo[2]);
                    nd[8 + 2 * k + 1] = round_up(bx.hi[2]);
                    set_int(nd + 12 + k, child_ref(w.kids[k]));
                } else {
                    nd[0 + k] = round_down(bx.lo[0]);
                    nd[4 + k] = round_up(bx.hi[0]);
                    nd[8 + k] = round_down(bx.lo[1]);
                    nd[12 + k] = round_up(bx.hi[1]);
                    nd[16 + k] = round_down(bx.lo[2]);
                    nd[20 + k] = round_up(bx.hi[2]);
                    set_int(nd + 24 + k, child_ref(w.kids[k]));
                }
            }
        }
        int64_t s = 0;
        for (int id : leaves) {
            const BuildNode &bn = b.nodes[id];
            for (int i = bn.first; i < bn.first + bn.count; ++i) {
                const int t = b.ref_tri[b.order[i]];
                const double *p = vertices + 9 * size_t(t);
                float *r = tris_out + 12 * s;
                r[0] = float(p[0]); r[1] = float(p[1]); r[2] = float(p[2]);
                set_int(r + 3, t);
                r[4] = float(p[3] - p[0]); r[5] = float(p[4] - p[1]); r[6] = float(p[5] - p[2]);
                r[7] = 0.f;
                r[8] = float(p[6] - p[0]); r[9] = float(p[7] - p[1]); r[10] = float(p[8] - p[2]);
                r[11] = 0.f;
                ++s;
            }
        }
        return PS_OK;
    } catch (const std::exception &e) {
        ps::set_last_error(e.what());
        return PS_ERR_VALUE;
    }
}

extern "C" int ps_bvh_build(const double *vertices, int64_t tri_count, int leaf_size,
                            ps_bvh_sizes *sizes, float *nodes_out, float *tris_out) {
    return bvh_build_impl(vertices, tri_count, leaf_size, 2, sizes, nodes_out, tris_out);
}

extern "C" int ps_bvh_build_wide(const double *vertices, int64_t tri_count, int leaf_size,
                                 int width, ps_bvh_sizes *sizes, float *nodes_out,
                                 float *tris_out) {
    return bvh_build_impl(vertices, tri_count, leaf_size, width, sizes, nodes_out, tris_out);
}
