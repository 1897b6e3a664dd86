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
        // width 5 = BVH4 with fp16 child boxes (64-byte nodes)
        if (width != 2 && width != 4 && width != 5) throw std::invalid_argument("width must be 2, 4 or 5");
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
                    if (k >= w.n) {
                        set_int(nd + 12 + k, EMPTY_CHILD);
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
