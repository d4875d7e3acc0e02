// Order-2 chain growth for sm_100a (K7): which triples p -> t -> a of admitted
// pairs survive build_matrix's Markov-2 filter (src/vismatrix.cpp:715-797):
//   feasible(p,t,a) = chain_triple_feasible(p,t,a)                (457-476)
//                   and for every plane in required_planes(t,a) that (p,t)
//                   also has: second_order_check(p,t,a,plane) != None (387-455)
// One thread per candidate triple (warp per prefix pair (p,t), lanes over the
// admitted aims of t), exact FP64 with the reference's operation order; the
// surviving triples are compacted with ballot/popc + one atomic per warp.
#include <algorithm>
#include <cstring>
#include <vector>

#include <cub/cub.cuh>

#include "capi_internal.h"
#include "device.h"

namespace visrt {

#ifndef VISRT_K7_MINB
#define VISRT_K7_MINB 5   // CTAs of 128 threads per SM the chain kernel's register budget targets (96 registers)
#endif

#ifdef VISRT_K7_STATS
// development aid: triples reaching each stage of triple_feasible (total, clip a,
// clip c, section non-empty sum of ns, hull non-empty, overlap, feasible)
__device__ unsigned long long g_k7_stats[8];
#define K7S(i, v) atomicAdd(&g_k7_stats[i], static_cast<unsigned long long>(v))
#else
#define K7S(i, v) ((void)0)
#endif

namespace {

constexpr unsigned kAll = 0xffffffffu;

struct V2 {
    double x, y;
};
struct V3 {
    double x, y, z;
};

__device__ __forceinline__ V3 v3sub(V3 a, V3 b) { return {dsub(a.x, b.x), dsub(a.y, b.y), dsub(a.z, b.z)}; }
__device__ __forceinline__ V3 v3add(V3 a, V3 b) { return {dadd(a.x, b.x), dadd(a.y, b.y), dadd(a.z, b.z)}; }
__device__ __forceinline__ V3 v3mul(V3 a, double s) { return {dmul(a.x, s), dmul(a.y, s), dmul(a.z, s)}; }
__device__ __forceinline__ double v3dot(V3 a, V3 b) {
    return dadd(dadd(dmul(a.x, b.x), dmul(a.y, b.y)), dmul(a.z, b.z));
}
__device__ __forceinline__ V3 v3cross(V3 a, V3 b) {
    return {dsub(dmul(a.y, b.z), dmul(a.z, b.y)), dsub(dmul(a.z, b.x), dmul(a.x, b.z)),
            dsub(dmul(a.x, b.y), dmul(a.y, b.x))};
}
__device__ __forceinline__ V2 v2sub(V2 a, V2 b) { return {dsub(a.x, b.x), dsub(a.y, b.y)}; }
__device__ __forceinline__ double v2dot(V2 a, V2 b) { return dadd(dmul(a.x, b.x), dmul(a.y, b.y)); }
__device__ __forceinline__ double v2cross(V2 a, V2 b) { return dsub(dmul(a.x, b.y), dmul(a.y, b.x)); }
__device__ __forceinline__ double v2norm(V2 a) { return __dsqrt_rn(v2dot(a, a)); }
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }   // std::min
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }   // std::max

// Caps for MAXV-vertex faces: clip <= 2*MAXV points, hull input <= 4*MAXV,
// slice section <= 4*MAXV + C(4*MAXV, 2).
template <int MAXV>
struct Caps {
    static constexpr int kClip = 2 * MAXV;
    static constexpr int kPts = 4 * MAXV;
    static constexpr int kSec = kPts + kPts * (kPts - 1) / 2;
};

struct PlaneD {
    V3 p, n;
    __device__ double sd(V3 q) const { return v3dot(v3sub(q, p), n); }
};

__device__ __forceinline__ V3 face_pt(const DevScene& s, int f, int k) {
    const double* P = s.pts + (static_cast<size_t>(f) * VISRT_MAX_VERTS + k) * 3;
    return {P[0], P[1], P[2]};
}

// clip_polygon_halfspace, src/geom.cpp:191-207
template <int MAXV>
__device__ __noinline__ int clip_halfspace(const DevScene& s, int f, const PlaneD& pl, V3* out) {
    const int n = s.nv[f];
    int c = 0;
    for (int i = 0; i < n; ++i) {
        const V3 a = face_pt(s, f, i), b = face_pt(s, f, (i + 1) % n);
        const double da = pl.sd(a), db = pl.sd(b);
        if (da >= -kEps) out[c++] = a;
        if ((da > kEps && db < -kEps) || (da < -kEps && db > kEps))
            out[c++] = v3add(a, v3mul(v3sub(b, a), __ddiv_rn(da, dsub(da, db))));
    }
    return c < 3 ? 0 : c;
}

// convex_hull_2d, src/geom.cpp:219-242 (sort, tolerance-unique against the
// last kept point like std::unique, Andrew's monotone chain). In place;
// `hull` needs 2*n slots. Returns the hull size (or n unchanged if n < 3).
__device__ __noinline__ int convex_hull(V2* pts, int n, V2* hull) {
    if (n < 3) return n;
    // insertion sort by (x, y)
    for (int i = 1; i < n; ++i) {
        const V2 v = pts[i];
        int j = i - 1;
        while (j >= 0 && (v.x < pts[j].x || (v.x == pts[j].x && v.y < pts[j].y))) {
            pts[j + 1] = pts[j];
            --j;
        }
        pts[j + 1] = v;
    }
    int m = 1;
    for (int i = 1; i < n; ++i) {
        if (fabs(dsub(pts[m - 1].x, pts[i].x)) < kEps && fabs(dsub(pts[m - 1].y, pts[i].y)) < kEps) continue;
        pts[m++] = pts[i];
    }
    n = m;
    if (n < 3) return n;
    int k = 0;
    for (int i = 0; i < n; ++i) {
        while (k >= 2 && v2cross(v2sub(hull[k - 1], hull[k - 2]), v2sub(pts[i], hull[k - 2])) <= 0) --k;
        hull[k++] = pts[i];
    }
    for (int i = n - 1, t = k + 1; i-- > 0;) {
        while (k >= t && v2cross(v2sub(hull[k - 1], hull[k - 2]), v2sub(pts[i], hull[k - 2])) <= 0) --k;
        hull[k++] = pts[i];
    }
    k -= 1;
    for (int i = 0; i < k; ++i) pts[i] = hull[i];
    return k;
}

// axis_separates / separating_axis / has_finite_edge, src/geom.cpp:245-279
__device__ bool axis_separates(const V2* a, int na, const V2* b, int nb, V2 axis) {
    double amin = 1e300, amax = -1e300, bmin = 1e300, bmax = -1e300;
    for (int i = 0; i < na; ++i) {
        const double d = v2dot(a[i], axis);
        amin = smin(amin, d);
        amax = smax(amax, d);
    }
    for (int i = 0; i < nb; ++i) {
        const double d = v2dot(b[i], axis);
        bmin = smin(bmin, d);
        bmax = smax(bmax, d);
    }
    return amax < dsub(bmin, kEps) || bmax < dsub(amin, kEps);
}
__device__ __noinline__ bool separating_axis(const V2* a, int na, const V2* b, int nb) {
    for (int i = 0; i < na; ++i) {
        const V2 e = v2sub(a[(i + 1) % na], a[i]);
        const double len = v2norm(e);
        if (len <= 1e-12) continue;
        if (axis_separates(a, na, b, nb, {__ddiv_rn(-e.y, len), __ddiv_rn(e.x, len)})) return true;
        if (axis_separates(a, na, b, nb, {__ddiv_rn(e.x, len), __ddiv_rn(e.y, len)})) return true;
    }
    return false;
}
__device__ bool has_finite_edge(const V2* p, int n) {
    for (int i = 0; i < n; ++i)
        if (v2norm(v2sub(p[(i + 1) % n], p[i])) > 1e-12) return true;
    return false;
}

// chain_triple_feasible, src/vismatrix.cpp:457-476
template <int MAXV>
__device__ __noinline__ bool triple_feasible(const DevScene& s, int a, int b, int c) {
    const double* N = s.normal + 3 * static_cast<size_t>(b);
    const PlaneD pl{face_pt(s, b, 0), {N[0], N[1], N[2]}};
    V3 pts[Caps<MAXV>::kPts];
    K7S(0, 1);
    const int nl = clip_halfspace<MAXV>(s, a, pl, pts);
    if (nl < 2) return false;
    K7S(1, 1);
    V3 tgt[Caps<MAXV>::kClip];
    const int nt = clip_halfspace<MAXV>(s, c, pl, tgt);
    if (nt < 2) return false;
    K7S(2, 1);
    int np = nl;
    for (int i = 0; i < nt; ++i) {
        const double d2 = dmul(2.0, pl.sd(tgt[i]));   // mirror_point
        pts[np++] = v3sub(tgt[i], v3mul(pl.n, d2));
    }
    // PlaneFrame::from_plane, src/geom.cpp:209-217
    const V3 axis = fabs(pl.n.x) < 0.9 ? V3{1, 0, 0} : V3{0, 1, 0};
    V3 u = v3cross(pl.n, axis);
    const double un = __dsqrt_rn(v3dot(u, u));
    if (un < kEps) return false;   // normalized() would throw; cannot happen for unit normals
    u = {__ddiv_rn(u.x, un), __ddiv_rn(u.y, un), __ddiv_rn(u.z, un)};
    const V3 v = v3cross(pl.n, u);
    auto to2d = [&](V3 p) {
        const V3 r = v3sub(p, pl.p);
        return V2{v3dot(r, u), v3dot(r, v)};
    };
    // hull_plane_slice, src/geom.cpp:292-307
    double d[Caps<MAXV>::kPts];
    for (int i = 0; i < np; ++i) d[i] = pl.sd(pts[i]);
    V2 sec[Caps<MAXV>::kSec];
    int ns = 0;
    for (int i = 0; i < np; ++i) {
        if (fabs(d[i]) <= kEps) sec[ns++] = to2d(pts[i]);
        for (int j = i + 1; j < np; ++j) {
            if ((d[i] > kEps && d[j] < -kEps) || (d[i] < -kEps && d[j] > kEps)) {
                const double t = __ddiv_rn(d[i], dsub(d[i], d[j]));
                sec[ns++] = to2d(v3add(pts[i], v3mul(v3sub(pts[j], pts[i]), t)));
            }
        }
    }
    V2 hull[2 * Caps<MAXV>::kSec];
    K7S(3, ns);
    ns = convex_hull(sec, ns, hull);
    if (ns == 0) return false;
    K7S(4, 1);
    K7S(7, ns);
    V2 mid2d[VISRT_MAX_VERTS];
    const int nm = s.nv[b];
    for (int k = 0; k < nm; ++k) mid2d[k] = to2d(face_pt(s, b, k));
    // convex_polygons_overlap_2d, src/geom.cpp:282-290
    if (separating_axis(sec, ns, mid2d, nm) || separating_axis(mid2d, nm, sec, ns)) return false;
    K7S(5, 1);
    if (!has_finite_edge(sec, ns) && !has_finite_edge(mid2d, nm)) return v2norm(v2sub(sec[0], mid2d[0])) <= kEps;
    K7S(6, 1);
    return true;
}

#ifndef VISRT_K7_SCREEN
#define VISRT_K7_SCREEN 1   // 0: kernel 1 passes every candidate on (A/B: the screen must not change the triples)
#endif
#ifndef VISRT_K7_SPLIT2
#define VISRT_K7_SPLIT2 1   // second_order_check runs as a third kernel over the hull-feasible triples
#endif
#ifndef VISRT_K7_MASKS
#define VISRT_K7_MASKS 1   // decide kernel: the section's crossing pairs from sign masks (same pairs, same order)
#endif
constexpr int kPreAx = 4;   // axes of t's polygon the screen tests (the first two non-degenerate edges)

// The (p, t) part of chain_triple_feasible, the same for every aim c of a
// prefix pair: the plane of t, p clipped to it, the plane frame and t's
// polygon in that frame. K7 forms it once per warp (shared memory) instead of
// once per lane. ok = false: infeasible for every aim (p clips to < 2 points
// or the frame degenerates), exactly where triple_feasible returns false.
template <int MAXV>
struct TriplePre {
    PlaneD pl;
    V3 u, v;
    V3 pa[Caps<MAXV>::kClip];
    double da[Caps<MAXV>::kClip];
    V2 mid2d[VISRT_MAX_VERTS];
    // the first kPreAx axes separating_axis(mid2d, ., sec, .) tests (edge normal,
    // edge direction of t's polygon) and t's own extents on them
    V2 axis[kPreAx];
    double amin[kPreAx], amax[kPreAx];
    unsigned apos, aneg, azero;   // signs of da[]: strictly in front / behind / on t's plane (bit i)
    int nl, nm, ok, nax;
};

template <int MAXV>
__device__ __noinline__ void triple_pre(const DevScene& s, int a, int b, TriplePre<MAXV>& P) {
    const double* N = s.normal + 3 * static_cast<size_t>(b);
    P.pl = PlaneD{face_pt(s, b, 0), {N[0], N[1], N[2]}};
    P.nl = clip_halfspace<MAXV>(s, a, P.pl, P.pa);
    P.ok = P.nl >= 2;
    // PlaneFrame::from_plane, src/geom.cpp:209-217
    const V3 axis = fabs(P.pl.n.x) < 0.9 ? V3{1, 0, 0} : V3{0, 1, 0};
    V3 u = v3cross(P.pl.n, axis);
    const double un = __dsqrt_rn(v3dot(u, u));
    if (un < kEps) {
        P.ok = 0;
        return;
    }
    u = {__ddiv_rn(u.x, un), __ddiv_rn(u.y, un), __ddiv_rn(u.z, un)};
    P.u = u;
    P.v = v3cross(P.pl.n, u);
    P.apos = P.aneg = P.azero = 0u;
    for (int i = 0; i < P.nl; ++i) {
        const double di = P.pl.sd(P.pa[i]);
        P.da[i] = di;
        if (fabs(di) <= kEps) P.azero |= 1u << i;
        else if (di > kEps) P.apos |= 1u << i;
        else if (di < -kEps) P.aneg |= 1u << i;
    }
    P.nm = s.nv[b];
    for (int k = 0; k < P.nm; ++k) {
        const V3 r = v3sub(face_pt(s, b, k), P.pl.p);
        P.mid2d[k] = V2{v3dot(r, P.u), v3dot(r, P.v)};
    }
    // separating_axis(mid2d, nm, ...)'s axes in its own order and arithmetic
    // (src/geom.cpp:257-270), with axis_separates' extents of mid2d
    P.nax = 0;
    for (int k = 0; k < kPreAx; ++k) P.axis[k] = V2{0.0, 0.0};
    for (int i = 0; i < P.nm && P.nax + 2 <= kPreAx; ++i) {
        const V2 e = v2sub(P.mid2d[(i + 1) % P.nm], P.mid2d[i]);
        const double len = v2norm(e);
        if (len <= 1e-12) continue;
        const V2 ax2[2] = {{__ddiv_rn(-e.y, len), __ddiv_rn(e.x, len)}, {__ddiv_rn(e.x, len), __ddiv_rn(e.y, len)}};
        for (int h = 0; h < 2; ++h) {
            double lo = 1e300, hi = -1e300;
            for (int k = 0; k < P.nm; ++k) {
                const double d = v2dot(P.mid2d[k], ax2[h]);
                lo = smin(lo, d);
                hi = smax(hi, d);
            }
            P.axis[P.nax] = ax2[h];
            P.amin[P.nax] = lo;
            P.amax[P.nax] = hi;
            ++P.nax;
        }
    }
}

// hull_plane_slice's section points (src/geom.cpp:292-307) in the reference's
// order, written to sec; returns their count.
template <int MAXV>
__device__ __forceinline__ int section_points(const TriplePre<MAXV>& P, const V3* pts, const double* d, int np,
                                              V2* sec) {
    const PlaneD& pl = P.pl;
    const V3 u = P.u, v = P.v;
    int ns = 0;
    auto to2d = [&](V3 p) {
        const V3 r = v3sub(p, pl.p);
        return V2{v3dot(r, u), v3dot(r, v)};
    };
#if VISRT_K7_MASKS
    // the same (i, j) pairs in the same order, found through sign masks instead
    // of np^2 comparisons: point i is on the plane (emitted first) or strictly on
    // one side, and then crosses with every later point strictly on the other
    unsigned pos = 0, neg = 0;
    for (int i = 0; i < np; ++i) {
        if (d[i] > kEps) pos |= 1u << i;
        else if (d[i] < -kEps) neg |= 1u << i;
    }
    for (int i = 0; i < np; ++i) {
        const unsigned bi = 1u << i;
        if (!((pos | neg) & bi)) {
            if (fabs(d[i]) <= kEps) sec[ns++] = to2d(pts[i]);
            continue;
        }
        const V3 pi = pts[i];
        const double di = d[i];
        for (unsigned m = ((pos & bi) ? neg : pos) & ~((bi << 1) - 1u); m; m &= m - 1) {
            const int j = __ffs(m) - 1;
            const double t = __ddiv_rn(di, dsub(di, d[j]));
            sec[ns++] = to2d(v3add(pi, v3mul(v3sub(pts[j], pi), t)));
        }
    }
#else
    for (int i = 0; i < np; ++i) {
        if (fabs(d[i]) <= kEps) sec[ns++] = to2d(pts[i]);
        for (int j = i + 1; j < np; ++j) {
            if ((d[i] > kEps && d[j] < -kEps) || (d[i] < -kEps && d[j] > kEps)) {
                const double t = __ddiv_rn(d[i], dsub(d[i], d[j]));
                sec[ns++] = to2d(v3add(pts[i], v3mul(v3sub(pts[j], pts[i]), t)));
            }
        }
    }
#endif
    return ns;
}

// The screen of K7's first kernel: is chain_triple_feasible(p, t, c) false because
// an axis of t's polygon separates it from the section? The same section points
// as section_points (each from the same operands in the same operation order; a
// crossing keeps the lower index as its base point), enumerated through sign
// masks instead of the np^2 pair loop and reduced to their extents on the prefix
// pair's axes — nothing is stored. A separating axis of t's polygon over ALL
// section points separates it from their hull too: the hull's vertices are a
// subset of the points (sort, tolerance-unique and the monotone chain only drop
// points), so its extent on an axis lies inside theirs and
// axis_separates(mid2d, ., hull, ., axis) holds a fortiori, i.e.
// convex_polygons_overlap_2d is false; an empty section is infeasible as well.
template <int MAXV>
__device__ __forceinline__ bool section_separated(const TriplePre<MAXV>& P, const V3* cp, const double* cd, int nt) {
    // point i < nl: the prefix pair's clipped polygon (shared memory, signs known);
    // point nl + k: the aim's clipped and mirrored point k (local)
    const PlaneD& pl = P.pl;
    const V3 u = P.u, v = P.v;
    const int nl = P.nl;
    unsigned pos = P.apos, neg = P.aneg, zero = P.azero;
    for (int k = 0; k < nt; ++k) {
        const double dk = cd[k];
        if (fabs(dk) <= kEps) zero |= 1u << (nl + k);
        else if (dk > kEps) pos |= 1u << (nl + k);
        else if (dk < -kEps) neg |= 1u << (nl + k);
    }
    if (zero == 0u && (pos == 0u || neg == 0u)) return true;   // empty section: infeasible
    auto pt = [&](int i) { return i < nl ? P.pa[i] : cp[i - nl]; };
    auto sd = [&](int i) { return i < nl ? P.da[i] : cd[i - nl]; };
    double emin[kPreAx], emax[kPreAx];
#pragma unroll
    for (int k = 0; k < kPreAx; ++k) {
        emin[k] = 1e300;
        emax[k] = -1e300;
    }
    auto ext = [&](V3 p) {
        const V3 r = v3sub(p, pl.p);
        const V2 q{v3dot(r, u), v3dot(r, v)};
#pragma unroll
        for (int k = 0; k < kPreAx; ++k) {
            const double e = v2dot(q, P.axis[k]);
            emin[k] = smin(emin[k], e);
            emax[k] = smax(emax[k], e);
        }
    };
    for (unsigned m = zero; m; m &= m - 1) ext(pt(__ffs(m) - 1));
    for (unsigned mi = pos | neg; mi; mi &= mi - 1) {
        const int i = __ffs(mi) - 1;
        const unsigned opp = (((pos >> i) & 1u) ? neg : pos) & ~((2u << i) - 1u);
        if (!opp) continue;
        const V3 pi = pt(i);
        const double di = sd(i);
        for (unsigned m = opp; m; m &= m - 1) {
            const int j = __ffs(m) - 1;
            const double t = __ddiv_rn(di, dsub(di, sd(j)));
            ext(v3add(pi, v3mul(v3sub(pt(j), pi), t)));
        }
    }
    bool sep = false;
#pragma unroll
    for (int k = 0; k < kPreAx; ++k)
        if (k < P.nax) sep |= P.amax[k] < dsub(emin[k], kEps) || emax[k] < dsub(P.amin[k], kEps);
    return sep;
}

// The aim's part of chain_triple_feasible's point set: c clipped to t's plane and
// mirrored through it, appended to the prefix pair's clipped polygon (pts, d of
// np points). Returns np, or 0 when c clips to < 2 points (infeasible).
template <int MAXV>
__device__ __forceinline__ int triple_points(const DevScene& s, const TriplePre<MAXV>& P, int c, V3* pts, double* d) {
    const PlaneD pl = P.pl;
    V3 tgt[Caps<MAXV>::kClip];
    const int nt = clip_halfspace<MAXV>(s, c, pl, tgt);
    if (nt < 2) return 0;
    const int nl = P.nl;
    for (int i = 0; i < nl; ++i) {
        pts[i] = P.pa[i];
        d[i] = P.da[i];
    }
    int np = nl;
    for (int i = 0; i < nt; ++i) {
        const double d2 = dmul(2.0, pl.sd(tgt[i]));   // mirror_point
        pts[np] = v3sub(tgt[i], v3mul(pl.n, d2));
        d[np] = pl.sd(pts[np]);
        ++np;
    }
    return np;
}

// triple_feasible(p, t, c) given TriplePre(p, t) with ok set: the same
// operations in the same order on the same values.
template <int MAXV>
__device__ __noinline__ bool triple_feasible_pre(const DevScene& s, const TriplePre<MAXV>& P, int c) {
    V3 pts[Caps<MAXV>::kPts];
    double d[Caps<MAXV>::kPts];
    K7S(0, 1);
    const int np = triple_points<MAXV>(s, P, c, pts, d);
    if (np == 0) return false;
    K7S(2, 1);
    V2 sec[Caps<MAXV>::kSec];
    int ns = section_points<MAXV>(P, pts, d, np, sec);
    V2 hull[2 * Caps<MAXV>::kSec];
    K7S(3, ns);
    ns = convex_hull(sec, ns, hull);
    if (ns == 0) return false;
    K7S(4, 1);
    K7S(7, ns);
    V2 mid2d[VISRT_MAX_VERTS];
    const int nm = P.nm;
    for (int k = 0; k < nm; ++k) mid2d[k] = P.mid2d[k];
    // convex_polygons_overlap_2d, src/geom.cpp:282-290
    if (separating_axis(sec, ns, mid2d, nm) || separating_axis(mid2d, nm, sec, ns)) return false;
    K7S(5, 1);
    if (!has_finite_edge(sec, ns) && !has_finite_edge(mid2d, nm)) return v2norm(v2sub(sec[0], mid2d[0])) <= kEps;
    return true;
}

// K7's screen for one aim: true = chain_triple_feasible(p, t, c) is certainly
// false (c clips away, or section_separated); false = undecided, kernel 2 runs
// the full predicate.
template <int MAXV>
__device__ __noinline__ bool triple_screened_out(const DevScene& s, const TriplePre<MAXV>& P, int c) {
    const PlaneD pl = P.pl;
    V3 cp[Caps<MAXV>::kClip];      // c clipped to t's plane, then mirrored through it in place
    double cd[Caps<MAXV>::kClip];
    const int nt = clip_halfspace<MAXV>(s, c, pl, cp);
    if (nt < 2) return true;
    for (int i = 0; i < nt; ++i) {   // the same operations as triple_points
        const double d2 = dmul(2.0, pl.sd(cp[i]));   // mirror_point
        cp[i] = v3sub(cp[i], v3mul(pl.n, d2));
        cd[i] = pl.sd(cp[i]);
    }
    return section_separated<MAXV>(P, cp, cd, nt);
}

// ---- interval sets, src/vismatrix.cpp:43-97 (<= 4 intervals here) ----
struct ISet {
    int n;
    double lo[4], hi[4];
};

__device__ void normalize_set(ISet& s) {
    // sort lexicographically (std::array<double,2> operator<)
    for (int i = 1; i < s.n; ++i) {
        const double a = s.lo[i], b = s.hi[i];
        int j = i - 1;
        while (j >= 0 && (a < s.lo[j] || (a == s.lo[j] && b < s.hi[j]))) {
            s.lo[j + 1] = s.lo[j];
            s.hi[j + 1] = s.hi[j];
            --j;
        }
        s.lo[j + 1] = a;
        s.hi[j + 1] = b;
    }
    int m = 0;
    for (int i = 0; i < s.n; ++i) {
        if (dsub(s.hi[i], s.lo[i]) < 0) continue;
        if (m > 0 && s.lo[i] <= dadd(s.hi[m - 1], 1e-15)) {
            s.hi[m - 1] = smax(s.hi[m - 1], s.hi[i]);
        } else {
            s.lo[m] = s.lo[i];
            s.hi[m] = s.hi[i];
            ++m;
        }
    }
    s.n = m;
}

__device__ void affine_halfline(double a, double b, bool leq, double lo, double hi, ISet& out) {
    out.n = 0;
    if (!leq) {
        a = -a;
        b = -b;
    }
    if (fabs(a) < 1e-300) {
        if (b <= 0) {
            out.n = 1;
            out.lo[0] = lo;
            out.hi[0] = hi;
        }
        return;
    }
    const double t = __ddiv_rn(-b, a);
    if (a > 0) {
        if (t < lo) return;
        out.n = 1;
        out.lo[0] = lo;
        out.hi[0] = smin(t, hi);
        return;
    }
    if (t > hi) return;
    out.n = 1;
    out.lo[0] = smax(t, lo);
    out.hi[0] = hi;
}

__device__ bool clip_param_to_upper(V2 p0, V2 p1, double& lo, double& hi) {
    lo = 0.0;
    hi = 1.0;
    const double y0 = p0.y, y1 = p1.y;
    const double dy = dsub(y1, y0);
    if (fabs(dy) < 1e-300) return y0 >= -kEps;
    const double tcross = __ddiv_rn(-y0, dy);
    if (dy > 0) lo = smax(0.0, tcross);
    else hi = smin(1.0, tcross);
    return dsub(hi, lo) > 1e-12;
}

// second_order_check verdict != None, src/vismatrix.cpp:387-455
__device__ __noinline__ bool second_order_reachable(const DevScene& s, int orig, int mid, int test, int pl) {
    const double* so = s.seg + (static_cast<size_t>(orig) * 3 + pl) * 6;
    const double* sm = s.seg + (static_cast<size_t>(mid) * 3 + pl) * 6;
    const double* st = s.seg + (static_cast<size_t>(test) * 3 + pl) * 6;
    // segment_frame, 114-128
    V2 origin{sm[0], sm[1]};
    const V2 dd{dsub(sm[2], sm[0]), dsub(sm[3], sm[1])};
    const double len = v2norm(dd);
    const double inv = __ddiv_rn(1.0, len);
    V2 ux{dmul(dd.x, inv), dmul(dd.y, inv)};
    const V2 uy{sm[4], sm[5]};
    if (v2cross(ux, uy) < 0) {
        origin = {sm[2], sm[3]};
        ux = {dmul(ux.x, -1.0), dmul(ux.y, -1.0)};
    }
    auto map = [&](double x, double y) {
        const V2 r{dsub(x, origin.x), dsub(y, origin.y)};
        return V2{v2dot(r, ux), v2dot(r, uy)};
    };
    const double length = v2norm(V2{dsub(sm[2], sm[0]), dsub(sm[3], sm[1])});
    V2 p0 = map(so[0], so[1]);
    V2 p1 = map(so[2], so[3]);
    {
        double lo, hi;
        if (!clip_param_to_upper(p0, p1, lo, hi)) return false;
        const V2 q0{dadd(p0.x, dmul(lo, dsub(p1.x, p0.x))), dadd(p0.y, dmul(lo, dsub(p1.y, p0.y)))};
        const V2 q1{dadd(p0.x, dmul(hi, dsub(p1.x, p0.x))), dadd(p0.y, dmul(hi, dsub(p1.y, p0.y)))};
        p0 = q0;
        p1 = q1;
    }
    const V2 c0 = map(st[0], st[1]);
    const V2 c1 = map(st[2], st[3]);
    double dlo, dhi;
    if (!clip_param_to_upper(c0, c1, dlo, dhi)) return false;
    const V2 m0{c0.x, -c0.y};
    const V2 md{dsub(c1.x, c0.x), -dsub(c1.y, c0.y)};
    auto condition = [&](V2 p, double bound, bool leq, ISet& out) {
        const double a_num = dsub(dmul(md.x, p.y), dmul(p.x, md.y));
        const double b_num = dsub(dmul(m0.x, p.y), dmul(p.x, m0.y));
        const double a_den = -md.y;
        const double b_den = dsub(p.y, m0.y);
        affine_halfline(dsub(a_num, dmul(bound, a_den)), dsub(b_num, dmul(bound, b_den)), leq, dlo, dhi, out);
    };
    ISet r0, r1, l0, l1;
    condition(p0, length, true, r0);
    condition(p1, length, true, r1);
    condition(p0, 0.0, false, l0);
    condition(p1, 0.0, false, l1);
    ISet right{0, {}, {}}, left{0, {}, {}};
    for (int i = 0; i < r0.n; ++i) { right.lo[right.n] = r0.lo[i]; right.hi[right.n++] = r0.hi[i]; }
    for (int i = 0; i < r1.n; ++i) { right.lo[right.n] = r1.lo[i]; right.hi[right.n++] = r1.hi[i]; }
    normalize_set(right);
    for (int i = 0; i < l0.n; ++i) { left.lo[left.n] = l0.lo[i]; left.hi[left.n++] = l0.hi[i]; }
    for (int i = 0; i < l1.n; ++i) { left.lo[left.n] = l1.lo[i]; left.hi[left.n++] = l1.hi[i]; }
    normalize_set(left);
    ISet reach{0, {}, {}};
    for (int i = 0; i < right.n; ++i)
        for (int j = 0; j < left.n; ++j) {
            const double lo = smax(right.lo[i], left.lo[j]);
            const double hi = smin(right.hi[i], left.hi[j]);
            if (lo <= hi) {
                reach.lo[reach.n] = lo;
                reach.hi[reach.n++] = hi;
            }
        }
    normalize_set(reach);
    double total = 0;
    for (int i = 0; i < reach.n; ++i) total = dadd(total, dsub(reach.hi[i], reach.lo[i]));
    return !(total <= 1e-12);
}

// required_planes bitmask (src/vismatrix.cpp:171-181) from the device plane segments
__device__ int req_planes(const DevScene& s, int i, int j) {
    int m = 0;
    for (int pl = 0; pl < 3; ++pl) {
        if (!s.seg_ok[3 * i + pl] || !s.seg_ok[3 * j + pl]) continue;
        const double* a = s.seg + (static_cast<size_t>(i) * 3 + pl) * 6;
        const double* b = s.seg + (static_cast<size_t>(j) * 3 + pl) * 6;
        const double d = fabs(dadd(dmul(a[4], b[4]), dmul(a[5], b[5])));
        if (d >= 1.0 - 1e-9 || d <= 1e-9) m |= 1 << pl;
    }
    return m;
}

struct ChainArgs {
    DevScene s;
    const int32_t* off1;
    const int32_t* idx1;
    const int32_t* pair_p;      // directed admitted pair (p, t) per rank
    const long long* word_off;  // first survivor word of each prefix pair (ceil(aims / 32) words each)
    uint32_t* surv;             // kernel 1 -> kernel 2: bit = the aim passed the screen
    long long npairs;
    int32_t* out;               // triples (p, t, a)
    unsigned long long* nout;
    long long cap;
    unsigned long long* cursor; // [0] kernel 1, [1] kernel 2
};

// K7 runs as two kernels over the same warp-per-prefix-pair walk (a warp takes a
// directed admitted pair (p, t), lanes take the admitted aims of t):
//   k_chain_screen  every candidate: clip + mirror + the section's extents on t's
//                   axes (triple_screened_out) — no section, hull or sort buffers,
//                   ~1.3k SASS instructions; leaves one survivor bit per aim;
//   k_chain_decide  survivors only (config 3: 20 % of the candidates), compacted so
//                   that every lane holds one: the full chain_triple_feasible and
//                   second_order_check, warp-compacted triples.
// One kernel doing both kept 95 KB of code live with warps in every phase (ncu:
// no_instruction the top stall, 6.1 warps per issue) and sized its local-memory
// frame (sec + hull: 6.5 KB per thread) for candidates that never reach the hull.
template <int MAXV>
__global__ void __launch_bounds__(128, 6) k_chain_screen(ChainArgs a) {
    const DevScene& s = a.s;
    const int lane = threadIdx.x & 31;
    __shared__ TriplePre<MAXV> pre_buf[4];   // per warp (128 threads)
    TriplePre<MAXV>& pre = pre_buf[threadIdx.x >> 5];
    for (;;) {
        unsigned long long r = 0;
        if (lane == 0) r = atomicAdd(a.cursor, 1ull);
        r = __shfl_sync(kAll, r, 0);
        if (static_cast<long long>(r) >= a.npairs) break;
        const int p = a.pair_p[r];
        const int t = a.idx1[r];
        const int lo = a.off1[t], hi = a.off1[t + 1];
        __syncwarp();
        if (lane == 0) triple_pre<MAXV>(s, p, t, pre);   // the prefix pair's part, once
        __syncwarp();
        if (!pre.ok) continue;                           // no aim of (p, t) is feasible (words stay 0)
        uint32_t* w = a.surv + a.word_off[r];
        for (int q0 = lo; q0 < hi; q0 += 32, ++w) {
            const int q = q0 + lane;
            const bool keep = q < hi && !(VISRT_K7_SCREEN && triple_screened_out<MAXV>(s, pre, a.idx1[q]));
            const unsigned m = __ballot_sync(kAll, keep);
            if (lane == 0) *w = m;
        }
    }
}

template <int MAXV>
__global__ void __launch_bounds__(128, VISRT_K7_MINB) k_chain_decide(ChainArgs a) {
    const DevScene& s = a.s;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    __shared__ TriplePre<MAXV> pre_buf[4];   // per warp (128 threads)
    __shared__ int queue_buf[4][64];         // per warp: survivor positions waiting for a full batch
    TriplePre<MAXV>& pre = pre_buf[threadIdx.x >> 5];
    int* queue = queue_buf[threadIdx.x >> 5];
    for (;;) {
        unsigned long long r = 0;
        if (lane == 0) r = atomicAdd(a.cursor + 1, 1ull);
        r = __shfl_sync(kAll, r, 0);
        if (static_cast<long long>(r) >= a.npairs) break;
        const int t = a.idx1[r];
        const int lo = a.off1[t], hi = a.off1[t + 1];
        const int nw = (hi - lo + 31) >> 5;
        const uint32_t* w = a.surv + a.word_off[r];
        bool any = false;
        for (int k = lane; k < nw; k += 32) any |= w[k] != 0u;
        if (!__any_sync(kAll, any)) continue;            // every aim screened out
        const int p = a.pair_p[r];
#if !VISRT_K7_SPLIT2
        const int rp_pt = req_planes(s, p, t);
#endif
        __syncwarp();
        if (lane == 0) triple_pre<MAXV>(s, p, t, pre);
        __syncwarp();
        int count = 0;                                   // queued survivors (warp-uniform)
        for (int k = 0; k < nw || count > 0; ++k) {
            if (k < nw) {
                const unsigned m = w[k];
                if ((m >> lane) & 1u) queue[count + __popc(m & lt)] = lo + 32 * k + lane;
                count += __popc(m);
                __syncwarp();
                if (count < 32 && k + 1 < nw) continue;  // wait for a full batch
            }
            // the first min(32, count) queued aims, one per lane
            const int take = min(count, 32);
            const int q = lane < take ? queue[lane] : -1;
            const int rest = lane < count - take ? queue[take + lane] : 0;
            __syncwarp();
            if (lane < count - take) queue[lane] = rest;
            count -= take;
            __syncwarp();
            bool ok = false;
            int c = -1;
            if (q >= 0) {
                c = a.idx1[q];
                ok = triple_feasible_pre<MAXV>(s, pre, c);
#if !VISRT_K7_SPLIT2
                if (ok) {
                    const int planes = req_planes(s, t, c) & rp_pt;
                    for (int pl = 0; pl < 3 && ok; ++pl)
                        if (planes >> pl & 1) ok = second_order_reachable(s, p, t, c, pl);
                }
#endif
            }
            const unsigned m = __ballot_sync(kAll, ok);
            if (!m) continue;
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(a.nout, static_cast<unsigned long long>(__popc(m)));
            base = __shfl_sync(kAll, base, 0);
            if (ok) {
                const long long slot = static_cast<long long>(base) + __popc(m & lt);
                if (slot < a.cap) {
                    a.out[3 * slot] = p;
                    a.out[3 * slot + 1] = t;
                    a.out[3 * slot + 2] = c;
                }
            }
        }
    }
}

// K7's third kernel (VISRT_K7_SPLIT2): second_order_check in every working plane the
// prefix pair and the aim pair share, thread per chain_triple_feasible triple — its
// 1.3k instructions of interval arithmetic stay out of the decide kernel's footprint.
__global__ void __launch_bounds__(256) k_chain_second(DevScene s, const int32_t* in, long long n, int32_t* out,
                                                      unsigned long long* nout, long long cap) {
    const int lane = threadIdx.x & 31;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long k0 = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) - lane; k0 < n; k0 += stride) {
        const long long k = k0 + lane;
        bool ok = k < n;
        int p = 0, t = 0, c = 0;
        if (ok) {
            p = in[3 * k];
            t = in[3 * k + 1];
            c = in[3 * k + 2];
            const int planes = req_planes(s, t, c) & req_planes(s, p, t);
            for (int pl = 0; pl < 3 && ok; ++pl)
                if (planes >> pl & 1) ok = second_order_reachable(s, p, t, c, pl);
        }
        const unsigned m = __ballot_sync(kAll, ok);
        if (!m) continue;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(nout, static_cast<unsigned long long>(__popc(m)));
        base = __shfl_sync(kAll, base, 0);
        if (ok) {
            const long long slot = static_cast<long long>(base) + __popc(m & ((1u << lane) - 1u));
            if (slot < cap) {
                out[3 * slot] = p;
                out[3 * slot + 1] = t;
                out[3 * slot + 2] = c;
            }
        }
    }
}

// chain_triple_feasible for an explicit triple list (the public predicate,
// include/rt/vismatrix.hpp:131), thread per triple.
template <int MAXV>
__global__ void k_triples_feasible(DevScene s, long long n, const int32_t* t, uint8_t* out) {
    for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<long long>(gridDim.x) * blockDim.x)
        out[k] = triple_feasible<MAXV>(s, t[3 * k], t[3 * k + 1], t[3 * k + 2]) ? 1 : 0;
}

__global__ void k_popc_words(const uint32_t* w, long long n, unsigned long long* total) {
    unsigned long long c = 0;
    for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<long long>(gridDim.x) * blockDim.x)
        c += __popc(w[k]);
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(kAll, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(total, c);
}

__global__ void k_pack_triples(const int32_t* t, long long m, unsigned long long* key) {
    for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < m;
         k += static_cast<long long>(gridDim.x) * blockDim.x)
        key[k] = (static_cast<unsigned long long>(t[3 * k]) << 42) |
                 (static_cast<unsigned long long>(t[3 * k + 1]) << 21) | static_cast<unsigned long long>(t[3 * k + 2]);
}

__global__ void k_unpack_triples(const unsigned long long* key, long long m, int32_t* t) {
    for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < m;
         k += static_cast<long long>(gridDim.x) * blockDim.x) {
        const unsigned long long v = key[k];
        t[3 * k] = static_cast<int32_t>(v >> 42);
        t[3 * k + 1] = static_cast<int32_t>((v >> 21) & 0x1FFFFFull);
        t[3 * k + 2] = static_cast<int32_t>(v & 0x1FFFFFull);
    }
}

}  // namespace
}  // namespace visrt

using visrt::ck;

#ifdef VISRT_K7_STATS
extern "C" int visrt_debug_k7_stats(unsigned long long* out) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, visrt::g_k7_stats, sizeof(visrt::g_k7_stats));
    static const unsigned long long zero[8] = {};
    return static_cast<int>(cudaMemcpyToSymbol(visrt::g_k7_stats, zero, sizeof(zero)));
}
#endif

// Order-2 chains of build_matrix(scene, 2) as (p, t, a) triples, from the
// admitted matrix (NULL: the scene's device bits of the last PREFILTERED call).
// out == NULL: count only (result cached for the next call).
extern "C" int visrt_chain_triples(visrt_scene* sc, const uint64_t* admitted_bits, int32_t* out, int64_t cap,
                                   int64_t* ntriples, visrt_stats* stats, void* stream) {
    return visrt::capi_guard([&] {
        visrt::ScopedDevice dev(sc);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const visrt::HostScene& hs = visrt::scene_host(sc);
        const visrt::DevScene& ds = visrt::scene_dev(sc);
        const int n = hs.n, words = (n + 63) / 64;
        std::vector<uint64_t> bits(static_cast<size_t>(n) * words);
        if (admitted_bits) std::memcpy(bits.data(), admitted_bits, bits.size() * 8);
        else ck(cudaMemcpy(bits.data(), visrt_matrix_bits_device(sc), bits.size() * 8, cudaMemcpyDeviceToHost), "D2H");
        if (n >= (1 << 21)) throw visrt::UsageError("chain triples pack face indices in 21 bits");
        uint64_t key = 1469598103934665603ull;
        {
            const unsigned char* b = reinterpret_cast<const unsigned char*>(bits.data());
            for (size_t k = 0; k < bits.size() * 8; ++k) {
                key ^= b[k];
                key *= 1099511628211ull;
            }
        }
        visrt::ChainCache& cache = visrt::scene_chain_cache(sc);
        if (cache.valid && cache.key == key) {
            const int64_t nc = static_cast<int64_t>(cache.tri.size() / 3);
            *ntriples = nc;
            if (out) {
                if (nc > cap) throw visrt::UsageError("triple capacity too small");
                std::copy(cache.tri.begin(), cache.tri.end(), out);
            }
            if (stats) {
                *stats = visrt_stats{};
                stats->pairs = cache.pairs;
                stats->candidates = cache.candidates;
                stats->admitted = nc;
                stats->tests_alg = static_cast<double>(cache.candidates);
                stats->tests_exec = cache.candidates;
                stats->ms = cache.ms;
            }
            return;
        }
        std::vector<int32_t> off1(n + 1, 0), idx1, pp;
        for (int p = 0; p < n; ++p) {
            for (int w = 0; w < words; ++w) {
                uint64_t m = bits[static_cast<size_t>(p) * words + w];
                while (m) {
                    const int b = __builtin_ctzll(m);
                    m &= m - 1;
                    idx1.push_back(w * 64 + b);
                    pp.push_back(p);
                }
            }
            off1[p + 1] = static_cast<int32_t>(idx1.size());
        }
        long long total = 0, words32 = 0;
        std::vector<long long> word_off(idx1.size() + 1, 0);
        for (size_t r = 0; r < idx1.size(); ++r) {
            const long long aims = off1[idx1[r] + 1] - off1[idx1[r]];
            total += aims;
            word_off[r] = words32;
            words32 += (aims + 31) / 32;
        }
        word_off[idx1.size()] = words32;
        std::vector<void*> tmp;
        visrt::FreeGuard guard{tmp};
        auto up = [&](const std::vector<int32_t>& v) {
            int32_t* d = visrt::dalloc<int32_t>(std::max<size_t>(v.size(), 1), tmp);
            if (!v.empty()) ck(cudaMemcpy(d, v.data(), v.size() * 4, cudaMemcpyHostToDevice), "H2D");
            return d;
        };
        visrt::ChainArgs a{};
        a.s = ds;
        a.off1 = up(off1);
        a.idx1 = up(idx1);
        a.pair_p = up(pp);
        a.npairs = static_cast<long long>(idx1.size());
        {
            long long* d_wo = visrt::dalloc<long long>(word_off.size(), tmp);
            ck(cudaMemcpy(d_wo, word_off.data(), word_off.size() * 8, cudaMemcpyHostToDevice), "H2D");
            a.word_off = d_wo;
        }
        a.surv = visrt::dalloc<uint32_t>(static_cast<size_t>(std::max<long long>(words32, 1)), tmp);
        ck(cudaMemsetAsync(a.surv, 0, static_cast<size_t>(std::max<long long>(words32, 1)) * 4, st), "memset");
        unsigned long long* ctr = visrt::dalloc<unsigned long long>(4, tmp);
        a.nout = ctr;
        a.cursor = ctr + 1;
        ck(cudaMemsetAsync(ctr, 0, 32, st), "memset");
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
        int sms = 0, per = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, visrt::scene_device(sc));
        unsigned long long* d_surv_count = ctr + 3;
        auto run2 = [&](auto screen, auto decide) {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, screen, 128, 0);
            screen<<<sms * std::max(per, 1), 128, 0, st>>>(a);
            ck(cudaGetLastError(), "k_chain_screen");
            // survivors bound the triples: count them, then size the output
            const long long nw = std::max<long long>(words32, 1);
            visrt::k_popc_words<<<std::min<long long>((nw + 255) / 256, 148 * 8), 256, 0, st>>>(a.surv, nw, d_surv_count);
            unsigned long long nsurv = 0;
            ck(cudaMemcpyAsync(&nsurv, d_surv_count, 8, cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaStreamSynchronize(st), "sync");
            a.cap = std::max<long long>(static_cast<long long>(nsurv), 1);
            a.out = visrt::dalloc<int32_t>(static_cast<size_t>(a.cap) * 3, tmp);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, decide, 128, 0);
            decide<<<sms * std::max(per, 1), 128, 0, st>>>(a);
            ck(cudaGetLastError(), "k_chain_decide");
#if VISRT_K7_SPLIT2
            // the hull-feasible triples through second_order_check, compacted into a second buffer
            unsigned long long n1 = 0;
            ck(cudaMemcpyAsync(&n1, a.nout, 8, cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaStreamSynchronize(st), "sync");
            if (n1) {
                int32_t* out2 = visrt::dalloc<int32_t>(static_cast<size_t>(n1) * 3, tmp);
                ck(cudaMemsetAsync(a.nout, 0, 8, st), "memset");
                const long long m1 = static_cast<long long>(n1);
                visrt::k_chain_second<<<static_cast<int>(std::min<long long>((m1 + 255) / 256, 148 * 8)), 256, 0, st>>>(
                    a.s, a.out, m1, out2, a.nout, m1);
                ck(cudaGetLastError(), "k_chain_second");
                a.out = out2;
            }
#endif
        };
        if (a.npairs > 0) {
            if (ds.maxv <= 4) run2(visrt::k_chain_screen<4>, visrt::k_chain_decide<4>);
            else run2(visrt::k_chain_screen<8>, visrt::k_chain_decide<8>);
        }
        cudaEventRecord(e1, st);
        unsigned long long nout = 0;
        ck(cudaMemcpyAsync(&nout, ctr, 8, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "sync");
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *ntriples = static_cast<int64_t>(nout);
        // deterministic order (p, t, a): radix sort of packed 63-bit keys on the GPU
        std::vector<int32_t> h(static_cast<size_t>(nout) * 3);
        if (nout) {
            const long long m = static_cast<long long>(nout);
            unsigned long long* k0 = visrt::dalloc<unsigned long long>(m, tmp);
            unsigned long long* k1 = visrt::dalloc<unsigned long long>(m, tmp);
            const int blocks = static_cast<int>(std::min<long long>((m + 255) / 256, 148 * 16));
            visrt::k_pack_triples<<<blocks, 256, 0, st>>>(a.out, m, k0);
            size_t tb = 0;
            cub::DeviceRadixSort::SortKeys(nullptr, tb, k0, k1, m, 0, 63, st);
            void* d_tb = visrt::dalloc<char>(tb, tmp);
            ck(cub::DeviceRadixSort::SortKeys(d_tb, tb, k0, k1, m, 0, 63, st), "sort");
            visrt::k_unpack_triples<<<blocks, 256, 0, st>>>(k1, m, a.out);
            ck(cudaGetLastError(), "unpack");
            ck(cudaMemcpyAsync(h.data(), a.out, h.size() * 4, cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaStreamSynchronize(st), "sync");
        }
        if (out) {
            if (static_cast<int64_t>(nout) > cap) throw visrt::UsageError("triple capacity too small");
            std::copy(h.begin(), h.end(), out);
        }
        cache.valid = true;
        cache.key = key;
        cache.tri = std::move(h);
        cache.pairs = static_cast<int64_t>(idx1.size());
        cache.candidates = total;
        cache.ms = ms;
        if (stats) {
            stats->pairs = static_cast<int64_t>(idx1.size());
            stats->candidates = total;
            stats->admitted = static_cast<int64_t>(nout);
            stats->tests_alg = static_cast<double>(total);
            stats->tests_exec = total;
            stats->ms = ms;
        }
    });
}

extern "C" int visrt_triples_feasible(visrt_scene* sc, int64_t n, const int32_t* triples, uint8_t* feasible,
                                      void* stream) {
    return visrt::capi_guard([&] {
        visrt::ScopedDevice dev(sc);
        const visrt::DevScene& ds = visrt::scene_dev(sc);
        for (int64_t k = 0; k < 3 * n; ++k)
            if (triples[k] < 0 || triples[k] >= ds.n) throw visrt::UsageError("bad face index");
        if (n <= 0) return;
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        std::vector<void*> tmp;
        visrt::FreeGuard guard{tmp};
        int32_t* d_t = visrt::dalloc<int32_t>(3 * n, tmp);
        uint8_t* d_o = visrt::dalloc<uint8_t>(n, tmp);
        ck(cudaMemcpyAsync(d_t, triples, 12 * n, cudaMemcpyHostToDevice, st), "H2D");
        const int blocks = static_cast<int>(std::min<long long>((n + 127) / 128, 148 * 8));
        if (ds.maxv <= 4) visrt::k_triples_feasible<4><<<blocks, 128, 0, st>>>(ds, n, d_t, d_o);
        else visrt::k_triples_feasible<8><<<blocks, 128, 0, st>>>(ds, n, d_t, d_o);
        ck(cudaGetLastError(), "k_triples_feasible");
        ck(cudaMemcpyAsync(feasible, d_o, n, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "sync");
    });
}
