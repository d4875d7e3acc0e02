// Host facet ingest (K0): per-face products computed ONCE with the reference's
// exact FP64 operation order, then uploaded as the device SoA/AoS records.
// Compiled with -ffp-contract=off (no FMA), like the reference build.
//
//   Newell normal + normalized       src/geom.cpp:126-140, 15-19
//   orientation                      src/scene.cpp:19-24
//   plane_segment (XY/YZ/XZ)         src/scene.cpp:213-254
//   contains() per-edge inward       src/geom.cpp:155-167
//   face_samples / centroid          src/vismatrix.cpp:226-249, src/geom.cpp:142-146
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <stdexcept>

#include "visrt_internal.h"

namespace visrt {
namespace {

struct V3 {
    double x, y, z;
};
struct V2 {
    double x, y;
};
inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 mul(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline V3 dvd(V3 a, double s) { return {a.x / s, a.y / s, a.z / s}; }
inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
inline double norm(V3 a) { return std::sqrt(dot(a, a)); }
inline double dot2(V2 a, V2 b) { return a.x * b.x + a.y * b.y; }
inline double cross2(V2 a, V2 b) { return a.x * b.y - a.y * b.x; }
inline double norm2(V2 a) { return std::sqrt(dot2(a, a)); }
inline double smin(double a, double b) { return (b < a) ? b : a; }
inline double smax(double a, double b) { return (a < b) ? b : a; }
inline V2 project(V3 p, int plane) {
    if (plane == 0) return {p.x, p.y};
    if (plane == 1) return {p.y, p.z};
    return {p.x, p.z};
}

// plane_segment, src/scene.cpp:213-254
bool plane_segment(const V3* pts, int nv, V3 normal, int plane, double* out6) {
    V2 p2[VISRT_MAX_VERTS];
    for (int i = 0; i < nv; ++i) p2[i] = project(pts[i], plane);
    V2 lo = p2[0], hi = p2[0];
    for (int i = 0; i < nv; ++i) {
        lo = {smin(lo.x, p2[i].x), smin(lo.y, p2[i].y)};
        hi = {smax(hi.x, p2[i].x), smax(hi.y, p2[i].y)};
    }
    V2 a, b;
    if (hi.x - lo.x <= kEps && hi.y - lo.y <= kEps) {
        return false;
    } else if (hi.x - lo.x <= kEps) {
        a = {lo.x, lo.y};
        b = {lo.x, hi.y};
    } else if (hi.y - lo.y <= kEps) {
        a = {lo.x, lo.y};
        b = {hi.x, lo.y};
    } else {
        const V2 d = {hi.x - lo.x, hi.y - lo.y};
        double tmin = DBL_MAX, tmax = -DBL_MAX;
        V2 pmin{0, 0}, pmax{0, 0};
        for (int i = 0; i < nv; ++i) {
            const V2 rel = {p2[i].x - lo.x, p2[i].y - lo.y};
            if (std::abs(cross2(d, rel)) > kEps * (norm2(d) + 1.0)) return false;
            const double t = dot2(d, rel);
            if (t < tmin) { tmin = t; pmin = p2[i]; }
            if (t > tmax) { tmax = t; pmax = p2[i]; }
        }
        a = pmin;
        b = pmax;
    }
    const V2 n2 = project(normal, plane);
    const double len = norm2(n2);
    if (len <= kEps) return false;
    const double inv = 1.0 / len;
    out6[0] = a.x; out6[1] = a.y; out6[2] = b.x; out6[3] = b.y;
    out6[4] = n2.x * inv; out6[5] = n2.y * inv;
    return true;
}

template <int MAXV>
void write_record(const V3* pts, int nv, V3 n, double* rec) {
    for (int k = 0; k < RecLayout<MAXV>::kStride; ++k) rec[k] = 0.0;
    rec[0] = pts[0].x; rec[1] = pts[0].y; rec[2] = pts[0].z;
    rec[3] = n.x; rec[4] = n.y; rec[5] = n.z;
    for (int k = 0; k < MAXV; ++k) {
        V3 inward{0.0, 0.0, 0.0};
        V3 a = pts[0];
        if (k < nv) {
            a = pts[k];
            const V3 b = pts[(k + 1) % nv];
            const V3 edge = sub(b, a);
            const double len = norm(edge);
            if (!(len < kEps)) inward = dvd(cross(n, edge), len);
        }
        double* slot = k == 0 ? rec + 6 : rec + 9 + (k - 1) * 6;
        if (k == 0) {
            slot[0] = inward.x; slot[1] = inward.y; slot[2] = inward.z;
        } else {
            slot[0] = a.x; slot[1] = a.y; slot[2] = a.z;
            slot[3] = inward.x; slot[4] = inward.y; slot[5] = inward.z;
        }
    }
}

}  // namespace

void ingest(const visrt_facets_v1& f, HostScene& hs) {
    if (f.nfaces <= 0) throw std::runtime_error("scene has no faces");
    const int n = f.nfaces;
    hs.n = n;
    hs.maxv = 0;
    hs.nv.assign(n, 0);
    hs.ns.assign(n, 0);
    hs.pts.assign(static_cast<size_t>(n) * VISRT_MAX_VERTS * 3, 0.0);
    hs.normal.assign(static_cast<size_t>(n) * 3, 0.0);
    hs.orient.assign(n, 0);
    hs.seg.assign(static_cast<size_t>(n) * 18, 0.0);
    hs.seg_ok.assign(static_cast<size_t>(n) * 3, 0);
    hs.samples.assign(static_cast<size_t>(n) * kMaxSamples * 3, 0.0);
    hs.aabb.assign(static_cast<size_t>(n) * 6, 0.0);
    hs.building.assign(n, -1);
    for (int i = 0; i < n; ++i) {
        const int nv = f.vert_off[i + 1] - f.vert_off[i];
        if (nv < 3) throw std::runtime_error("face " + std::to_string(i) + " has fewer than 3 vertices");
        if (nv > VISRT_MAX_VERTS)
            throw std::runtime_error("face " + std::to_string(i) + " has more than " +
                                     std::to_string(VISRT_MAX_VERTS) + " vertices");
        hs.nv[i] = nv;
        if (nv > hs.maxv) hs.maxv = nv;
        if (f.building) hs.building[i] = f.building[i];
        V3 pts[VISRT_MAX_VERTS];
        for (int k = 0; k < nv; ++k) {
            const double* p = f.verts + 3 * static_cast<size_t>(f.vert_off[i] + k);
            pts[k] = {p[0], p[1], p[2]};
            double* dst = &hs.pts[(static_cast<size_t>(i) * VISRT_MAX_VERTS + k) * 3];
            dst[0] = p[0]; dst[1] = p[1]; dst[2] = p[2];
        }
        // Newell, src/geom.cpp:126-140
        V3 nn{0, 0, 0};
        for (int k = 0; k < nv; ++k) {
            const V3 a = pts[k], b = pts[(k + 1) % nv];
            nn.x += (a.y - b.y) * (a.z + b.z);
            nn.y += (a.z - b.z) * (a.x + b.x);
            nn.z += (a.x - b.x) * (a.y + b.y);
        }
        const double len = norm(nn);
        if (len < kEps) throw std::runtime_error("face " + std::to_string(i) + ": cannot normalize zero-length vector");
        const V3 nrm = dvd(nn, len);
        hs.normal[3 * i] = nrm.x; hs.normal[3 * i + 1] = nrm.y; hs.normal[3 * i + 2] = nrm.z;
        // classify_orientation, src/scene.cpp:19-24
        {
            const double ax = std::abs(nrm.x), ay = std::abs(nrm.y), az = std::abs(nrm.z);
            hs.orient[i] = (ax <= 1e-9 && ay <= 1e-9) ? 0 : (az <= 1e-9 ? 1 : 2);
        }
        for (int pl = 0; pl < 3; ++pl)
            hs.seg_ok[3 * i + pl] = plane_segment(pts, nv, nrm, pl, &hs.seg[(static_cast<size_t>(i) * 3 + pl) * 6]) ? 1 : 0;
        // face_samples, src/vismatrix.cpp:226-249
        double* smp = &hs.samples[static_cast<size_t>(i) * kMaxSamples * 3];
        int c = 0;
        auto put = [&](V3 p) { smp[3 * c] = p.x; smp[3 * c + 1] = p.y; smp[3 * c + 2] = p.z; ++c; };
        for (int k = 0; k < nv; ++k) put(pts[k]);
        V3 cen{0, 0, 0};
        for (int k = 0; k < nv; ++k) cen = add(cen, pts[k]);
        cen = dvd(cen, static_cast<double>(nv));
        put(cen);
        if (nv == 4) {
            for (int a = 0; a < 4; ++a) {
                for (int b = 0; b < 4; ++b) {
                    const double u = (a + 0.5) / 4.0;
                    const double v = (b + 0.5) / 4.0;
                    put(add(add(add(mul(pts[0], (1 - u) * (1 - v)), mul(pts[1], u * (1 - v))),
                                mul(pts[2], u * v)),
                            mul(pts[3], (1 - u) * v)));
                }
            }
        } else {
            const double ss[3] = {0.25, 0.5, 0.75};
            for (int k = 0; k < nv; ++k)
                for (double s : ss) put(add(cen, mul(sub(pts[k], cen), s)));
        }
        hs.ns[i] = c;
        // AABB
        V3 lo = pts[0], hi = pts[0];
        for (int k = 0; k < nv; ++k) {
            lo = {smin(lo.x, pts[k].x), smin(lo.y, pts[k].y), smin(lo.z, pts[k].z)};
            hi = {smax(hi.x, pts[k].x), smax(hi.y, pts[k].y), smax(hi.z, pts[k].z)};
        }
        double* bb = &hs.aabb[static_cast<size_t>(i) * 6];
        bb[0] = lo.x; bb[1] = lo.y; bb[2] = lo.z; bb[3] = hi.x; bb[4] = hi.y; bb[5] = hi.z;
    }
    // fp32 culling boxes relative to the scene centre.
    {
        double lo[3] = {hs.aabb[0], hs.aabb[1], hs.aabb[2]};
        double hi[3] = {hs.aabb[3], hs.aabb[4], hs.aabb[5]};
        for (int i = 0; i < n; ++i)
            for (int d = 0; d < 3; ++d) {
                lo[d] = smin(lo[d], hs.aabb[6 * i + d]);
                hi[d] = smax(hi[d], hs.aabb[6 * i + 3 + d]);
            }
        hs.extent = 0;
        for (int d = 0; d < 3; ++d) {
            hs.origin[d] = std::floor(0.5 * (lo[d] + hi[d]));
            hs.extent = smax(hs.extent, smax(std::abs(hi[d] - hs.origin[d]), std::abs(lo[d] - hs.origin[d])));
        }
        hs.box.assign(static_cast<size_t>(n) * 8, 0.0f);
        for (int i = 0; i < n; ++i) {
            // eps-miter of the face: 1e-9 / sin(theta/2) at its sharpest vertex
            double miter = 1e-9;
            const int nv = hs.nv[i];
            for (int k = 0; k < nv; ++k) {
                const double* p0 = &hs.pts[(static_cast<size_t>(i) * VISRT_MAX_VERTS + (k + nv - 1) % nv) * 3];
                const double* p1 = &hs.pts[(static_cast<size_t>(i) * VISRT_MAX_VERTS + k) * 3];
                const double* p2 = &hs.pts[(static_cast<size_t>(i) * VISRT_MAX_VERTS + (k + 1) % nv) * 3];
                const V3 u = sub({p0[0], p0[1], p0[2]}, {p1[0], p1[1], p1[2]});
                const V3 v = sub({p2[0], p2[1], p2[2]}, {p1[0], p1[1], p1[2]});
                const double nu = norm(u), nvv = norm(v);
                if (nu < kEps || nvv < kEps) { miter = 1.0; continue; }   // degenerate edge: be generous
                const double c = std::max(-1.0, std::min(1.0, dot(u, v) / (nu * nvv)));
                // sin(theta / 2) = sqrt((1 - cos theta) / 2), trig-free; the 1 %
                // slack covers its rounding (a conservative margin only)
                const double s = std::sqrt(0.5 * (1.0 - c));
                miter = std::max(miter, s > 1e-12 ? 2.02e-9 / s : 1.0);
            }
            const double m = box_margin(hs.extent, miter);
            const double* bb = &hs.aabb[static_cast<size_t>(i) * 6];
            float* o = &hs.box[static_cast<size_t>(i) * 8];
            for (int d = 0; d < 3; ++d) {
                o[d] = static_cast<float>(0.5 * (bb[d] + bb[3 + d]) - hs.origin[d]);
                o[4 + d] = static_cast<float>(0.5 * (bb[3 + d] - bb[d]) + m);
            }
        }
    }
    // Occluder records in the narrowest layout that fits.
    if (hs.maxv <= 4) {
        hs.rec4.assign(static_cast<size_t>(n) * RecLayout<4>::kStride, 0.0);
        for (int i = 0; i < n; ++i) {
            V3 pts[VISRT_MAX_VERTS];
            for (int k = 0; k < hs.nv[i]; ++k) {
                const double* p = &hs.pts[(static_cast<size_t>(i) * VISRT_MAX_VERTS + k) * 3];
                pts[k] = {p[0], p[1], p[2]};
            }
            write_record<4>(pts, hs.nv[i], {hs.normal[3 * i], hs.normal[3 * i + 1], hs.normal[3 * i + 2]},
                            &hs.rec4[static_cast<size_t>(i) * RecLayout<4>::kStride]);
        }
    }
    if (hs.maxv > 4) hs.rec8.assign(static_cast<size_t>(n) * RecLayout<8>::kStride, 0.0);
    for (int i = 0; i < n && hs.maxv > 4; ++i) {
        V3 pts[VISRT_MAX_VERTS];
        for (int k = 0; k < hs.nv[i]; ++k) {
            const double* p = &hs.pts[(static_cast<size_t>(i) * VISRT_MAX_VERTS + k) * 3];
            pts[k] = {p[0], p[1], p[2]};
        }
        write_record<8>(pts, hs.nv[i], {hs.normal[3 * i], hs.normal[3 * i + 1], hs.normal[3 * i + 2]},
                        &hs.rec8[static_cast<size_t>(i) * RecLayout<8>::kStride]);
    }
    build_hierarchy(hs);
}

// Two-level culling hierarchy (sweep.h): Morton order of the xy AABB centres
// (16 bits per axis over the scene extent, ties by face index), tiles of 64
// consecutive faces, tile box = union of the member boxes rounded outward.
// Only the ORDER in which occluders are examined changes; every verdict is
// still the exact predicate's.
void quantise_members(HostScene& hs);

void build_hierarchy(HostScene& hs) {
    const int n = hs.n;
    const double ext = std::max(hs.extent, 1.0);
    auto spread = [](uint32_t v) {
        uint64_t x = v & 0xffffu;
        x = (x | (x << 8)) & 0x00ff00ffu;
        x = (x | (x << 4)) & 0x0f0f0f0fu;
        x = (x | (x << 2)) & 0x33333333u;
        x = (x | (x << 1)) & 0x55555555u;
        return x;
    };
    std::vector<std::pair<uint64_t, int32_t>> key(n);
    for (int i = 0; i < n; ++i) {
        const double* bb = &hs.aabb[static_cast<size_t>(i) * 6];
        const double cx = 0.5 * (bb[0] + bb[3]) - hs.origin[0];
        const double cy = 0.5 * (bb[1] + bb[4]) - hs.origin[1];
        const auto q = [&](double c) {
            const double u = (c + ext) / (2.0 * ext);
            return static_cast<uint32_t>(std::min(65535.0, std::max(0.0, u * 65535.0)));
        };
        key[i] = {spread(q(cx)) | (spread(q(cy)) << 1), i};
    }
    std::sort(key.begin(), key.end());
    hs.perm.resize(n);
    hs.inv.resize(n);
    for (int k = 0; k < n; ++k) {
        hs.perm[k] = key[k].second;
        hs.inv[key[k].second] = k;
    }
    const bool narrow = hs.maxv <= 4;
    const int stride = narrow ? RecLayout<4>::kStride : RecLayout<8>::kStride;
    const std::vector<double>& rec = narrow ? hs.rec4 : hs.rec8;
    hs.srec.resize(static_cast<size_t>(n) * stride);
    hs.sbox.resize(static_cast<size_t>(n) * 8);
    for (int k = 0; k < n; ++k) {
        const int f = hs.perm[k];
        std::copy_n(&rec[static_cast<size_t>(f) * stride], stride, &hs.srec[static_cast<size_t>(k) * stride]);
        std::copy_n(&hs.box[static_cast<size_t>(f) * 8], 8, &hs.sbox[static_cast<size_t>(k) * 8]);
    }
    hs.ntiles = (n + 63) / 64;
    hs.nchunks = (hs.ntiles + 63) / 64;
    hs.ngroups = (n + kGroup - 1) / kGroup;
    // union boxes of `size` consecutive member boxes (tiles of 64, groups of 16)
    auto unions = [&](int size, int count, std::vector<float>& out) {
        out.assign(static_cast<size_t>(count) * 8, 0.0f);
        for (int t = 0; t < count; ++t) {
            double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
            for (int k = t * size; k < std::min(n, t * size + size); ++k) {
                const float* b = &hs.sbox[static_cast<size_t>(k) * 8];
                for (int d = 0; d < 3; ++d) {
                    lo[d] = std::min(lo[d], static_cast<double>(b[d]) - static_cast<double>(b[4 + d]));
                    hi[d] = std::max(hi[d], static_cast<double>(b[d]) + static_cast<double>(b[4 + d]));
                }
            }
            float* o = &out[static_cast<size_t>(t) * 8];
            for (int d = 0; d < 3; ++d) {
                // a member box lies inside [lo, hi]; the fp32 centre/half of the
                // union are padded by a few ulps of the extent so it still does
                o[d] = static_cast<float>(0.5 * (lo[d] + hi[d]));
                o[4 + d] = static_cast<float>(0.5 * (hi[d] - lo[d]) + 1e-4 + 8.0 * ext * 1.1920928955078125e-7);
            }
        }
    };
    unions(64, hs.ntiles, hs.tbox);
    unions(kGroup, hs.ngroups, hs.gbox);
    unions(64 * 64, hs.nchunks, hs.cbox);
    quantise_members(hs);
}

// 8-bit member boxes in their tile's frame (sweep.h qsat). Frame of tile t:
// step s_d = max(size_d / 251, extent * 2^-14) and origin o_d = lo_d - 2 s_d,
// so every member box maps into [2, 253]; it is stored rounded outward plus
// ONE more step on each side. That step absorbs the device's fp32 transform
// of the segment into the frame and the SAT's rounding there: with
// |coordinates| <= 2 extent / s_min + 510 = 2^15 + 510 frame units the fp32
// products err by < 2^-8 units, far inside the extra step. The float boxes
// quantised here already carry box_margin(), so the culling stays one-sided:
// the quantised box contains the float box contains every true hit.
void quantise_members(HostScene& hs) {
    const int n = hs.n;
    const double ext = std::max(hs.extent, 1.0);
    const double smin = ext * 6.103515625e-05;   // 2^-14
    hs.tframe.assign(static_cast<size_t>(hs.ntiles) * 8, 0.0f);
    hs.qbox.assign(static_cast<size_t>((n + 1) / 2 * 2) * 2, 0u);
    for (int t = 0; t < hs.ntiles; ++t) {
        const float* tb = &hs.tbox[static_cast<size_t>(t) * 8];
        float* F = &hs.tframe[static_cast<size_t>(t) * 8];
        double o[3], inv[3];
        for (int d = 0; d < 3; ++d) {
            const double lo = static_cast<double>(tb[d]) - static_cast<double>(tb[4 + d]);
            const double hi = static_cast<double>(tb[d]) + static_cast<double>(tb[4 + d]);
            const double st = std::max((hi - lo) / 251.0, smin);
            F[d] = static_cast<float>(lo - 2.0 * st);
            F[4 + d] = static_cast<float>(1.0 / st);
            o[d] = F[d];
            inv[d] = F[4 + d];
        }
        for (int k = t * 64; k < std::min(n, t * 64 + 64); ++k) {
            const float* b = &hs.sbox[static_cast<size_t>(k) * 8];
            uint32_t q[6];
            for (int d = 0; d < 3; ++d) {
                const double lo = (static_cast<double>(b[d]) - static_cast<double>(b[4 + d]) - o[d]) * inv[d];
                const double hi = (static_cast<double>(b[d]) + static_cast<double>(b[4 + d]) - o[d]) * inv[d];
                const double ql = std::floor(lo) - 1.0, qh = std::ceil(hi) + 1.0;
                if (ql < 0.0 || qh > 255.0) throw std::runtime_error("quantised member box out of its tile frame");
                q[d] = static_cast<uint32_t>(ql);
                q[3 + d] = static_cast<uint32_t>(qh);
            }
            hs.qbox[2 * static_cast<size_t>(k)] = q[0] | (q[1] << 8) | (q[2] << 16) | (q[3] << 24);
            hs.qbox[2 * static_cast<size_t>(k) + 1] = q[4] | (q[5] << 8);
        }
    }
}

}  // namespace visrt
