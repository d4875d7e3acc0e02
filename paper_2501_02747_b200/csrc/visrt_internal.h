// Internal layout shared by the host ingest and the sm_100a kernels.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/visrt.h"

namespace visrt {

constexpr double kEps = 1e-9;  // reference kEps, include/rt/geom.hpp:14

// Occluder record (device AoS, one per face, double precision):
//   [0..2]  P  = pts[0]          (plane point, include/rt/geom.hpp:110)
//   [3..5]  n  = Newell normal   (src/geom.cpp:126-140)
//   [6..8]  inward_0             (edge pts[0]->pts[1]; a_0 = P)
//   then for k = 1..MAXV-1: a_k (3), inward_k (3)
// inward_k = cross(n, e_k) / |e_k| computed on the host exactly as
// ConvexPolygon::contains does (src/geom.cpp:155-167); an edge the reference
// skips (|e| < kEps) or a padding edge (k >= nv) stores inward = 0, which
// makes dot(p - a, inward) = 0 >= -eps: the same "skip" without a branch.
template <int MAXV>
struct RecLayout {
    static constexpr int kDoubles = 6 + 3 + (MAXV - 1) * 6;
    static constexpr int kStride = (kDoubles + 1) / 2 * 2;  // 16-B multiple
};

constexpr int kGroup = 16;   // faces per culling group (the mid level of the non-resident sweep)

// Samples (face_samples, src/vismatrix.cpp:226-249): vertices, centroid,
// then the grid (quads: 16 bilinear points; k-gons: 3 per vertex).
constexpr int kMaxSamples = VISRT_MAX_VERTS + 1 + 3 * VISRT_MAX_VERTS;

struct HostScene {
    int32_t n = 0;
    int32_t maxv = 0;                 // max vertices over faces
    std::vector<int32_t> nv;          // vertices per face
    std::vector<int32_t> ns;          // samples per face
    std::vector<double> pts;          // [n][MAXV_ALL][3] padded rings
    std::vector<double> normal;       // [n][3]
    std::vector<int32_t> orient;      // 0 H, 1 V, 2 O
    std::vector<double> seg;          // [n][3][6]
    std::vector<int32_t> seg_ok;      // [n][3]
    std::vector<double> samples;      // [n][kMaxSamples][3]
    std::vector<double> rec4;         // occluder records, MAXV = 4 layout (if maxv <= 4)
    std::vector<double> rec8;         // occluder records, MAXV = 8 layout
    std::vector<double> aabb;         // [n][6] lo.xyz hi.xyz
    std::vector<int32_t> building;    // [n], -1 none
    // fp32 conservative culling boxes: centre (relative to `origin`) and
    // dilated half-size, [n][8] = cx cy cz 0 hx hy hz 0 (see box_margin()).
    std::vector<float> box;
    double origin[3] = {0, 0, 0};
    double extent = 0;                // max |coordinate - origin| over the scene
    // two-level culling hierarchy: Morton order of the xy AABB centres,
    // tiles of 64 consecutive faces with union boxes (sweep.h)
    std::vector<int32_t> perm, inv;
    std::vector<float> sbox, tbox, gbox, cbox;   // member / tile (64) / group (16) / chunk (4096) boxes, Morton order
    std::vector<double> srec;         // records in Morton order (layout of rec4/rec8)
    // quantised member boxes (sweep.h QRES): per tile a frame [o.xyz 0 inv.xyz 0]
    // (fp32 origin and inverse step of an 8-bit grid), per member 8 bytes
    // (lo.x lo.y lo.z hi.x | hi.y hi.z 0 0), rounded outward plus one step
    std::vector<float> tframe;
    std::vector<uint32_t> qbox;       // [n rounded up to even][2]
    int32_t ntiles = 0, nchunks = 0, ngroups = 0;
};

// Dilation of the fp32 culling boxes. A true hit of segment_face_intersection
// lies on the segment (t in (0,1), rounding ~1e-12 m) and inside the face's
// eps-mitered polygon (|plane dist| <= 1e-9, every edge dot >= -1e-9: at most
// 1e-9/sin(theta_min/2) outside the polygon). The fp32 SAT compares products of
// magnitude <= (2*extent)^2 with relative error ~4*2^-24; its absolute error is
// absorbed by a dilation of 2^-20*extent*16. 0.01 m adds a further floor.
inline double box_margin(double extent, double miter) {
    return 0.01 + 16.0 * extent * 9.5367431640625e-7 + 4.0 * miter;
}

// Host ingest with the reference's exact arithmetic. Throws std::runtime_error
// with the reference's SceneError-style message on invalid input.
void ingest(const visrt_facets_v1& f, HostScene& hs);
void build_hierarchy(HostScene& hs);

// Sightline count S(i,j) of occlusion_judgment (src/vismatrix.cpp:263-273).
inline int sightline_count(int nr, int nsr, int na, int nsa) {
    const int gr = nsr - nr - 1, ga = nsa - na - 1;
    return nr * na + 1 + (gr < ga ? gr : ga);
}

}  // namespace visrt
