// Host-side angle records (the transcendental part of the matrix entries,
// kept on the host so atan2 rounds exactly as the reference's libm call).
//
//   oriented_angle_deg        src/geom.cpp:64-73
//   clamp_visibility_angle    src/geom.cpp:75-77
//   angle_record              src/vismatrix.cpp:332-351
//   range_is_degenerate       src/vismatrix.cpp:353-356
//   first_order_ranges        src/vismatrix.cpp:372-385
//   required_planes           src/vismatrix.cpp:171-181
#pragma once

#include <cmath>

#include "visrt_internal.h"

namespace visrt {

struct AngleRec {
    double vx, vy;      // vertex
    double dx, dy;      // ref_dir
    double ox, oy;      // outward
    double low, high;
};

inline double oriented_angle_deg(double dx, double dy, double nx, double ny, double vx, double vy) {
    constexpr double kPi = 3.14159265358979323846;
    constexpr double kRad2Deg = 180.0 / kPi;
    const double s = (dx * ny - dy * nx) >= 0.0 ? 1.0 : -1.0;
    double a = std::atan2(s * (dx * vy - dy * vx), dx * vx + dy * vy) * kRad2Deg;
    if (a < 0.0) a += 360.0;
    if (a >= 360.0) a -= 360.0;
    return a;
}

inline double clamp_visibility_angle(double a) { return a < 180.0 ? a : 0.0; }

// seg = a.x a.y b.x b.y n.x n.y
inline AngleRec angle_record(double atx, double aty, double otx, double oty, double ox, double oy,
                             const double* aim_seg) {
    AngleRec r;
    r.vx = atx;
    r.vy = aty;
    r.ox = ox;
    r.oy = oy;
    const double ddx = otx - atx, ddy = oty - aty;
    const double inv = 1.0 / std::sqrt(ddx * ddx + ddy * ddy);
    r.dx = ddx * inv;
    r.dy = ddy * inv;
    auto angle_to = [&](double tx, double ty) {
        const double vx = tx - atx, vy = ty - aty;
        if (std::sqrt(vx * vx + vy * vy) <= kEps) return 0.0;
        return clamp_visibility_angle(oriented_angle_deg(r.dx, r.dy, ox, oy, vx, vy));
    };
    const double a1 = angle_to(aim_seg[0], aim_seg[1]);
    const double a2 = angle_to(aim_seg[2], aim_seg[3]);
    r.low = a2 < a1 ? a2 : a1;    // std::min
    r.high = a1 < a2 ? a2 : a1;   // std::max
    return r;
}

inline void first_order_ranges(const HostScene& hs, int ref, int aim, int plane, AngleRec& at_a,
                               AngleRec& at_b) {
    const double* sr = &hs.seg[(static_cast<size_t>(ref) * 3 + plane) * 6];
    const double* sa = &hs.seg[(static_cast<size_t>(aim) * 3 + plane) * 6];
    at_a = angle_record(sr[0], sr[1], sr[2], sr[3], sr[4], sr[5], sa);
    at_b = angle_record(sr[2], sr[3], sr[0], sr[1], sr[4], sr[5], sa);
}

inline bool range_is_degenerate(const AngleRec& a, const AngleRec& b) {
    return std::abs(a.high - a.low) <= 1e-12 && std::abs(b.high - b.low) <= 1e-12;
}

inline int required_planes(const HostScene& hs, int i, int j) {
    int m = 0;
    for (int pl = 0; pl < 3; ++pl) {
        if (!hs.seg_ok[3 * i + pl] || !hs.seg_ok[3 * j + pl]) continue;
        const double* a = &hs.seg[(static_cast<size_t>(i) * 3 + pl) * 6];
        const double* b = &hs.seg[(static_cast<size_t>(j) * 3 + pl) * 6];
        const double d = std::abs(a[4] * b[4] + a[5] * b[5]);
        if (d >= 1.0 - 1e-9 || d <= 1e-9) m |= 1 << pl;
    }
    return m;
}

// Conservative screen (no atan2): true when the angle record at `at` is
// certainly NOT degenerate — both aim endpoints clearly in front of the ref
// line (angles strictly inside (0, 180), never clamped) at clearly different
// angles, or one clearly in front and the other clearly behind (clamped to 0).
// The 1e-6 relative margins dwarf every rounding of the exact path, whose
// threshold is 1e-12 degrees; anything near a boundary goes to the exact check.
inline bool record_clearly_open(double atx, double aty, double otx, double oty, double ox, double oy,
                                const double* aim_seg) {
    constexpr double kM = 1e-6;
    const double dx = otx - atx, dy = oty - aty;
    const double dl = std::sqrt(dx * dx + dy * dy);
    if (!(dl > 0.0)) return false;
    const double ux = dx / dl, uy = dy / dl;
    const double sg = (ux * oy - uy * ox) >= 0.0 ? 1.0 : -1.0;
    double y[2], r[2], vx[2], vy[2];
    for (int q = 0; q < 2; ++q) {
        vx[q] = aim_seg[2 * q] - atx;
        vy[q] = aim_seg[2 * q + 1] - aty;
        r[q] = std::sqrt(vx[q] * vx[q] + vy[q] * vy[q]);
        if (!(r[q] > 1e-6)) return false;   // near-coincident endpoint: exact path
        y[q] = sg * (ux * vy[q] - uy * vx[q]);
    }
    const bool f0 = y[0] > kM * r[0], f1 = y[1] > kM * r[1];
    const bool b0 = y[0] < -kM * r[0], b1 = y[1] < -kM * r[1];
    if (f0 && f1) return std::fabs(vx[0] * vy[1] - vy[0] * vx[1]) > kM * r[0] * r[1];
    return (f0 && b1) || (b0 && f1);
}

inline bool range_clearly_open(const HostScene& hs, int ref, int aim, int plane) {
    const double* sr = &hs.seg[(static_cast<size_t>(ref) * 3 + plane) * 6];
    const double* sa = &hs.seg[(static_cast<size_t>(aim) * 3 + plane) * 6];
    return record_clearly_open(sr[0], sr[1], sr[2], sr[3], sr[4], sr[5], sa) ||
           record_clearly_open(sr[2], sr[3], sr[0], sr[1], sr[4], sr[5], sa);
}

// first_order_pair drops the pair when any (plane, direction) range is
// degenerate (src/vismatrix.cpp:614-624). The screen settles almost every
// range without atan2; the rest run the reference's exact records.
inline bool pair_range_degenerate(const HostScene& hs, int i, int j) {
    const int planes = required_planes(hs, i, j);
    for (int pl = 0; pl < 3; ++pl) {
        if (!(planes >> pl & 1)) continue;
        AngleRec a, b;
        if (!range_clearly_open(hs, i, j, pl)) {
            first_order_ranges(hs, i, j, pl, a, b);
            if (range_is_degenerate(a, b)) return true;
        }
        if (!range_clearly_open(hs, j, i, pl)) {
            first_order_ranges(hs, j, i, pl, a, b);
            if (range_is_degenerate(a, b)) return true;
        }
    }
    return false;
}

}  // namespace visrt
