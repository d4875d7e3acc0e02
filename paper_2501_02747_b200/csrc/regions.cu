// (2) Per-snapshot point regions: illuminated_region(source, face) for every
// (snapshot source, face), batched over all snapshots at once (K4).
//
// Reference: src/vistable.cpp:287-334 (illuminated_region), 140-193
// (visible_intervals: 65 columns x <= 7 transverse samples, bisection
// refine() <= 50 iterations), 102-126 (column_span), 84-98 (face_param),
// 38-44 (sightline_clear).
//
// One lane = one (source, face) region, a sequential state machine:
//   plane XY, YZ, XZ (those with a face_param) ->
//     SCAN   columns u_i = i/64, each col_vis(u) = first clear of <= 7
//            sightlines source -> face point;
//     REFINE for each visible run, bisect its interior boundaries (same
//            midpoints, same 1e-15 stop, same iteration cap);
//     best interval (first largest) -> sub[2], clipped.
// Every sightline is one culled any-hit sweep (sweep.h) over all faces but
// the target, with the 2-entry blocker cache. The lane's arithmetic follows
// the reference operation by operation, so sub[] is bit-identical.
//
// K4w (k_point_regions_warp, the default since r01) runs the same algorithm
// with a WARP per region as uniform straight-line code and one
// warp-cooperative sweep (coop_any_hit) per sightline; it also has a
// presence-only mode (scan until the first visible column) for callers that
// only need whether a region exists (trajectory keys of order 1).
// K5 (k_beam_rows): TableBuilder::reach through 1..4 reflectors.
#include <algorithm>
#include <cstdlib>

#include "device.h"
#include "sweep.h"
#include "tables.h"

namespace visrt {


__device__ __forceinline__ double dmin_std(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double dmax_std(double a, double b) { return (a < b) ? b : a; }

// face_param (src/vistable.cpp:84-98) recomputed on the fly from the face
// ring: (u, s) of vertex k.
__device__ __forceinline__ void face_us(const DevScene& s, int f, int pl, int k, double ax, double ay, double dx,
                                        double dy, double len2, double& u, double& sv) {
    const double* P = s.pts + (static_cast<size_t>(f) * VISRT_MAX_VERTS + k) * 3;
    double qx, qy;
    if (pl == 0) {
        qx = P[0]; qy = P[1]; sv = P[2];
    } else if (pl == 1) {
        qx = P[1]; qy = P[2]; sv = P[0];
    } else {
        qx = P[0]; qy = P[2]; sv = P[1];
    }
    u = __ddiv_rn(dadd(dmul(dsub(qx, ax), dx), dmul(dsub(qy, ay), dy)), len2);
}

// column_span (src/vistable.cpp:102-126)
__device__ bool column_span(const DevScene& s, int f, int pl, double ax, double ay, double dx, double dy,
                            double len2, double u, double& lo_o, double& hi_o) {
    const int nv = s.nv[f];
    double lo = 0.0, hi = 0.0;
    bool any = false;
    double u0, s0v;
    face_us(s, f, pl, 0, ax, ay, dx, dy, len2, u0, s0v);
    double ua = u0, sa = s0v;
    for (int i = 0; i < nv; ++i) {
        double ub, sb;
        if (i + 1 < nv) face_us(s, f, pl, i + 1, ax, ay, dx, dy, len2, ub, sb);
        else { ub = u0; sb = s0v; }
        const double da = dsub(ua, u), db = dsub(ub, u);
        if (fabs(da) <= 1e-12) {
            if (!any) { lo = hi = sa; any = true; }
            else { lo = dmin_std(lo, sa); hi = dmax_std(hi, sa); }
        }
        if ((da < 0.0) != (db < 0.0) && fabs(dsub(da, db)) > 1e-15) {
            const double sv = dadd(sa, dmul(dsub(sb, sa), __ddiv_rn(da, dsub(da, db))));
            if (!any) { lo = hi = sv; any = true; }
            else { lo = dmin_std(lo, sv); hi = dmax_std(hi, sv); }
        }
        ua = ub;
        sa = sb;
    }
    lo_o = lo;
    hi_o = hi;
    return any;
}

// column_span on the face's (u, s) ring precomputed once per plane (the
// reference's FaceParam::poly_us, src/vistable.cpp:84-98): same values, no
// per-call divisions.
__device__ bool column_span_us(const double* us, int nv, double u, double& lo_o, double& hi_o) {
    double lo = 0.0, hi = 0.0;
    bool any = false;
    double ua = us[0], sa = us[1];
#pragma unroll 1
    for (int i = 0; i < nv; ++i) {
        const double ub = i + 1 < nv ? us[2 * i + 2] : us[0];
        const double sb = i + 1 < nv ? us[2 * i + 3] : us[1];
        const double da = dsub(ua, u), db = dsub(ub, u);
        if (fabs(da) <= 1e-12) {
            if (!any) { lo = hi = sa; any = true; }
            else { lo = dmin_std(lo, sa); hi = dmax_std(hi, sa); }
        }
        if ((da < 0.0) != (db < 0.0) && fabs(dsub(da, db)) > 1e-15) {
            const double sv = dadd(sa, dmul(dsub(sb, sa), __ddiv_rn(da, dsub(da, db))));
            if (!any) { lo = hi = sv; any = true; }
            else { lo = dmin_std(lo, sv); hi = dmax_std(hi, sv); }
        }
        ua = ub;
        sa = sb;
    }
    lo_o = lo;
    hi_o = hi;
    return any;
}

// column_span_us for one warp-uniform u with the polygon edges on lanes
// 0..nv-1: each lane forms its edge's taken values in the reference's order,
// then an order-preserving tree reduction (std::min / std::max keep the
// earlier of equal values, and "leftmost extremum" is associative) gives the
// sequential fold's lo / hi. All lanes; uniform result.
__device__ bool column_span_warp(const double* us, int nv, double u, double& lo_o, double& hi_o) {
    const int lane = threadIdx.x & 31;
    double lo = __longlong_as_double(0x7ff0000000000000LL), hi = -lo;   // +inf / -inf: nothing taken
    if (lane < nv) {
        const double ua = us[2 * lane], sa = us[2 * lane + 1];
        const double ub = lane + 1 < nv ? us[2 * lane + 2] : us[0];
        const double sb = lane + 1 < nv ? us[2 * lane + 3] : us[1];
        const double da = dsub(ua, u), db = dsub(ub, u);
        if (fabs(da) <= 1e-12) {
            lo = sa;
            hi = sa;
        }
        if ((da < 0.0) != (db < 0.0) && fabs(dsub(da, db)) > 1e-15) {
            const double sv = dadd(sa, dmul(dsub(sb, sa), __ddiv_rn(da, dsub(da, db))));
            lo = dmin_std(lo, sv);
            hi = dmax_std(hi, sv);
        }
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {   // lane l combines with lane l + o (its right neighbour run)
        const double rl = __shfl_down_sync(kFull, lo, o), rh = __shfl_down_sync(kFull, hi, o);
        lo = dmin_std(lo, rl);
        hi = dmax_std(hi, rh);
    }
    lo = __shfl_sync(kFull, lo, 0);
    hi = __shfl_sync(kFull, hi, 0);
    lo_o = lo;
    hi_o = hi;
    return lo <= hi;
}

// double(j) / (kTransverse - 1), j = 0..6 (correctly rounded, as the reference)
__constant__ double kSampFrac[7] = {0.0 / 6.0, 1.0 / 6.0, 2.0 / 6.0, 3.0 / 6.0, 4.0 / 6.0, 5.0 / 6.0, 6.0 / 6.0};

template <int MAXV, bool RESIDENT>
__global__ void __launch_bounds__(kThreads, 2) k_point_regions(RegionArgs a) {
    constexpr int STRIDE = RecLayout<MAXV>::kStride;
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t bar[1];
    const DevScene& s = a.s;
    const int n = s.n;
    const int lane = threadIdx.x & 31;
    const SweepCtx ctx = sweep_setup<RESIDENT>(s, smem, bar);

    // ---- lane state --------------------------------------------------------
    bool active = false, exhausted = false, querying = false;
    long long tid = 0;
    int f = 0, pl = 0;
    double sx = 0, sy = 0, sz = 0;      // source
    double ax = 0, ay = 0, dx = 0, dy = 0, len2 = 0;   // face_param of plane pl
    double us[2 * MAXV];                // face_param poly_us of plane pl
    auto load_us = [&]() {
        const int nv = s.nv[f];
        for (int k = 0; k < nv; ++k) face_us(s, f, pl, k, ax, ay, dx, dy, len2, us[2 * k], us[2 * k + 1]);
    };
    // SCAN / REFINE
    int phase = 0;                      // 0 scan, 1 refine
    int col = 0;                        // scan column
    unsigned long long vis = 0;         // columns 0..63
    bool vis64 = false;                 // column 64
    int run_i = 0, run_j = 0, which = 0, it = 0;
    double lo = 0, hi = 0, r_start = 0;
    bool lo_vis = false;
    bool have_best = false;
    double best0 = 0, best1 = 0;
    // col_vis in progress
    double cu = 0, cs0 = 0, cs1 = 0, inset = 0;
    int samp = 0;
    // region output
    int8_t has[3] = {0, 0, 0}, clp[3] = {0, 0, 0};
    double sub[6] = {0, 0, 0, 0, 0, 0};
    // sightline query
    double qx = 0, qy = 0, qz = 0;
    Sweep sw{};
    int sf = 0, bc0 = -1, bc1 = -1;     // sf: Morton index of the target face; cache: Morton indices
    unsigned long long tests = 0, queries = 0;
    (void)n;

    auto vis_at = [&](int i) { return i == 64 ? vis64 : ((vis >> i) & 1ull) != 0; };
    auto exact = [&](int k) {
        ++tests;
        return seg_hits<MAXV>(s.srec + static_cast<size_t>(k) * STRIDE, sx, sy, sz, qx, qy, qz);
    };
    auto write_out = [&](int8_t present) {
        visrt_region r;
        r.present = present;
        r.pad = 0;
        for (int t = 0; t < 3; ++t) {
            r.has[t] = present == 1 ? has[t] : 0;
            r.clipped[t] = present == 1 ? clp[t] : 0;
        }
        for (int t = 0; t < 6; ++t) r.sub[t] = present == 1 ? sub[t] : 0.0;
        a.out[tid] = r;
        active = false;
        querying = false;
    };
    // Set up sample `samp` of the current column; returns false when all 7
    // samples are used (column not visible). Samples the blocker cache
    // already blocks are settled here.
    auto next_sample = [&]() -> bool {
        for (; samp < 7; ++samp) {
            const double fj = kSampFrac[samp];
            const double sv = dmin_std(dsub(cs1, inset), dmax_std(dadd(cs0, inset), dadd(cs0, dmul(dsub(cs1, cs0), fj))));
            const double px = dadd(ax, dmul(dx, cu));
            const double py = dadd(ay, dmul(dy, cu));
            if (pl == 0) { qx = px; qy = py; qz = sv; }
            else if (pl == 1) { qx = sv; qy = px; qz = py; }
            else { qx = px; qy = sv; qz = py; }
            ++queries;
            if (bc0 >= 0 && bc0 != sf && exact(bc0)) continue;
            if (bc1 >= 0 && bc1 != sf && exact(bc1)) {
                const int t = bc0;
                bc0 = bc1;
                bc1 = t;
                continue;
            }
            sw.start(make_segf(s, sx, sy, sz, qx, qy, qz), sf, -1, home_chunk(s, f), ctx.nchunks);
            return true;
        }
        return false;
    };
    // Begin col_vis(u); returns true when a sweep is pending, false when the
    // column was decided without one (result in `res`).
    auto begin_col = [&](double u, bool& res) -> bool {
        cu = u < 0.0 ? 0.0 : (1.0 < u ? 1.0 : u);   // std::clamp
        if (!column_span_us(us, s.nv[f], cu, cs0, cs1)) {
            res = false;
            return false;
        }
        inset = dmul(dsub(cs1, cs0), 1e-6);
        samp = 0;
        if (next_sample()) return true;
        res = false;
        return false;
    };
    // Drive the state machine until a sweep is pending or the region is done.
    // `have` / `res`: a col_vis result to consume first.
    auto pump = [&](bool have, bool res) {
        for (;;) {
            if (have) {
                have = false;
                if (phase == 0) {
                    if (res) {
                        if (col == 64) vis64 = true;
                        else vis |= 1ull << col;
                    }
                    ++col;
                } else {
                    // refine step (src/vistable.cpp:164-173)
                    const double mid = dmul(0.5, dadd(lo, hi));
                    if (res == lo_vis) lo = mid;
                    else hi = mid;
                    ++it;
                }
            }
            if (phase == 0) {
                if (col < 65) {
                    bool r = false;
                    if (begin_col(__ddiv_rn(static_cast<double>(col), 64.0), r)) {
                        querying = true;
                        return;
                    }
                    have = true;
                    res = r;
                    continue;
                }
                // scan done: set up runs (src/vistable.cpp:175-192)
                phase = 1;
                run_i = 0;
                which = -1;
                have_best = false;
            }
            // ---- REFINE ----
            if (which >= 0 && it < 50 && dsub(hi, lo) > 1e-15) {
                bool r = false;
                if (begin_col(dmul(0.5, dadd(lo, hi)), r)) {
                    querying = true;
                    return;
                }
                have = true;
                res = r;
                continue;
            }
            if (which == 0) {
                // start refined: r_start
                r_start = dmul(0.5, dadd(lo, hi));
                which = -2;   // proceed to the end boundary
            } else if (which == 1) {
                const double end = dmul(0.5, dadd(lo, hi));
                if (!have_best || dsub(best1, best0) < dsub(end, r_start)) {
                    best0 = r_start;
                    best1 = end;
                    have_best = true;
                }
                run_i = run_j + 1;
                which = -1;
            }
            if (which == -2) {
                // end boundary of run [run_i .. run_j]
                if (run_j + 1 < 65) {
                    lo = __ddiv_rn(static_cast<double>(run_j), 64.0);
                    hi = dadd(lo, __ddiv_rn(1.0, 64.0));
                    lo_vis = true;
                    it = 0;
                    which = 1;
                    continue;
                }
                const double end = __ddiv_rn(static_cast<double>(run_j), 64.0);
                if (!have_best || dsub(best1, best0) < dsub(end, r_start)) {
                    best0 = r_start;
                    best1 = end;
                    have_best = true;
                }
                run_i = run_j + 1;
                which = -1;
            }
            // which == -1: find the next run
            while (run_i < 65 && !vis_at(run_i)) ++run_i;
            if (run_i < 65) {
                run_j = run_i;
                while (run_j + 1 < 65 && vis_at(run_j + 1)) ++run_j;
                r_start = __ddiv_rn(static_cast<double>(run_i), 64.0);
                if (run_i > 0) {
                    hi = r_start;
                    lo = dsub(r_start, __ddiv_rn(1.0, 64.0));
                    lo_vis = false;
                    it = 0;
                    which = 0;
                } else {
                    which = -2;
                }
                continue;
            }
            // all runs done: plane result
            if (!have_best) {
                write_out(0);   // fully hidden in this plane: no region
                return;
            }
            has[pl] = 1;
            sub[2 * pl] = best0;
            sub[2 * pl + 1] = best1;
            clp[pl] = (best0 > 1e-9 || best1 < 1.0 - 1e-9) ? 1 : 0;
            // next plane with a face_param
            for (;;) {
                if (++pl == 3) {
                    write_out((has[0] | has[1] | has[2]) ? 1 : 0);
                    return;
                }
                if (!s.seg_ok[3 * f + pl]) continue;
                const double* sg = s.seg + (static_cast<size_t>(f) * 3 + pl) * 6;
                ax = sg[0];
                ay = sg[1];
                dx = dsub(sg[2], sg[0]);
                dy = dsub(sg[3], sg[1]);
                len2 = dadd(dmul(dx, dx), dmul(dy, dy));
                if (len2 <= kEps * kEps) continue;
                break;
            }
            load_us();
            phase = 0;
            col = 0;
            vis = 0;
            vis64 = false;
        }
    };
    auto start_task = [&](long long t) {
        const RegionTask rt = region_task(a, t, n);   // a.face_major == 0 for this kernel
        tid = rt.out;
        const long long k = rt.k;
        f = rt.f;
        sf = s.inv[f];
        sx = a.src[3 * k];
        sy = a.src[3 * k + 1];
        sz = a.src[3 * k + 2];
        for (int q = 0; q < 3; ++q) { has[q] = 0; clp[q] = 0; sub[2 * q] = 0; sub[2 * q + 1] = 0; }
        active = true;
        // back-face test (src/vistable.cpp:289-294)
        const double* P = s.pts + static_cast<size_t>(f) * VISRT_MAX_VERTS * 3;
        const double* N = s.normal + 3 * static_cast<size_t>(f);
        const double dist = dot_rel(sx, sy, sz, P[0], P[1], P[2], N[0], N[1], N[2]);
        if (fabs(dist) <= kEps) { write_out(-1); return; }
        if (dist < 0.0) { write_out(0); return; }
        pl = -1;
        for (;;) {
            if (++pl == 3) { write_out(0); return; }
            if (!s.seg_ok[3 * f + pl]) continue;
            const double* sg = s.seg + (static_cast<size_t>(f) * 3 + pl) * 6;
            ax = sg[0];
            ay = sg[1];
            dx = dsub(sg[2], sg[0]);
            dy = dsub(sg[3], sg[1]);
            len2 = dadd(dmul(dx, dx), dmul(dy, dy));
            if (len2 <= kEps * kEps) continue;
            break;
        }
        load_us();
        phase = 0;
        col = 0;
        vis = 0;
        vis64 = false;
        pump(false, false);
    };
    auto refill = [&]() {
        unsigned need = __ballot_sync(kFull, !active && !exhausted);
        while (need) {
            const int leader = __ffs(need) - 1;
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(&a.counter[0], static_cast<unsigned long long>(__popc(need)));
            base = __shfl_sync(kFull, base, leader);
            if (!active && !exhausted) {
                const long long my = static_cast<long long>(base) + __popc(need & ((1u << lane) - 1u));
                if (my >= a.ntasks) exhausted = true;
                else start_task(my);
            }
            need = __ballot_sync(kFull, !active && !exhausted);
        }
    };
    // One virtual tile of the current sightline sweep.
    // One 64-box culling batch of the current sightline sweep.
    __shared__ int slots[kThreads];
    int* slot = slots + (threadIdx.x & ~31);
    auto step = [&]() {
        unsigned long long mask = 0;
        int base = 0;
        if (querying) mask = sweep_batch(sw, ctx, base);
        const int hk = coop_exact<MAXV>(s.srec, mask, base, sx, sy, sz, qx, qy, qz, slot, tests, 0ull,
                                        [](int, unsigned long long) {});
        if (!querying) return;
        if (hk >= 0) {
            if (hk != bc0) {
                bc1 = bc0;
                bc0 = hk;
            }
            // blocked sample: try the next sample of this column
            ++samp;
            if (next_sample()) return;
            querying = false;
            pump(true, false);
        } else if (sw.done()) {
            querying = false;
            pump(true, true);   // clear sightline: column visible
        }
    };

    refill();
    for (;;) {
        step();
        refill();
        if (!__any_sync(kFull, active || !exhausted)) break;
    }
    for (int o = 16; o > 0; o >>= 1) {
        tests += __shfl_down_sync(kFull, tests, o);
        queries += __shfl_down_sync(kFull, queries, o);
    }
    if (lane == 0) {
        atomicAdd(&a.counter[1], tests);
        atomicAdd(&a.counter[2], queries);
    }
}

// K4w: illuminated_region with a WARP per (source, face) task. The region
// algorithm runs warp-uniformly as straight-line code that mirrors the
// reference (planes -> 65 col_vis columns -> run refinement -> first largest
// interval), and every sightline_clear is ONE warp-cooperative culled sweep
// (sweep.h coop_any_hit) after a one-entry warp blocker cache. Same
// arithmetic, same call order, so every output is bit-identical to K4 — with
// converged lanes and a short per-region critical path (small batches and
// trajectory probes are latency-bound on K4's lane state machines).
#ifndef VISRT_K4W_NI
#define VISRT_K4W_NI 1   // 1: one out-of-line copy of the sweep / blocker test for the K4w helpers
#endif
// The warp sweep and the fp32-SAT + exact blocker test as single out-of-line
// copies: inlined at each call site of the lane-parallel scan and col_vis
// they overflowed the instruction cache (ncu: stall_no_inst).
template <int MAXV, int RES>
__device__ __noinline__ int k4w_sweep(const DevScene& s, const SweepCtx& ctx, double sx, double sy, double sz,
                                      double bx, double by, double bz, int sf, unsigned char* sv,
                                      unsigned long long& tests, unsigned long long& batches) {
    return coop_any_hit<MAXV, 0, RES>(ctx, s.srec, make_segf(s, sx, sy, sz, bx, by, bz), sx, sy, sz, bx, by, bz, sf, -1, sf,
                              sv, tests, batches);
}
// One out-of-line copy of the exact predicate for the K4w helpers (i-cache:
// ncu put 41 % of K4w's warp samples on stall_no_instruction).
#ifndef VISRT_K4W_SEGNI
#define VISRT_K4W_SEGNI 1
#endif
template <int MAXV>
__device__ __noinline__ bool k4w_seg(const double* __restrict__ R, double ax, double ay, double az, double bx, double by,
                                     double bz) {
    return seg_hits<MAXV>(R, ax, ay, az, bx, by, bz);
}
template <int MAXV>
__device__ __forceinline__ bool k4w_exact(const double* __restrict__ R, double ax, double ay, double az, double bx,
                                          double by, double bz) {
    if (VISRT_K4W_SEGNI) return k4w_seg<MAXV>(R, ax, ay, az, bx, by, bz);
    return seg_hits<MAXV>(R, ax, ay, az, bx, by, bz);
}

template <int MAXV, int RES>
__device__ __noinline__ bool k4w_blocked(const DevScene& s, const SweepCtx& ctx, int k, double sx, double sy,
                                         double sz, double qx, double qy, double qz, unsigned long long& tests) {
    if (!member_maybe<RES>(ctx, k, make_segf(s, sx, sy, sz, qx, qy, qz))) return false;
    ++tests;
    return k4w_exact<MAXV>(s.srec + static_cast<size_t>(k) * RecLayout<MAXV>::kStride, sx, sy, sz, qx, qy, qz);
}

// Development aid (-DVISRT_K4W_PROF): per-phase cycle and sweep counters of K4w.
#ifdef VISRT_K4W_PROF
__shared__ unsigned long long k4w_sprof[24];
__device__ unsigned long long g_k4w_prof[24];
#define K4P(i, v)                                                                                     \
    do {                                                                                              \
        if ((threadIdx.x & 31) == 0) atomicAdd(&k4w_sprof[i], static_cast<unsigned long long>(v));     \
    } while (0)
#define K4CLK() clock64()
#else
#define K4P(i, v) \
    do {          \
    } while (0)
#define K4CLK() 0ll
#endif

// K4w walks its tasks face-major by default (RegionArgs::face_major: neighbouring
// warps take one face for consecutive snapshots; r01: config 3 -12 %, config-5
// Tx -9 %, Rx -2.5 %); VISRT_K4W_FACEMAJOR=0 selects the source-major walk.
#ifndef VISRT_K4W_WC
#define VISRT_K4W_WC 3   // warp blocker-cache entries, most recent first (r01, face-major walk, 1/2/3/4 swept: 3 best overall)
#endif
#ifndef VISRT_K4W_CHUNK
#define VISRT_K4W_CHUNK 1   // consecutive (source, face) tasks per warp grab on the streamed big scenes (x 4 on resident scenes, see launch_regions_t)
#endif
// Warp blocker cache: lane q < VISRT_K4W_WC holds entry q (Morton index or
// -1); `next` is the warp-uniform insertion slot. Entries are distinct.
struct WCache {
    int v = -1;
    int next = 0;
    __device__ __forceinline__ int entry(int i) const {   // i-th most recent (call with all lanes)
        return __shfl_sync(kFull, v, (next + 2 * VISRT_K4W_WC - 1 - i) % VISRT_K4W_WC);
    }
    __device__ __forceinline__ void put(int h) {   // all lanes, warp-uniform h
        const int lane = threadIdx.x & 31;
        if (__any_sync(kFull, lane < VISRT_K4W_WC && v == h)) return;
        if (lane == next) v = h;
        next = next + 1 == VISRT_K4W_WC ? 0 : next + 1;
    }
};

#ifndef VISRT_K4W_PCOL
#define VISRT_K4W_PCOL 1   // 1: col_vis decides its 7 samples on 7 lanes; 0: one sample after the other
#endif
// col_vis (src/vistable.cpp:146-159) for the warp kernel: warp-uniform
// arithmetic, one warp-cooperative sweep per transverse sample. Out of line:
// it has three call sites (scan, both refine directions) and inlining them
// blew the instruction cache (ncu: stall_no_inst dominated).
template <int MAXV, int RES>
__device__ __noinline__ bool col_vis_warp(const DevScene& s, const SweepCtx& ctx, const double* us, int nv, int pl,
                                          double ax, double ay, double dx, double dy, double u, double sx,
                                          double sy, double sz, int sf, unsigned char* sv, WCache& cache,
                                          unsigned long long& tests, unsigned long long& queries,
                                          unsigned long long& batches) {
    constexpr int STRIDE = RecLayout<MAXV>::kStride;
    const int lane = threadIdx.x & 31;
    const double cu = u < 0.0 ? 0.0 : (1.0 < u ? 1.0 : u);   // std::clamp
    double cs0, cs1;
    if (!column_span_us(us, nv, cu, cs0, cs1)) return false;
    const double inset = dmul(dsub(cs1, cs0), 1e-6);
    const double px = dadd(ax, dmul(dx, cu));
    const double py = dadd(ay, dmul(dy, cu));
#if VISRT_K4W_PCOL
    {   // the 7 transverse samples on lanes 0..6: col_vis is their OR, so the
        // order they are decided in does not change the verdict
        const int j = lane;
        bool pending = j < 7;
        double qx = 0, qy = 0, qz = 0;
        if (pending) {
            const double sv_ = dmin_std(dsub(cs1, inset),
                                        dmax_std(dadd(cs0, inset), dadd(cs0, dmul(dsub(cs1, cs0), kSampFrac[j]))));
            if (pl == 0) { qx = px; qy = py; qz = sv_; }
            else if (pl == 1) { qx = sv_; qy = px; qz = py; }
            else { qx = px; qy = sv_; qz = py; }
            queries += lane == 0 ? 7 : 0;
        }
        auto blocked_by = [&](int k) {
#if VISRT_K4W_NI
            return k4w_blocked<MAXV, RES>(s, ctx, k, sx, sy, sz, qx, qy, qz, tests);
#else
            return member_maybe<RES>(ctx, k, make_segf(s, sx, sy, sz, qx, qy, qz)) &&
                   (++tests, seg_hits<MAXV>(s.srec + static_cast<size_t>(k) * STRIDE, sx, sy, sz, qx, qy, qz));
#endif
        };
        for (int i = 0; i < VISRT_K4W_WC; ++i) {
            const int k = cache.entry(i);
            if (pending && k >= 0 && k != sf && blocked_by(k)) pending = false;
        }
        for (;;) {
            const unsigned who = __ballot_sync(kFull, pending);
            if (!who) return false;   // every sample blocked
            const int L = __ffs(who) - 1;
            const double bx = __shfl_sync(kFull, qx, L), by = __shfl_sync(kFull, qy, L),
                         bz = __shfl_sync(kFull, qz, L);
#if VISRT_K4W_NI
            const int h = k4w_sweep<MAXV, RES>(s, ctx, sx, sy, sz, bx, by, bz, sf, sv, tests, batches);
#else
            const int h = coop_any_hit<MAXV, 0, RES>(ctx, s.srec, make_segf(s, sx, sy, sz, bx, by, bz), sx, sy, sz, bx, by, bz,
                                             sf, -1, sf, sv, tests, batches);
#endif
            K4P(4, 1);
            if (h < 0) {
                K4P(5, 1);
                return true;
            }
            cache.put(h);
            if (lane == L) pending = false;
            else if (pending && blocked_by(h)) pending = false;
        }
    }
#endif
    for (int j = 0; j < 7; ++j) {
        const double sv_ = dmin_std(dsub(cs1, inset),
                                    dmax_std(dadd(cs0, inset), dadd(cs0, dmul(dsub(cs1, cs0), kSampFrac[j]))));
        double qx, qy, qz;
        if (pl == 0) { qx = px; qy = py; qz = sv_; }
        else if (pl == 1) { qx = sv_; qy = px; qz = py; }
        else { qx = px; qy = sv_; qz = py; }
        queries += lane == 0;   // warp-uniform sample
        const int c0 = cache.entry(0);
        if (c0 >= 0 && c0 != sf) {
            tests += lane == 0;   // warp-uniform test: count it once
            if (seg_hits<MAXV>(s.srec + static_cast<size_t>(c0) * STRIDE, sx, sy, sz, qx, qy, qz)) continue;
        }
        const int h = coop_any_hit<MAXV, 0, RES>(ctx, s.srec, make_segf(s, sx, sy, sz, qx, qy, qz), sx, sy, sz, qx, qy, qz, sf,
                                         -1, sf, sv, tests, batches);
        if (h < 0) return true;
        cache.put(h);
    }
    return false;
}

// REFINE with fan candidate lists (src/vistable.cpp:163-172). Every sightline
// the bisection of one run boundary can ask about for transverse sample j runs
// from the source S to q_j(u), u in [lo, hi]; q_j is piecewise linear in u
// (breakpoints at the face's vertices), so those end points lie in the box
// spanned by q_j at lo, hi and the breakpoints between, and every such sightline
// stays within R_j (the box's half-diagonal) of the axis S -> c_j (its centre).
// One collecting sweep per sample (coop_collect: culling boxes dilated by R_j)
// lists every face that could block any of them; the <= 50 bisection steps then
// decide col_vis(mid) by exact tests against those lists alone — the same
// verdicts as sweeping every sightline, since no other face can block one.
// Returns false (nothing decided) when a list overflows kFanCap.
#ifndef VISRT_K4W_FAN
#define VISRT_K4W_FAN 1
#endif
constexpr int kFanCap = 32;

// The entries of a cone list whose box, dilated by R, meets g (in list order)
// -> fl; returns their count or -1 when more than cap qualify.
__device__ __forceinline__ int cone_filter(ConeBuf cbuf, int L, const SegF& g, float R, int* fl, int cap) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    int cnt = 0;
    for (int e0 = 0; e0 < L; e0 += 32) {
        const int e = e0 + lane;
        bool v = false;
        int m = 0;
        if (e < L) {
            const float4* E = cbuf.at(e);
            float4 c = E[0];
            float4 h = E[1];
            m = __float_as_int(c.w);
            h.x += R;
            h.y += R;
            h.z += R;
            v = sat_maybe4(c, h, g);
        }
        const unsigned b = __ballot_sync(kFull, v);
        const int at = cnt + __popc(b & lt);
        if (v && at < cap) fl[at] = m;
        cnt += __popc(b);
        if (cnt > cap) return -1;
    }
    return cnt;
}

template <int MAXV, int RES>
__device__ __noinline__ bool refine_fan(const DevScene& s, const SweepCtx& ctx, const double* us, int nv, int pl,
                                        double ax, double ay, double dx, double dy, double& lo_io, double& hi_io,
                                        bool lo_vis, double sx, double sy, double sz, int sf, int* fl,
                                        unsigned long long& tests, unsigned long long& queries,
                                        unsigned long long& batches, int& iters, ConeBuf cbuf, int coneL) {
    constexpr int STRIDE = RecLayout<MAXV>::kStride;
    const int lane = threadIdx.x & 31;
    double lo = lo_io, hi = hi_io;
    // per-sample end-point boxes (lane j < 7)
    // sample j of column u from its span [cs0, cs1] (col_vis, src/vistable.cpp:150-156)
    auto point_at = [&](double cu, double cs0, double cs1, int j, double& qx, double& qy, double& qz) {
        const double inset = dmul(dsub(cs1, cs0), 1e-6);
        const double px = dadd(ax, dmul(dx, cu));
        const double py = dadd(ay, dmul(dy, cu));
        const double v = dmin_std(dsub(cs1, inset), dmax_std(dadd(cs0, inset), dadd(cs0, dmul(dsub(cs1, cs0), kSampFrac[j]))));
        if (pl == 0) { qx = px; qy = py; qz = v; }
        else if (pl == 1) { qx = v; qy = px; qz = py; }
        else { qx = px; qy = v; qz = py; }
    };
    auto sample = [&](double u, int j, double& qx, double& qy, double& qz) -> bool {
        const double cu = u < 0.0 ? 0.0 : (1.0 < u ? 1.0 : u);   // std::clamp
        double cs0, cs1;
        if (!column_span_us(us, nv, cu, cs0, cs1)) return false;
        const double inset = dmul(dsub(cs1, cs0), 1e-6);
        const double px = dadd(ax, dmul(dx, cu));
        const double py = dadd(ay, dmul(dy, cu));
        const double v = dmin_std(dsub(cs1, inset), dmax_std(dadd(cs0, inset), dadd(cs0, dmul(dsub(cs1, cs0), kSampFrac[j]))));
        if (pl == 0) { qx = px; qy = py; qz = v; }
        else if (pl == 1) { qx = v; qy = px; qz = py; }
        else { qx = px; qy = v; qz = py; }
        return true;
    };
    const long long fclk0 = K4CLK();
    double bl[3] = {1e300, 1e300, 1e300}, bh[3] = {-1e300, -1e300, -1e300};
    if (lane < 7) {
        auto grow = [&](double u) {
            double q[3];
            if (!sample(u, lane, q[0], q[1], q[2])) return;
            for (int d = 0; d < 3; ++d) {
                bl[d] = fmin(bl[d], q[d]);
                bh[d] = fmax(bh[d], q[d]);
            }
        };
        // lo, hi and every vertex column strictly between (one call site: i-cache)
#pragma unroll 1
        for (int q = -2; q < nv; ++q) {
            const double u = q == -2 ? lo : (q == -1 ? hi : us[2 * q]);
            if (q < 0 || (u > lo && u < hi)) grow(u);
        }
    }
    int my_cnt = 0;   // lane j < 7: the length of sample j's fan list
#pragma unroll 1
    for (int j = 0; j < 7; ++j) {
        const double c0 = __shfl_sync(kFull, 0.5 * (bl[0] + bh[0]), j), c1 = __shfl_sync(kFull, 0.5 * (bl[1] + bh[1]), j),
                     c2 = __shfl_sync(kFull, 0.5 * (bl[2] + bh[2]), j);
        const double e0 = __shfl_sync(kFull, bh[0] - bl[0], j), e1 = __shfl_sync(kFull, bh[1] - bl[1], j),
                     e2 = __shfl_sync(kFull, bh[2] - bl[2], j);
        int cj = 0;   // no column span anywhere in [lo, hi]: col_vis is false throughout
        if (e0 >= 0.0) {
            // half-diagonal, rounded up generously (fp32 box test)
            const float R = static_cast<float>(0.5 * sqrt(e0 * e0 + e1 * e1 + e2 * e2) * 1.0001 + 1e-6);
            const SegF gj = make_segf(s, sx, sy, sz, c0, c1, c2);
            // the task's cone list holds every face that can block a sightline to
            // the face: filter it (without one — an overflowing cone — the
            // caller bisects with per-sightline sweeps instead)
            cj = coneL >= 0 ? cone_filter(cbuf, coneL, gj, R, fl + j * kFanCap, kFanCap) : -1;
            if (cj < 0) return false;
        }
        if (lane == j) my_cnt = cj;
    }
    __syncwarp();
    K4P(16, K4CLK() - fclk0);
    int T = my_cnt;   // every sample's fan: the pairs of one step
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) T += __shfl_xor_sync(kFull, T, o) * (lane < 8 ? 1 : 0);
    T = __shfl_sync(kFull, T, 0);
    K4P(17, T);
    K4P(18, 1);
    // Each step deals its (sample, fan entry) pairs 32 per round in a rotated
    // sample order — the sample found clear by the previous step leads
    // (neighbouring midpoints mostly share the verdict). A lane's pair in
    // rounds 0 and 1 is fixed for a given order (precomputed), every lane forms
    // its own sample's end point from the step's column span (uniform), and the
    // verdict is kept as per-SAMPLE bit masks: the step stops as soon as a
    // sample has been tested against its whole fan without a hit (visible) or
    // every sample is blocked (hidden) — the same verdict as testing all pairs.
    int rot = 0, jl = 0, cl = 0, excl = 0;   // lane l < 7: sample jl of the order, its fan size, prefix
    int pj0 = -1, pe0 = 0, pj1 = -1, pe1 = 0;
    unsigned done0 = 0, done1 = 0, empty = 0;
    auto owner = [&](int g, int& j, int& e) {   // all lanes: pair g of the order -> (sample, fan entry)
        int l = 0;
#pragma unroll
        for (int k = 1; k < 7; ++k)
            if (__shfl_sync(kFull, excl, k) <= g) l = k;
        j = __shfl_sync(kFull, jl, l);
        e = g - __shfl_sync(kFull, excl, l);
        if (g >= T) j = -1;
    };
    auto done_by = [&](int r_end) {   // samples whose pairs all lie before pair r_end
        return __reduce_or_sync(kFull, (lane < 7 && excl + cl <= r_end) ? 1u << jl : 0u);
    };
    auto order = [&]() {
        jl = lane < 7 ? (lane + rot >= 7 ? lane + rot - 7 : lane + rot) : 0;
        cl = __shfl_sync(kFull, my_cnt, jl);
        if (lane >= 7) cl = 0;
        excl = cl;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const int v = __shfl_up_sync(kFull, excl, o);
            if (lane >= o) excl += v;
        }
        excl -= cl;
        owner(lane, pj0, pe0);
        owner(32 + lane, pj1, pe1);
        done0 = done_by(32);
        done1 = done_by(64);
        empty = __reduce_or_sync(kFull, (lane < 7 && cl == 0) ? 1u << jl : 0u);
    };
    order();
    int it = 0;
    for (; it < 50 && dsub(hi, lo) > 1e-15; ++it) {
        const double mid = dmul(0.5, dadd(lo, hi));
        const long long sc0_ = K4CLK();
        // the step's column span once, its edges on lanes (column_span_warp)
        const double cu = mid < 0.0 ? 0.0 : (1.0 < mid ? 1.0 : mid);   // std::clamp
        double cs0, cs1;
        const bool span = column_span_warp(us, nv, cu, cs0, cs1);
        K4P(22, K4CLK() - sc0_);
        unsigned blocked = 0;   // bit j: sample j is blocked
        bool vis = false;
        int clear_s = -1;
        if (span) {   // no span: no sample, col_vis is false
            if (empty) {   // a sample with an empty fan is clear
                vis = true;
                clear_s = __ffs(empty) - 1;
            }
            for (int r = 0; r < T && !vis; r += 32) {
                int j, e;
                if (r == 0) {
                    j = pj0;
                    e = pe0;
                } else if (r == 32) {
                    j = pj1;
                    e = pe1;
                } else {
                    owner(r + lane, j, e);
                }
                bool hit = false;
                if (j >= 0 && !((blocked >> j) & 1u)) {
                    double qx, qy, qz;
                    point_at(cu, cs0, cs1, j, qx, qy, qz);
                    ++tests;
                    hit = k4w_exact<MAXV>(s.srec + static_cast<size_t>(fl[j * kFanCap + e]) * STRIDE, sx, sy, sz, qx,
                                          qy, qz);
                }
                blocked |= __reduce_or_sync(kFull, hit ? 1u << j : 0u);
                const unsigned dm = r == 0 ? done0 : (r == 32 ? done1 : done_by(r + 32));
                const unsigned clr = dm & ~blocked & 0x7fu;
                if (clr) {   // a sample clear of its whole fan
                    vis = true;
                    clear_s = __ffs(clr) - 1;
                } else if ((~blocked & 0x7fu) == 0u) {
                    break;   // every sample blocked
                }
            }
        }
        K4P(23, K4CLK() - sc0_);
        queries += lane == 0 ? 7 : 0;
        if (vis == lo_vis) lo = mid;
        else hi = mid;
        if (vis && clear_s != rot) {
            rot = clear_s;
            order();
        }
    }
    iters = it;
    lo_io = lo;
    hi_io = hi;
    return true;
}

// The cone list of task (source S, face f): every face but f whose culling
// box may meet hull(S, f) (sweep.h ConeF / coop_collect_cone), written to the
// warp's slice of the launch's cone buffer. Every sightline of
// visible_intervals runs from S to a point of f, so a face outside the list
// blocks none of them. Returns the count, or -1 (overflow / quantised boxes).
constexpr int kConeUnbuilt = -2;
template <int MAXV, int RES>
__device__ __noinline__ int build_cone(const DevScene& s, const SweepCtx& ctx, int f, double sx, double sy, double sz,
                                       int sf, ConeBuf cbuf, unsigned long long& batches) {
    const double* bb = s.aabb + static_cast<size_t>(f) * 6;
    const double cx = 0.5 * (bb[0] + bb[3]), cy = 0.5 * (bb[1] + bb[4]), cz = 0.5 * (bb[2] + bb[5]);
    const double ex = bb[3] - bb[0], ey = bb[4] - bb[1], ez = bb[5] - bb[2];
    const double r = 0.5 * sqrt(ex * ex + ey * ey + ez * ez) * 1.0001 + 1e-6;
    ConeF cone;
    const double tk[4] = {0.0, 0.5, 0.75, 1.0};
#pragma unroll
    for (int p = 0; p < 3; ++p) {
        const double t0 = tk[p], t1 = tk[p + 1];
        cone.g[p] = make_segf(s, sx + t0 * (cx - sx), sy + t0 * (cy - sy), sz + t0 * (cz - sz), sx + t1 * (cx - sx),
                              sy + t1 * (cy - sy), sz + t1 * (cz - sz));
        cone.R[p] = static_cast<float>(t1 * r * 1.0001 + 1e-6);
    }
    const int L = coop_collect_cone<RES>(ctx, cone, sf, cbuf, batches);
    __syncwarp();   // the list's stores are read back by every lane
    return L;
}

// The SCAN of visible_intervals// The SCAN of visible_intervals (src/vistable.cpp:175-176: col_vis(i / 64) for
// the 65 columns) with the columns spread over the lanes: lane l owns column
// 32 * pass + l. col_vis is an OR over its <= 7 transverse samples, so the
// per-column verdict does not depend on the order the samples are decided in:
// every lane first drops the samples the warp's last blocker already blocks
// (fp32 SAT + exact test), then the warp sweeps ONE pending sample at a time
// (coop_any_hit) — a clear sample makes its column visible, a blocker found is
// immediately tested on every lane's pending sample (a hidden face's columns
// are mostly blocked by the same few faces). Same arithmetic per sightline as
// col_vis_warp, so the 65 verdicts are identical. stop_at_first: return after
// the first visible column (presence mode).
template <int MAXV, int RES>
__device__ __noinline__ unsigned long long scan_cols_warp(const DevScene& s, const SweepCtx& ctx, const double* us,
                                                          int nv, int pl, double ax, double ay, double dx, double dy,
                                                          double sx, double sy, double sz, int sf, unsigned char* sv,
                                                          WCache& cache, bool stop_at_first, bool& vis64,
                                                          unsigned long long& tests, unsigned long long& queries,
                                                          unsigned long long& batches, int f, ConeBuf cbuf,
                                                          int& coneL) {
    constexpr int STRIDE = RecLayout<MAXV>::kStride;
    const int lane = threadIdx.x & 31;
    unsigned long long vis = 0;
    vis64 = false;
    for (int pass = 0; pass < 3; ++pass) {
        const int col = 32 * pass + lane;
        double cs0 = 0, cs1 = 0, inset = 0, px = 0, py = 0;
        bool pending = col < 65 && column_span_us(us, nv, __ddiv_rn(static_cast<double>(col), 64.0), cs0, cs1);
        if (pending) {
            const double cu = __ddiv_rn(static_cast<double>(col), 64.0);   // in [0, 1]: std::clamp is the identity
            inset = dmul(dsub(cs1, cs0), 1e-6);
            px = dadd(ax, dmul(dx, cu));
            py = dadd(ay, dmul(dy, cu));
        }
        int j = 0;
        double qx = 0, qy = 0, qz = 0;
        auto point = [&]() {
            const double v = dmin_std(dsub(cs1, inset),
                                      dmax_std(dadd(cs0, inset), dadd(cs0, dmul(dsub(cs1, cs0), kSampFrac[j]))));
            if (pl == 0) { qx = px; qy = py; qz = v; }
            else if (pl == 1) { qx = v; qy = px; qz = py; }
            else { qx = px; qy = v; qz = py; }
            ++queries;
        };
        if (pending) point();
        // advance this lane's column over the samples occluder k (Morton index)
        // blocks (warp-uniform k: the lanes test one record in lockstep — a
        // per-lane walk over the whole cache was measured slower, divergent)
        auto settle = [&](int k) {
            while (pending && k4w_blocked<MAXV, RES>(s, ctx, k, sx, sy, sz, qx, qy, qz, tests)) {
                if (++j == 7) pending = false;   // every sample blocked: column hidden
                else point();
            }
        };
        for (int i = 0; i < VISRT_K4W_WC; ++i) {   // the warp cache, most recent first
            const int k = cache.entry(i);
            if (k >= 0 && k != sf) settle(k);
        }
        bool visible = false;
        // cone mode: every pending sample of the pass against the task's cone
        // list (build_cone) — the same verdicts as sweeping the whole scene
        auto cone_scan = [&]() {
            const int Lc = coneL;
            if (Lc == 0) {
                if (pending) visible = true;
                pending = false;
                return;
            }
            SegF g{};
            if (pending) g = make_segf(s, sx, sy, sz, qx, qy, qz);
            int left = Lc, c = 0;
            float4 n0 = cbuf.at(0)[0], n1 = cbuf.at(0)[1];   // entry c, loaded one iteration ahead
            while (__any_sync(kFull, pending)) {
                if (stop_at_first && __any_sync(kFull, visible)) break;
                K4P(15, 1);
                const float4 b0 = n0, b1 = n1;
                const int cn = c + 1 == Lc ? 0 : c + 1;
                const float4* E = cbuf.at(cn);
                n0 = E[0];
                n1 = E[1];
                if (pending) {
                    // entry c against this lane's sample, and against the next
                    // samples of the column while it blocks them (a blocker of
                    // one sample mostly blocks its neighbours)
                    bool blk_any = false;
                    const double* R = s.srec + static_cast<size_t>(__float_as_int(b0.w)) * STRIDE;
                    while (pending && sat_maybe4(b0, b1, g) && (++tests, k4w_exact<MAXV>(R, sx, sy, sz, qx, qy, qz))) {
                        blk_any = true;
                        if (++j == 7) {
                            pending = false;   // every sample blocked: column hidden
                        } else {
                            point();
                            g = make_segf(s, sx, sy, sz, qx, qy, qz);
                        }
                    }
                    if (pending) {
                        left = blk_any ? Lc - 1 : left - 1;   // a new sample has passed entry c already
                        if (left == 0) {   // clear of every face of the cone
                            visible = true;
                            pending = false;
                        }
                    }
                }
                c = cn;
            }
        };
        for (;;) {
            if (coneL >= 0) {
                { const long long c0_ = K4CLK(); cone_scan(); K4P(20, K4CLK() - c0_); }
                break;
            }
            const unsigned who = __ballot_sync(kFull, pending);
            if (!who) break;
            const int L = __ffs(who) - 1;
            const double bx = __shfl_sync(kFull, qx, L), by = __shfl_sync(kFull, qy, L),
                         bz = __shfl_sync(kFull, qz, L);
#if VISRT_K4W_NI
            const long long w0_ = K4CLK();
            const int h = k4w_sweep<MAXV, RES>(s, ctx, sx, sy, sz, bx, by, bz, sf, sv, tests, batches);
#else
            const int h = coop_any_hit<MAXV, 0, RES>(ctx, s.srec, make_segf(s, sx, sy, sz, bx, by, bz), sx, sy, sz, bx, by, bz,
                                             sf, -1, sf, sv, tests, batches);
#endif
            K4P(2, 1);
            K4P(21, K4CLK() - w0_);
            if (h < 0) K4P(3, 1);
            if (h < 0) {   // a clear sample: column L is visible
                if (lane == L) {
                    visible = true;
                    pending = false;
                }
                if (stop_at_first) break;
                // a (partly) visible face: its remaining samples are mostly clear
                // and a clear sweep visits every candidate along the segment —
                // decide them against the face's cone list instead
                if (coneL == kConeUnbuilt && cbuf.cap > 0) {
                    const long long b0_ = K4CLK();
                    coneL = build_cone<MAXV, RES>(s, ctx, f, sx, sy, sz, sf, cbuf, batches);
                    K4P(19, K4CLK() - b0_);
                    K4P(12, 1);
                    K4P(13, coneL < 0 ? 1 : 0);
                    K4P(14, coneL < 0 ? 0 : coneL);
                }
            } else {
                cache.put(h);
                if (lane == L) {   // the sweep proved this sample blocked
                    if (++j == 7) pending = false;
                    else point();
                }
                settle(h);
            }
        }
        const unsigned vb = __ballot_sync(kFull, visible);
        if (pass < 2) vis |= static_cast<unsigned long long>(vb) << (32 * pass);
        else vis64 = (vb & 1u) != 0;
        if (stop_at_first && (vis || vis64)) break;
    }
    return vis;
}

#ifndef VISRT_K4W_MINB
#define VISRT_K4W_MINB 2
#endif
#ifndef VISRT_K4R_MINB
#define VISRT_K4R_MINB 2   // CTAs per SM the refine kernel's register budget targets
#endif
// face_param of face f in working plane pl (src/vistable.cpp:84-98): the
// projected segment a + u d and the (u, s) ring us[]; false = no face_param.
template <int MAXV>
__device__ __forceinline__ bool plane_param(const DevScene& s, int f, int nv, int pl, double& ax, double& ay,
                                            double& dx, double& dy, double* us) {
    if (!s.seg_ok[3 * f + pl]) return false;
    const double* sg = s.seg + (static_cast<size_t>(f) * 3 + pl) * 6;
    ax = sg[0];
    ay = sg[1];
    dx = dsub(sg[2], sg[0]);
    dy = dsub(sg[3], sg[1]);
    const double len2 = dadd(dmul(dx, dx), dmul(dy, dy));
    if (len2 <= kEps * kEps) return false;
#pragma unroll 1
    for (int q = 0; q < nv; ++q) face_us(s, f, pl, q, ax, ay, dx, dy, len2, us[2 * q], us[2 * q + 1]);
    return true;
}

// K4w runs in two kernels so that each one's hot code stays small (ncu put
// 41 % of the single kernel's warp samples on stall_no_instruction: its
// 136 KB of code thrashed the instruction caches while warps sat in
// different phases):
//   k_point_regions_warp: back-face test + the 65-column scan of every plane
//     (present / has final; a plane whose 65 columns are all visible gets
//     sub = [0, 1] at once); planes with interior run boundaries are
//     DEFERRED: their column masks go to a RefineTask;
//   k_region_refine: warp per RefineTask — the run boundaries' bisections
//     (refine_fan over the face's cone list, else per-sightline sweeps) and
//     the first-largest interval -> sub / clipped of the deferred planes.
struct RefineTask {
    long long out;              // region record
    long long k;                // source
    int f, planes;              // face, deferred-plane bits
    unsigned long long vis[3];  // columns 0..63 per plane
    int vis64;                  // column 64 per plane (bits)
    int pad;
};

template <int MAXV, int RES, int NT = kThreads, int MINB = VISRT_K4W_MINB>
__global__ void __launch_bounds__(NT, MINB) k_point_regions_warp(RegionArgs a) {
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t bar[1];
    __shared__ unsigned char surv_buf[NT / 32][64];
    const DevScene& s = a.s;
    const int n = s.n;
    const int lane = threadIdx.x & 31;
    const SweepCtx ctx = sweep_setup<RES>(s, smem, bar);
    unsigned char* sv = surv_buf[threadIdx.x >> 5];
    ConeBuf cbuf;   // this warp's cone list
    cbuf.cap = a.cone_buf ? a.cone_cap : 0;
    cbuf.g = a.cone_buf ? a.cone_buf + static_cast<size_t>((blockIdx.x * NT + threadIdx.x) >> 5) * 2 * a.cone_cap
                        : nullptr;
    unsigned long long tests = 0, queries = 0, batches = 0;
    WCache cache;   // the last blockers (Morton indices)
#ifdef VISRT_K4W_PROF
    if (threadIdx.x < 24) k4w_sprof[threadIdx.x] = 0;
    __syncthreads();
#endif
    long long tnext = 0, tend = 0;
    for (;;) {
        if (tnext == tend) {   // a.chunk consecutive tasks (region_task: walk order a.face_major)
            unsigned long long tw = 0;
            if (lane == 0) tw = atomicAdd(&a.counter[0], static_cast<unsigned long long>(a.chunk));
            tnext = static_cast<long long>(__shfl_sync(kFull, tw, 0));
            if (tnext >= a.ntasks) break;
            tend = min(tnext + a.chunk, a.ntasks);
        }
        const long long t = tnext++;
        const RegionTask rt = region_task(a, t, n);
        const long long k = rt.k, li = rt.li;
        const int f = rt.f;
        const int sf = s.inv[f];
        const int nv = s.nv[f];
        const double sx = a.src[3 * k], sy = a.src[3 * k + 1], sz = a.src[3 * k + 2];
        const bool presence = a.presence_only ||
                              (a.presence_of && a.task_face &&
                               a.presence_of[a.paired ? t : li]);
        const long long tclk0 = K4CLK();
        int8_t present = 1;
        int8_t has[3] = {0, 0, 0};
        int deferred = 0, dv64 = 0;
        unsigned long long dvis[3] = {0, 0, 0};
        int coneL = kConeUnbuilt;   // this task's cone list: built at its first clear sample
        // back-face test (src/vistable.cpp:289-294)
        {
            const double* P = s.pts + static_cast<size_t>(f) * VISRT_MAX_VERTS * 3;
            const double* N = s.normal + 3 * static_cast<size_t>(f);
            const double dist = dot_rel(sx, sy, sz, P[0], P[1], P[2], N[0], N[1], N[2]);
            if (fabs(dist) <= kEps) present = -1;
            else if (dist < 0.0) present = 0;
        }
        if (present == 1) K4P(9, 1);
#pragma unroll 1
        for (int pl = 0; pl < 3 && present == 1; ++pl) {
            double ax, ay, dx, dy, us[2 * MAXV];
            if (!plane_param<MAXV>(s, f, nv, pl, ax, ay, dx, dy, us)) continue;
            // SCAN (src/vistable.cpp:175-176); presence: stop at the first visible column
            bool vis64 = false;
            const long long sclk0 = K4CLK();
            const unsigned long long vis = scan_cols_warp<MAXV, RES>(s, ctx, us, nv, pl, ax, ay, dx, dy, sx, sy, sz, sf,
                                                                     sv, cache, presence, vis64, tests, queries,
                                                                     batches, f, cbuf, coneL);
            K4P(0, K4CLK() - sclk0);
            if (vis == 0ull && !vis64) {
                present = 0;   // fully hidden in this plane: no region
                break;
            }
            has[pl] = 1;
            if (!presence && !(vis == ~0ull && vis64)) {   // interior run boundaries: k_region_refine
                deferred |= 1 << pl;
                dvis[pl] = vis;
                dv64 |= static_cast<int>(vis64) << pl;
            }
        }
        if (present == 1 && !(has[0] | has[1] | has[2])) present = 0;
        K4P(8, K4CLK() - tclk0);
        if (present == 1) {
            K4P(10, K4CLK() - tclk0);
            K4P(11, 1);
        }
        if (lane == 0) {
            visrt_region r;
            r.present = present;
            r.pad = 0;
            for (int q = 0; q < 3; ++q) {
                r.has[q] = present == 1 ? has[q] : 0;
                r.clipped[q] = 0;   // a plane with every column visible: [0, 1], not clipped
                const bool full = present == 1 && has[q] && !presence && !((deferred >> q) & 1);
                r.sub[2 * q] = 0.0;
                r.sub[2 * q + 1] = full ? 1.0 : 0.0;
            }
            a.out[rt.out] = r;
            if (present == 1 && deferred) {
                // tasks whose cone list overflowed refine by per-sightline sweeps
                // (~30x dearer): listed from the END of the buffer so the refine
                // kernel starts them first (no long tail behind cheap tasks)
                const bool heavy = coneL == -1;
                const unsigned long long slot =
                    heavy ? static_cast<unsigned long long>(a.ntasks) - 1ull - atomicAdd(a.refine_count + 2, 1ull)
                          : atomicAdd(a.refine_count, 1ull);
                RefineTask q;
                q.out = rt.out;
                q.k = k;
                q.f = f;
                q.planes = deferred;
                q.vis[0] = dvis[0];
                q.vis[1] = dvis[1];
                q.vis[2] = dvis[2];
                q.vis64 = dv64;
                q.pad = 0;
                reinterpret_cast<RefineTask*>(a.refine_tasks)[slot] = q;
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        tests += __shfl_down_sync(kFull, tests, o);
        queries += __shfl_down_sync(kFull, queries, o);
    }
    if (lane == 0) {
        atomicAdd(&a.counter[1], tests);
        atomicAdd(&a.counter[2], queries);
    }
#ifdef VISRT_K4W_PROF
    __syncthreads();
    if (threadIdx.x < 24) atomicAdd(&g_k4w_prof[threadIdx.x], k4w_sprof[threadIdx.x]);
#endif
}

// The deferred planes of k_point_regions_warp: refine every interior run
// boundary (src/vistable.cpp:163-172) and take the first largest interval
// (175-192), warp per RefineTask.
template <int MAXV, int RES, int NT = kThreads, int MINB = VISRT_K4W_MINB>
__global__ void __launch_bounds__(NT, MINB) k_region_refine(RegionArgs a) {
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t bar[1];
    __shared__ unsigned char surv_buf[NT / 32][64];
    __shared__ int fan_buf[NT / 32][7 * kFanCap];   // per warp: refine_fan candidate lists
    const DevScene& s = a.s;
    const int lane = threadIdx.x & 31;
    const SweepCtx ctx = sweep_setup<RES>(s, smem, bar);
    int* fan = fan_buf[threadIdx.x >> 5];
    unsigned char* sv = surv_buf[threadIdx.x >> 5];
    ConeBuf cbuf;
    cbuf.cap = a.cone_buf ? a.cone_cap : 0;
    cbuf.g = a.cone_buf ? a.cone_buf + static_cast<size_t>((blockIdx.x * NT + threadIdx.x) >> 5) * 2 * a.cone_cap
                        : nullptr;
    unsigned long long tests = 0, queries = 0, batches = 0;
    WCache cache;
#ifdef VISRT_K4W_PROF
    if (threadIdx.x < 24) k4w_sprof[threadIdx.x] = 0;
    __syncthreads();
#endif
    const long long nheavy = static_cast<long long>(a.refine_count[2]);
    const long long ntask = static_cast<long long>(a.refine_count[0]) + nheavy;
    const RefineTask* tasks = reinterpret_cast<const RefineTask*>(a.refine_tasks);
    for (;;) {
        unsigned long long tw = 0;
        if (lane == 0) tw = atomicAdd(a.refine_count + 1, 1ull);
        const long long qi = static_cast<long long>(__shfl_sync(kFull, tw, 0));
        if (qi >= ntask) break;
        const RefineTask q = tasks[qi < nheavy ? a.ntasks - 1 - qi : qi - nheavy];   // heavy (buffer end) first
        const int f = q.f;
        const int sf = s.inv[f];
        const int nv = s.nv[f];
        const double sx = a.src[3 * q.k], sy = a.src[3 * q.k + 1], sz = a.src[3 * q.k + 2];
        int coneL = kConeUnbuilt;
        if (a.fan && cbuf.cap > 0) coneL = build_cone<MAXV, RES>(s, ctx, f, sx, sy, sz, sf, cbuf, batches);
        double sub[6];
        int8_t clp[3];
#pragma unroll 1
        for (int pl = 0; pl < 3; ++pl) {
            if (!((q.planes >> pl) & 1)) continue;
            double ax, ay, dx, dy, us[2 * MAXV];
            plane_param<MAXV>(s, f, nv, pl, ax, ay, dx, dy, us);
            const unsigned long long vis = q.vis[pl];
            const bool vis64 = (q.vis64 >> pl) & 1;
            auto V = [&](int i) { return i == 64 ? vis64 : ((vis >> i) & 1ull) != 0; };
            auto refine = [&](double lo, double hi, bool lo_vis) {
                if (a.fan == 2) return lo;   // development aid (VISRT_K4W_FAN=2): time the scan alone, regions WRONG
                const long long rclk0 = K4CLK();
                int it = 0;
                if (VISRT_K4W_FAN && a.fan &&
                    refine_fan<MAXV, RES>(s, ctx, us, nv, pl, ax, ay, dx, dy, lo, hi, lo_vis, sx, sy, sz, sf, fan,
                                          tests, queries, batches, it, cbuf, coneL)) {
                    K4P(1, K4CLK() - rclk0);
                    K4P(6, 1);
                    K4P(7, it);
                    return dmul(0.5, dadd(lo, hi));
                }
                for (; it < 50 && dsub(hi, lo) > 1e-15; ++it) {   // col_vis per midpoint (per-sightline sweeps)
                    const double mid = dmul(0.5, dadd(lo, hi));
                    if (col_vis_warp<MAXV, RES>(s, ctx, us, nv, pl, ax, ay, dx, dy, mid, sx, sy, sz, sf, sv, cache,
                                                tests, queries, batches) == lo_vis)
                        lo = mid;
                    else
                        hi = mid;
                }
                K4P(1, K4CLK() - rclk0);
                K4P(6, 1);
                K4P(7, it);
                return dmul(0.5, dadd(lo, hi));
            };
            const double step = __ddiv_rn(1.0, 64.0);
            bool have = false;
            double b0 = 0, b1 = 0;
            int i = 0;
            while (i < 65) {   // runs (src/vistable.cpp:175-192)
                if (!V(i)) {
                    ++i;
                    continue;
                }
                double start = __ddiv_rn(static_cast<double>(i), 64.0);
                int j = i;
                while (j + 1 < 65 && V(j + 1)) ++j;
                double end = __ddiv_rn(static_cast<double>(j), 64.0);
                // the run's interior boundaries, start then end (one refine call site: i-cache)
#pragma unroll 1
                for (int side = 0; side < 2; ++side) {
                    if (side == 0 ? i == 0 : j + 1 == 65) continue;
                    const double r = refine(side == 0 ? dsub(start, step) : end, side == 0 ? start : dadd(end, step),
                                            side == 1);
                    if (side == 0) start = r;
                    else end = r;
                }
                if (!have || dsub(b1, b0) < dsub(end, start)) {   // std::max_element: first largest
                    b0 = start;
                    b1 = end;
                    have = true;
                }
                i = j + 1;
            }
            sub[2 * pl] = b0;
            sub[2 * pl + 1] = b1;
            clp[pl] = (b0 > 1e-9 || b1 < 1.0 - 1e-9) ? 1 : 0;
        }
        if (lane == 0) {
            visrt_region* r = a.out + q.out;
#pragma unroll
            for (int pl = 0; pl < 3; ++pl)
                if ((q.planes >> pl) & 1) {
                    r->sub[2 * pl] = sub[2 * pl];
                    r->sub[2 * pl + 1] = sub[2 * pl + 1];
                    r->clipped[pl] = clp[pl];
                }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        tests += __shfl_down_sync(kFull, tests, o);
        queries += __shfl_down_sync(kFull, queries, o);
    }
    if (lane == 0) {
        atomicAdd(&a.counter[1], tests);
        atomicAdd(&a.counter[2], queries);
    }
#ifdef VISRT_K4W_PROF
    __syncthreads();
    if (threadIdx.x < 24) atomicAdd(&g_k4w_prof[threadIdx.x], k4w_sprof[threadIdx.x]);
#endif
}

#ifdef VISRT_K4W_PROF
}  // namespace visrt
extern "C" int visrt_debug_k4w_prof(unsigned long long* out) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, visrt::g_k4w_prof, sizeof(visrt::g_k4w_prof));
    static const unsigned long long zero[24] = {};
    return static_cast<int>(cudaMemcpyToSymbol(visrt::g_k4w_prof, zero, sizeof(zero)));
}
namespace visrt {
#endif

static int persistent_grid_r(const void* fn, size_t smem, int device, int threads = kThreads) {
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, smem);
    if (per < 1) per = 1;
    return sms * per;
}

// K4w cone-list capacity per warp (VISRT_K4W_CONE, entries of 32 B; 0 = no cone lists)
static int cone_cap_r() {
    static const int c = [] {
        const char* e = std::getenv("VISRT_K4W_CONE");
        return e ? std::max(0, std::atoi(e)) : 1024;
    }();
    return c;
}
// per-launch scratch (cone lists, refine tasks): stream-ordered allocations
// from the device's default pool (capi.cu pool_setup keeps freed blocks), so
// no allocation synchronises the device inside a caller's timed region
static void* region_scratch_alloc(size_t bytes, cudaStream_t st) {
    void* p = nullptr;
    return cudaMallocAsync(&p, bytes, st) == cudaSuccess ? p : nullptr;
}
static void region_scratch_release(void* p, cudaStream_t st) { cudaFreeAsync(p, st); }

template <class K>
static cudaError_t launch_r(K fn, size_t smem, const RegionArgs& a0, int device, cudaStream_t st,
                            int threads = kThreads, bool cone = false) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    RegionArgs a = a0;
    if (cone && cone_cap_r() > 0 && !a.presence_only) a.cone_cap = cone_cap_r();
    const int grid = persistent_grid_r(reinterpret_cast<const void*>(fn), smem, device, threads);
    void* cb = nullptr;
    if (a.cone_cap > 0) {
        cb = region_scratch_alloc(static_cast<size_t>(grid) * (threads / 32) * a.cone_cap * 32, st);
        if (!cb) return cudaErrorMemoryAllocation;
        a.cone_buf = static_cast<float4*>(cb);
    }
    fn<<<grid, threads, smem, st>>>(a);
    e = cudaGetLastError();
    if (cb) region_scratch_release(cb, st);
    return e;
}

// K4w threads per QUANTISED CTA (one CTA per SM: 16 warps at 128 registers)
constexpr int kQThreadsK4 = 512;

static int quant_mode_r() {
    static const int m = [] {
        const char* e = std::getenv("VISRT_QUANT");
        return e ? std::atoi(e) : 0;   // off by default: measured slower
    }();
    return m;
}

template <int MAXV>
static cudaError_t launch_regions_t(const RegionArgs& a0, int device, cudaStream_t st) {
    RegionArgs a = a0;
    {   // K4w task grabs: VISRT_K4W_CHUNK consecutive tasks, fewer when that leaves < 8 grabs per warp
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        const long long warps = static_cast<long long>(sms) * 2 * (kThreads / 32);
        // resident scenes take 4 consecutive tasks per grab (one face, 4 neighbouring snapshots: the
        // warp cache stays warm; r02, config 3 2,000 x 2,756 regions: 1 -> 116.5 ms, 2 -> 111.3, 4 -> 109.4,
        // 8 -> 109.3, 16 -> 110.9); the streamed big scenes keep 1 (config 5, 500 snapshots: 1 -> 412 ms,
        // 2 -> 423, 4 -> 442, 8 -> 463: heavy faces cluster and the tail grows)
        const int want = a.s.n > kResidentMaxBoxes ? VISRT_K4W_CHUNK : 4 * VISRT_K4W_CHUNK;
        a.chunk = static_cast<int>(std::max<long long>(1, std::min<long long>(want, a.ntasks / (8 * warps))));
    }
    const char* e = std::getenv("VISRT_FORCE_STREAM");
    const bool res = !(e && e[0] == '1') && a.s.n <= kResidentMaxBoxes;
    const size_t smem = sweep_smem_bytes(a.s.n, a.s.ntiles, res);
    // K4w for latency-bound launches (fewer tasks than ~2x the resident lanes:
    // small snapshot batches, trajectory probes), K4 lanes for throughput.
    // VISRT_K4_WARP=0/1 forces either kernel.
    static const int force = [] {
        const char* w = std::getenv("VISRT_K4_WARP");
        return w ? (w[0] == '1' ? 1 : 0) : -1;
    }();
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const bool warp = a.presence_only || a.presence_of || (force >= 0 ? force == 1 : true);   // K4w: faster at every size
    static const int face_major = [] {
        const char* e = std::getenv("VISRT_K4W_FACEMAJOR");
        return e && e[0] == '0' ? 0 : 1;
    }();
    a.face_major = warp ? face_major : 0;   // the lane kernel K4 walks source-major
    static const int fan = [] {   // VISRT_K4W_FAN=0: refine by per-sightline sweeps (A/B and tests)
        const char* e = std::getenv("VISRT_K4W_FAN");
        return e && e[0] == '0' ? 0 : (e && e[0] == '2' ? 2 : 1);
    }();
    a.fan = fan;
    if (warp && quant_mode_r() != 0 && a.s.n <= kQuantisedMaxBoxes && (quant_mode_r() == 2 || !res)) {
        int smem_sm = 0;
        cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
        const size_t qsm = sweep_smem_bytes(a.s.n, a.s.ntiles, kQuantised);
        if (qsm + (kQThreadsK4 / 32) * 64 + 1024 <= static_cast<size_t>(smem_sm)) {
            void* rt = nullptr;
            if (!a.presence_only) {
                rt = region_scratch_alloc(64 + static_cast<size_t>(a.ntasks) * sizeof(RefineTask), st);
                if (!rt) return cudaErrorMemoryAllocation;
                a.refine_count = static_cast<unsigned long long*>(rt);
                a.refine_tasks = static_cast<char*>(rt) + 64;
                cudaError_t e2 = cudaMemsetAsync(rt, 0, 64, st);
                if (e2 != cudaSuccess) return e2;
            }
            cudaError_t e1 =
                launch_r(k_point_regions_warp<MAXV, kQuantised, kQThreadsK4, 1>, qsm, a, device, st, kQThreadsK4);
            if (e1 == cudaSuccess && rt)
                e1 = launch_r(k_region_refine<MAXV, kQuantised, kQThreadsK4, 1>, qsm, a, device, st, kQThreadsK4);
            if (rt) region_scratch_release(rt, st);
            return e1;
        }
    }
    if (warp) {
        // scan kernel, then the refine kernel over the deferred planes it listed
        void* rt = nullptr;
        if (!a.presence_only) {
            const size_t bytes = 64 + static_cast<size_t>(a.ntasks) * sizeof(RefineTask);
            rt = region_scratch_alloc(bytes, st);
            if (!rt) return cudaErrorMemoryAllocation;
            a.refine_count = static_cast<unsigned long long*>(rt);
            a.refine_tasks = static_cast<char*>(rt) + 64;
            cudaError_t e2 = cudaMemsetAsync(rt, 0, 64, st);
            if (e2 != cudaSuccess) return e2;
        }
        cudaError_t e1 = res ? launch_r(k_point_regions_warp<MAXV, kResident>, smem, a, device, st, kThreads, true)
                             : launch_r(k_point_regions_warp<MAXV, kStreamed>, smem, a, device, st, kThreads, true);
        if (e1 == cudaSuccess && rt)
            e1 = res ? launch_r(k_region_refine<MAXV, kResident, kThreads, VISRT_K4R_MINB>, smem, a, device, st, kThreads,
                                true)
                     : launch_r(k_region_refine<MAXV, kStreamed, kThreads, VISRT_K4R_MINB>, smem, a, device, st, kThreads,
                                true);
        if (rt) region_scratch_release(rt, st);
        return e1;
    }
    return res ? launch_r(k_point_regions<MAXV, true>, smem, a, device, st)
               : launch_r(k_point_regions<MAXV, false>, smem, a, device, st);
}

cudaError_t launch_point_regions(const RegionArgs& a, int device, cudaStream_t st) {
    return a.s.maxv <= 4 ? launch_regions_t<4>(a, device, st) : launch_regions_t<8>(a, device, st);
}

// ---------------------------------------------------------------------------
// K5: TableBuilder::reach for matrix entries of order 1 / 2 (beam cascade).
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(256) k_beam_rows(BeamArgs a) {
    const DevScene& s = a.s;
    const long long total = a.paired ? a.nent : a.nsrc * a.nent;
    for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long k = a.paired ? t : t / a.nent;
        const long long e = a.paired ? t : t - k * a.nent;
        const visrt_entry E = a.ent[e];
        const int head = E.chain[0];
        const size_t ri = a.paired ? static_cast<size_t>(t)
                        : a.slot ? static_cast<size_t>(k) * a.rstride + a.slot[head]
                                 : static_cast<size_t>(k) * s.n + head;
        const visrt_region& R = a.regions[ri];
        bool row = false, full = false;
        if (R.present == 1) {
            // BeamState after the head (src/vistable.cpp:409-421): per plane the
            // region's window and Full flag; image = source mirrored by the head
            double wx0[3], wy0[3], wx1[3], wy1[3];
            bool hw[3], fl[3];
            for (int pl = 0; pl < 3; ++pl) {
                hw[pl] = R.has[pl] != 0;
                fl[pl] = hw[pl] && !R.clipped[pl];
                wx0[pl] = wy0[pl] = wx1[pl] = wy1[pl] = 0.0;
                if (hw[pl]) {
                    const double* fs = s.seg + (static_cast<size_t>(head) * 3 + pl) * 6;
                    const double dx = dsub(fs[2], fs[0]), dy = dsub(fs[3], fs[1]);
                    wx0[pl] = dadd(fs[0], dmul(dx, R.sub[2 * pl]));
                    wy0[pl] = dadd(fs[1], dmul(dy, R.sub[2 * pl]));
                    wx1[pl] = dadd(fs[0], dmul(dx, R.sub[2 * pl + 1]));
                    wy1[pl] = dadd(fs[1], dmul(dy, R.sub[2 * pl + 1]));
                }
            }
            double ix, iy, iz;
            {
                const double* P = s.pts + static_cast<size_t>(head) * VISRT_MAX_VERTS * 3;
                const double* N = s.normal + 3 * static_cast<size_t>(head);
                const double sx = a.src[3 * k], sy = a.src[3 * k + 1], sz = a.src[3 * k + 2];
                const double d2 = dmul(2.0, dot_rel(sx, sy, sz, P[0], P[1], P[2], N[0], N[1], N[2]));
                ix = dsub(sx, dmul(N[0], d2));   // mirror_point
                iy = dsub(sy, dmul(N[1], d2));
                iz = dsub(sz, dmul(N[2], d2));
            }
            bool ok = true;
            // TableBuilder::step along the reflector chain (src/vistable.cpp:432-467)
            for (int c = 1; c < E.order && ok; ++c) {
                const int from = E.chain[c - 1], to = E.chain[c];
                double nx0[3], ny0[3], nx1[3], ny1[3];
                bool nh[3] = {false, false, false}, nf[3] = {false, false, false};
                bool any = false;
                for (int pl = 0; pl < 3; ++pl) {
                    nx0[pl] = ny0[pl] = nx1[pl] = ny1[pl] = 0.0;
                    if (!s.seg_ok[3 * from + pl] || !s.seg_ok[3 * to + pl]) continue;
                    const double* fs = s.seg + (static_cast<size_t>(from) * 3 + pl) * 6;
                    const double* gs = s.seg + (static_cast<size_t>(to) * 3 + pl) * 6;
                    const double dd = fabs(dadd(dmul(fs[4], gs[4]), dmul(fs[5], gs[5])));
                    if (!(dd >= 1.0 - 1e-9 || dd <= 1e-9)) continue;   // required_planes(from, to)
                    // the window in this plane, or the whole face when never constrained
                    const double w0x = hw[pl] ? wx0[pl] : fs[0], w0y = hw[pl] ? wy0[pl] : fs[1];
                    const double w1x = hw[pl] ? wx1[pl] : fs[2], w1y = hw[pl] ? wy1[pl] : fs[3];
                    const bool was_full = hw[pl] ? fl[pl] : true;
                    double apx, apy;
                    proj(pl, ix, iy, iz, apx, apy);
                    const Cov cv = beam_coverage(apx, apy, w0x, w0y, w1x, w1y, fs[4], fs[5], gs[0], gs[1], gs[2], gs[3]);
                    if (cv.verdict == 2) {
                        ok = false;
                        break;
                    }
                    const double qx = dsub(gs[2], gs[0]), qy = dsub(gs[3], gs[1]);
                    nx0[pl] = dadd(gs[0], dmul(qx, cv.lo));
                    ny0[pl] = dadd(gs[1], dmul(qy, cv.lo));
                    nx1[pl] = dadd(gs[0], dmul(qx, cv.hi));
                    ny1[pl] = dadd(gs[1], dmul(qy, cv.hi));
                    nh[pl] = true;
                    nf[pl] = was_full && cv.verdict == 0;
                    any = true;
                }
                if (!ok || !any) {
                    ok = false;
                    break;
                }
                for (int pl = 0; pl < 3; ++pl) {
                    hw[pl] = nh[pl];
                    fl[pl] = nf[pl];
                    wx0[pl] = nx0[pl];
                    wy0[pl] = ny0[pl];
                    wx1[pl] = nx1[pl];
                    wy1[pl] = ny1[pl];
                }
                // image3 mirrored through the new tail face
                const double* P = s.pts + static_cast<size_t>(to) * VISRT_MAX_VERTS * 3;
                const double* N = s.normal + 3 * static_cast<size_t>(to);
                const double d2 = dmul(2.0, dot_rel(ix, iy, iz, P[0], P[1], P[2], N[0], N[1], N[2]));
                ix = dsub(ix, dmul(N[0], d2));
                iy = dsub(iy, dmul(N[1], d2));
                iz = dsub(iz, dmul(N[2], d2));
            }
            row = ok;
            full = ok && hw[E.plane] && fl[E.plane];
        }
        const size_t w = (a.paired ? 0 : static_cast<size_t>(k) * a.words) + static_cast<size_t>(e >> 5);
        if (row) atomicOr(a.row_bits + w, 1u << (e & 31));
        if (full) atomicOr(a.full_bits + w, 1u << (e & 31));
    }
}

// Batched sightline_clear: lane per segment, culled any-hit sweep, no face skipped.
template <int MAXV, bool RESIDENT>
__global__ void __launch_bounds__(kThreads, 3) k_segments_clear(DevScene s, long long nseg, const double* A,
                                                                const double* B, uint8_t* clear,
                                                                unsigned long long* counter) {
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t bar[1];
    __shared__ int slots[kThreads];
    const int lane = threadIdx.x & 31;
    int* slot = slots + (threadIdx.x & ~31);
    const SweepCtx ctx = sweep_setup<RESIDENT>(s, smem, bar);
    bool active = false, exhausted = false;
    long long id = 0;
    double ax = 0, ay = 0, az = 0, bx = 0, by = 0, bz = 0;
    Sweep sw{};
    unsigned long long tests = 0;
    auto refill = [&]() {
        unsigned need = __ballot_sync(kFull, !active && !exhausted);
        while (need) {
            const int leader = __ffs(need) - 1;
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(&counter[0], static_cast<unsigned long long>(__popc(need)));
            base = __shfl_sync(kFull, base, leader);
            if (!active && !exhausted) {
                const long long my = static_cast<long long>(base) + __popc(need & ((1u << lane) - 1u));
                if (my >= nseg) {
                    exhausted = true;
                } else {
                    id = my;
                    ax = A[3 * my]; ay = A[3 * my + 1]; az = A[3 * my + 2];
                    bx = B[3 * my]; by = B[3 * my + 1]; bz = B[3 * my + 2];
                    sw.start(make_segf(s, ax, ay, az, bx, by, bz), -1, -1, 0, ctx.nchunks);
                    active = true;
                }
            }
            need = __ballot_sync(kFull, !active && !exhausted);
        }
    };
    refill();
    for (;;) {
        unsigned long long mask = 0;
        int base = 0;
        if (active) mask = sweep_batch(sw, ctx, base);
        const int hk = coop_exact<MAXV>(s.srec, mask, base, ax, ay, az, bx, by, bz, slot, tests, 0ull,
                                        [](int, unsigned long long) {});
        if (active) {
            if (hk >= 0) {
                clear[id] = 0;
                active = false;
            } else if (sw.done()) {
                clear[id] = 1;
                active = false;
            }
        }
        refill();
        if (!__any_sync(kFull, active || !exhausted)) break;
    }
    for (int o = 16; o > 0; o >>= 1) tests += __shfl_down_sync(kFull, tests, o);
    if (lane == 0) atomicAdd(&counter[1], tests);
}

// Warp-per-segment variant (coop_any_hit), the default: converged culling and
// exact phases like K2w / K4w.
template <int MAXV, int RES, int NT = kThreads, int MINB = 3>
__global__ void __launch_bounds__(NT, MINB) k_segments_clear_warp(DevScene s, long long nseg, const double* A,
                                                                  const double* B, uint8_t* clear,
                                                                  unsigned long long* counter) {
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t bar[1];
    __shared__ unsigned char surv_buf[NT / 32][64];
    const int lane = threadIdx.x & 31;
    const SweepCtx ctx = sweep_setup<RES>(s, smem, bar);
    unsigned char* sv = surv_buf[threadIdx.x >> 5];
    unsigned long long tests = 0, batches = 0;
    int cache = -1;
    for (;;) {
        unsigned long long qw = 0;
        if (lane == 0) qw = atomicAdd(&counter[0], 1ull);
        const long long q = static_cast<long long>(__shfl_sync(kFull, qw, 0));
        if (q >= nseg) break;
        const double ax = A[3 * q], ay = A[3 * q + 1], az = A[3 * q + 2];
        const double bx = B[3 * q], by = B[3 * q + 1], bz = B[3 * q + 2];
        bool blocked = false;
        if (cache >= 0) {
            tests += lane == 0;
            blocked = seg_hits<MAXV>(s.srec + static_cast<size_t>(cache) * RecLayout<MAXV>::kStride, ax, ay, az, bx,
                                     by, bz);
        }
        if (!blocked) {
            const int h = coop_any_hit<MAXV, 0, RES>(ctx, s.srec, make_segf(s, ax, ay, az, bx, by, bz), ax, ay, az, bx, by,
                                             bz, -1, -1, -1, sv, tests, batches);
            blocked = h >= 0;
            if (blocked) cache = h;
        }
        if (lane == 0) clear[q] = blocked ? 0 : 1;
    }
    for (int o = 16; o > 0; o >>= 1) tests += __shfl_down_sync(kFull, tests, o);
    if (lane == 0) atomicAdd(&counter[1], tests);
}

template <int MAXV>
static cudaError_t launch_segments_t(const DevScene& s, long long nseg, const double* A, const double* B,
                                     uint8_t* clear, unsigned long long* ctr, int device, cudaStream_t st) {
    const char* e = std::getenv("VISRT_FORCE_STREAM");
    const bool res = !(e && e[0] == '1') && s.n <= kResidentMaxBoxes;
    size_t smem = sweep_smem_bytes(s.n, s.ntiles, res);
    int threads = kThreads;
    auto go = [&](auto fn) {
        cudaError_t err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (err != cudaSuccess) return err;
        fn<<<persistent_grid_r(reinterpret_cast<const void*>(fn), smem, device, threads), threads, smem, st>>>(
            s, nseg, A, B, clear, ctr);
        return cudaGetLastError();
    };
    static const bool lane_kernel = [] {
        const char* w = std::getenv("VISRT_SEG_WARP");
        return w && w[0] == '0';
    }();
    if (!lane_kernel && quant_mode_r() != 0 && s.n <= kQuantisedMaxBoxes && (quant_mode_r() == 2 || !res)) {
        int smem_sm = 0;
        cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
        const size_t qsm = sweep_smem_bytes(s.n, s.ntiles, kQuantised);
        if (qsm + (kQThreads / 32) * 64 + 1024 <= static_cast<size_t>(smem_sm)) {
            smem = qsm;
            threads = kQThreads;
            return go(k_segments_clear_warp<MAXV, kQuantised, kQThreads, 1>);
        }
    }
    if (!lane_kernel)
        return res ? go(k_segments_clear_warp<MAXV, kResident>) : go(k_segments_clear_warp<MAXV, kStreamed>);
    return res ? go(k_segments_clear<MAXV, true>) : go(k_segments_clear<MAXV, false>);
}

cudaError_t launch_segments_clear(const DevScene& s, long long nseg, const double* A, const double* B,
                                  uint8_t* clear, unsigned long long* counter, int device, cudaStream_t st) {
    return s.maxv <= 4 ? launch_segments_t<4>(s, nseg, A, B, clear, counter, device, st)
                       : launch_segments_t<8>(s, nseg, A, B, clear, counter, device, st);
}

cudaError_t launch_beam_rows(const BeamArgs& a, cudaStream_t st) {
    const long long work = a.paired ? a.nent : a.nsrc * a.nent;
    if (work <= 0) return cudaSuccess;
    const int blocks = static_cast<int>(std::min<long long>((work + 255) / 256, 148 * 32));
    k_beam_rows<<<blocks, 256, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace visrt

// ---------------------------------------------------------------------------
// C-ABI entry (include/visrt.h)
// ---------------------------------------------------------------------------
#include "capi_internal.h"

extern "C" int visrt_point_regions(visrt_scene* sc, int64_t nsrc, const double* src_xyz, visrt_region* out,
                                   visrt_stats* stats, void* stream) {
    return visrt::capi_guard([&] {
        visrt::ScopedDevice dev(sc);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const visrt::DevScene& ds = visrt::scene_dev(sc);
        const long long ntasks = static_cast<long long>(nsrc) * ds.n;
        std::vector<void*> tmp;
        visrt::FreeGuard guard{tmp};
        double* d_src = visrt::dalloc<double>(static_cast<size_t>(nsrc) * 3, tmp);
        visrt_region* d_out = visrt::dalloc<visrt_region>(static_cast<size_t>(ntasks), tmp);
        unsigned long long* d_ctr = visrt::dalloc<unsigned long long>(4, tmp);
        visrt::ck(cudaMemcpyAsync(d_src, src_xyz, nsrc * 3 * sizeof(double), cudaMemcpyHostToDevice, st), "H2D src");
        visrt::ck(cudaMemsetAsync(d_ctr, 0, 4 * sizeof(unsigned long long), st), "memset");
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
        visrt::RegionArgs a{ds, ntasks, d_src, d_out, d_ctr};
        if (ntasks > 0) visrt::ck(visrt::launch_point_regions(a, visrt::scene_device(sc), st), "k_point_regions");
        cudaEventRecord(e1, st);
        unsigned long long ctr[4] = {0, 0, 0, 0};
        if (ntasks > 0)
            visrt::ck(cudaMemcpyAsync(out, d_out, ntasks * sizeof(visrt_region), cudaMemcpyDeviceToHost, st), "D2H");
        visrt::ck(cudaMemcpyAsync(ctr, d_ctr, sizeof(ctr), cudaMemcpyDeviceToHost, st), "D2H");
        visrt::ck(cudaStreamSynchronize(st), "sync");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (stats) {
            stats->pairs = ntasks;
            stats->candidates = static_cast<int64_t>(ctr[2]);   // sightline queries
            stats->admitted = -1;
            stats->tests_alg = 0;
            stats->tests_exec = static_cast<int64_t>(ctr[1]);
            stats->ms = ms;
        }
    });
}

extern "C" int visrt_point_tables(visrt_scene* sc, int64_t nsrc, const double* src_xyz, int64_t nent,
                                  const visrt_entry* entries, uint32_t* row_bits, uint32_t* full_bits,
                                  visrt_region* regions_out, visrt_stats* stats, void* stream) {
    return visrt::capi_guard([&] {
        visrt::ScopedDevice dev(sc);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const visrt::DevScene& ds = visrt::scene_dev(sc);
        for (int64_t e = 0; e < nent; ++e) {
            if (entries[e].order < 1 || entries[e].order > 4)
                throw visrt::UsageError("point tables cover matrix entries of order 1..4");
            for (int c = 0; c <= entries[e].order; ++c)
                if (entries[e].chain[c] < 0 || entries[e].chain[c] >= ds.n) throw visrt::UsageError("bad face index");
            if (entries[e].plane < 0 || entries[e].plane > 2) throw visrt::UsageError("bad plane tag");
        }
        const long long ntasks = static_cast<long long>(nsrc) * ds.n;
        const int words = static_cast<int>((nent + 31) / 32);
        std::vector<void*> tmp;
        visrt::FreeGuard guard{tmp};
        double* d_src = visrt::dalloc<double>(static_cast<size_t>(nsrc) * 3, tmp);
        visrt_region* d_reg = visrt::dalloc<visrt_region>(static_cast<size_t>(ntasks), tmp);
        visrt_entry* d_ent = visrt::dalloc<visrt_entry>(static_cast<size_t>(nent), tmp);
        uint32_t* d_rows = visrt::dalloc<uint32_t>(static_cast<size_t>(nsrc) * words, tmp);
        uint32_t* d_full = visrt::dalloc<uint32_t>(static_cast<size_t>(nsrc) * words, tmp);
        unsigned long long* d_ctr = visrt::dalloc<unsigned long long>(4, tmp);
        visrt::ck(cudaMemcpyAsync(d_src, src_xyz, nsrc * 3 * sizeof(double), cudaMemcpyHostToDevice, st), "H2D");
        if (nent) visrt::ck(cudaMemcpyAsync(d_ent, entries, nent * sizeof(visrt_entry), cudaMemcpyHostToDevice, st), "H2D");
        visrt::ck(cudaMemsetAsync(d_rows, 0, static_cast<size_t>(nsrc) * words * 4, st), "memset");
        visrt::ck(cudaMemsetAsync(d_full, 0, static_cast<size_t>(nsrc) * words * 4, st), "memset");
        visrt::ck(cudaMemsetAsync(d_ctr, 0, 4 * sizeof(unsigned long long), st), "memset");
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
        visrt::RegionArgs ra{ds, ntasks, d_src, d_reg, d_ctr};
        if (ntasks > 0) visrt::ck(visrt::launch_point_regions(ra, visrt::scene_device(sc), st), "k_point_regions");
        visrt::BeamArgs ba{ds, nsrc, nent, d_src, d_reg, d_ent, d_rows, d_full, words};
        if (nsrc * nent > 0) {
            const long long work = nsrc * nent;
            const int blocks = static_cast<int>(std::min<long long>((work + 255) / 256, 148 * 32));
            visrt::k_beam_rows<<<blocks, 256, 0, st>>>(ba);
            visrt::ck(cudaGetLastError(), "k_beam_rows");
        }
        cudaEventRecord(e1, st);
        if (nsrc * words > 0) {
            visrt::ck(cudaMemcpyAsync(row_bits, d_rows, static_cast<size_t>(nsrc) * words * 4, cudaMemcpyDeviceToHost, st), "D2H");
            visrt::ck(cudaMemcpyAsync(full_bits, d_full, static_cast<size_t>(nsrc) * words * 4, cudaMemcpyDeviceToHost, st), "D2H");
        }
        if (regions_out && ntasks > 0)
            visrt::ck(cudaMemcpyAsync(regions_out, d_reg, ntasks * sizeof(visrt_region), cudaMemcpyDeviceToHost, st), "D2H");
        unsigned long long ctr[4] = {0, 0, 0, 0};
        visrt::ck(cudaMemcpyAsync(ctr, d_ctr, sizeof(ctr), cudaMemcpyDeviceToHost, st), "D2H");
        visrt::ck(cudaStreamSynchronize(st), "sync");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (stats) {
            *stats = visrt_stats{};
            stats->pairs = ntasks;
            stats->candidates = static_cast<int64_t>(ctr[2]);
            stats->admitted = nsrc * nent;
            stats->tests_exec = static_cast<int64_t>(ctr[1]);
            stats->ms = ms;
        }
    });
}

extern "C" int visrt_segments_clear(visrt_scene* sc, int64_t nseg, const double* a_xyz, const double* b_xyz,
                                    uint8_t* clear, visrt_stats* stats, void* stream) {
    return visrt::capi_guard([&] {
        visrt::ScopedDevice dev(sc);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const visrt::DevScene& ds = visrt::scene_dev(sc);
        std::vector<void*> tmp;
        visrt::FreeGuard guard{tmp};
        double* dA = visrt::dalloc<double>(static_cast<size_t>(nseg) * 3, tmp);
        double* dB = visrt::dalloc<double>(static_cast<size_t>(nseg) * 3, tmp);
        uint8_t* dC = visrt::dalloc<uint8_t>(static_cast<size_t>(nseg), tmp);
        unsigned long long* d_ctr = visrt::dalloc<unsigned long long>(2, tmp);
        visrt::ck(cudaMemcpyAsync(dA, a_xyz, nseg * 24, cudaMemcpyHostToDevice, st), "H2D");
        visrt::ck(cudaMemcpyAsync(dB, b_xyz, nseg * 24, cudaMemcpyHostToDevice, st), "H2D");
        visrt::ck(cudaMemsetAsync(d_ctr, 0, 16, st), "memset");
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
        if (nseg > 0) {
            if (ds.maxv <= 4) visrt::ck(visrt::launch_segments_t<4>(ds, nseg, dA, dB, dC, d_ctr, visrt::scene_device(sc), st), "k_segments_clear");
            else visrt::ck(visrt::launch_segments_t<8>(ds, nseg, dA, dB, dC, d_ctr, visrt::scene_device(sc), st), "k_segments_clear");
        }
        cudaEventRecord(e1, st);
        if (nseg > 0) visrt::ck(cudaMemcpyAsync(clear, dC, nseg, cudaMemcpyDeviceToHost, st), "D2H");
        unsigned long long ctr[2] = {0, 0};
        visrt::ck(cudaMemcpyAsync(ctr, d_ctr, sizeof(ctr), cudaMemcpyDeviceToHost, st), "D2H");
        visrt::ck(cudaStreamSynchronize(st), "sync");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (stats) {
            *stats = visrt_stats{};
            stats->pairs = nseg;
            stats->tests_exec = static_cast<int64_t>(ctr[1]);
            stats->ms = ms;
        }
    });
}
