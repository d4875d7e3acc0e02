// (2) Trajectory visibility tables: trajectory_vis_table (src/vistable.cpp:822-940)
// with MobileSampler (681-812) and the plan-view membership (563-669).
//
// The reference samples the route every kTrajectoryStep = 0.5 m, computes one
// MobileSampler::snapshot per sample (a set of SigKey{order, parent, node,
// vertex}), bisects every membership change to kBoundaryTolerance = 1e-3 m,
// classifies each boundary (vertical-plane or plan-view, blocking building)
// and assembles labelled per-node ranges. Here:
//   * the sampling pass is ONE batched GPU pass over every sample: K4 regions
//     for the faces that head a reflector chain (face-list task mode), K5 beam
//     cascade for every (sample, chain), then one batched sightline sweep for
//     the face-corner (vertex) nodes;
//   * the bisections of all boundaries advance in lockstep, one batched GPU
//     round per halving step (K4/K5 in paired query mode + the sightline
//     sweep), the same midpoints in the same order as the reference's
//     per-boundary loops, so every s is bit-identical;
//   * classify() runs batched too: chain reach at both probe points, the
//     plan-view membership (k_plan_member / k_plan_clear, warp per query) and
//     the blocker sets (k_seg_hits, warp per segment);
//   * sets, labels, ranges and merging are host C++ on face indices, with the
//     string orders of the reference's SigKey / row sorts supplied as ranks
//     (visrt_names), so tie-breaking matches std::set / std::sort exactly.
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <chrono>
#include <array>
#include <cmath>
#include <iterator>
#include <map>
#include <tuple>
#include <unordered_map>
#include <utility>
#include <vector>

#include "capi_internal.h"
#include "sweep.h"
#include "tables.h"

struct visrt_mobile_table {
    std::vector<visrt_mobile_row> rows;
};

namespace visrt {
namespace {

constexpr double kStep = 0.5;         // kTrajectoryStep, include/rt/vistable.hpp:110
constexpr double kBoundTol = 1e-3;    // kBoundaryTolerance, include/rt/vistable.hpp:111

// ---------------------------------------------------------------------------
// Device: plan-view membership (src/vistable.cpp:573-669), warp per query.
// ---------------------------------------------------------------------------

// plan_segment_blocks (src/vistable.cpp:573-582)
__device__ __forceinline__ bool plan_blocks(double px, double py, double qx, double qy, double ax, double ay,
                                            double bx, double by) {
    const double dx = dsub(qx, px), dy = dsub(qy, py);
    const double ex = dsub(bx, ax), ey = dsub(by, ay);
    const double denom = dsub(dmul(dx, ey), dmul(dy, ex));
    const double nd = __dsqrt_rn(dadd(dmul(dx, dx), dmul(dy, dy)));
    const double ne = __dsqrt_rn(dadd(dmul(ex, ex), dmul(ey, ey)));
    if (fabs(denom) <= dmul(1e-15, dadd(dmul(nd, ne), 1.0))) return false;   // parallel
    const double rx = dsub(ax, px), ry = dsub(ay, py);
    const double t = __ddiv_rn(dsub(dmul(rx, ey), dmul(ry, ex)), denom);
    const double u = __ddiv_rn(dsub(dmul(rx, dy), dmul(ry, dx)), denom);
    return t > 1e-9 && t < 1.0 - 1e-9 && u > 1e-9 && u < 1.0 - 1e-9;
}

// Conservative fp32 test of a plan-view (xy) segment against the xy footprint
// of a culling box (2 box axes + the segment normal). A plan blocker's xy
// segment crosses the query strictly inside both, so its face's box (dilated
// by box_margin(), which bounds the fp32 rounding) passes: one-sided culling.
struct Seg2F {
    float mx, my, ex, ey, ax, ay;
};
__device__ __forceinline__ Seg2F make_seg2f(const DevScene& s, double px, double py, double qx, double qy) {
    Seg2F g;
    g.mx = static_cast<float>(0.5 * (px + qx) - s.ox);
    g.my = static_cast<float>(0.5 * (py + qy) - s.oy);
    g.ex = static_cast<float>(0.5 * (qx - px));
    g.ey = static_cast<float>(0.5 * (qy - py));
    g.ax = fabsf(g.ex);
    g.ay = fabsf(g.ey);
    return g;
}
__device__ __forceinline__ bool sat2_maybe(const float* __restrict__ B, const Seg2F& g) {
    const float dx = g.mx - B[0], dy = g.my - B[1];
    const float hx = B[4], hy = B[5];
    bool ok = fabsf(dx) <= hx + g.ax;
    ok &= fabsf(dy) <= hy + g.ay;
    ok &= fabsf(__fmaf_rn(dx, g.ey, -dy * g.ex)) <= __fmaf_rn(hx, g.ay, hy * g.ax);
    return ok;
}

// plan_sightline_clear (584-592): any face's xy segment strictly crossing p->q
// blocks. Culled over the Morton hierarchy: lanes test tile footprints, then
// the members of each candidate tile (2 per lane), exact plan_blocks on the
// survivors (face index perm[m]).
__device__ bool plan_clear_warp(const DevScene& s, double px, double py, double qx, double qy, int skip) {
    const int lane = threadIdx.x & 31;
    const Seg2F g = make_seg2f(s, px, py, qx, qy);
    for (int t0 = 0; t0 < s.ntiles; t0 += 32) {
        const int t = t0 + lane;
        unsigned cand = __ballot_sync(kFull, t < s.ntiles && sat2_maybe(s.tbox + static_cast<size_t>(t) * 8, g));
        while (cand) {
            const int base = (t0 + __ffs(cand) - 1) * 64;
            cand &= cand - 1;
            bool hit = false;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int m = base + lane + 32 * h;
                if (m < s.n && sat2_maybe(s.sbox + static_cast<size_t>(m) * 8, g)) {
                    const int f = s.perm[m];
                    if (f != skip && s.seg_ok[3 * f]) {
                        const double* sg = s.seg + static_cast<size_t>(f) * 18;
                        hit |= plan_blocks(px, py, qx, qy, sg[0], sg[1], sg[2], sg[3]);
                    }
                }
            }
            if (__any_sync(kFull, hit)) return false;
        }
    }
    return true;
}

// mirror_across_segment (src/vistable.cpp:205-210)
__device__ __forceinline__ void mirror2(double qx, double qy, double ax, double ay, double bx, double by,
                                        double& mx, double& my) {
    const double dx = dsub(bx, ax), dy = dsub(by, ay);
    const double len2 = dadd(dmul(dx, dx), dmul(dy, dy));
    const double t = __ddiv_rn(dadd(dmul(dsub(qx, ax), dx), dmul(dsub(qy, ay), dy)), len2);
    const double fx = dadd(ax, dmul(dx, t)), fy = dadd(ay, dmul(dy, t));
    mx = dsub(dmul(fx, 2.0), qx);
    my = dsub(dmul(fy, 2.0), qy);
}

__global__ void __launch_bounds__(256) k_plan_clear(DevScene s, int nq, const double* P, const double* Q,
                                                    uint8_t* out) {
    const int lane = threadIdx.x & 31;
    for (int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < nq; q += (gridDim.x * blockDim.x) >> 5) {
        const bool c = plan_clear_warp(s, P[2 * q], P[2 * q + 1], Q[2 * q], Q[2 * q + 1], -1);
        if (lane == 0) out[q] = c ? 1 : 0;
    }
}

// plan_member_chain (src/vistable.cpp:635-669) with plan_visible_intervals
// (594-633) inlined: query q = (source xy, reflector chain[4], -1 padded).
__global__ void __launch_bounds__(256) k_plan_member(DevScene s, int nq, const double* S2, const int32_t* chain,
                                                     uint8_t* out) {
    const int lane = threadIdx.x & 31;
    for (int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < nq; q += (gridDim.x * blockDim.x) >> 5) {
        const double sx = S2[2 * q], sy = S2[2 * q + 1];
        const int head = chain[4 * q];
        bool member = false;
        do {
            if (!s.seg_ok[3 * head]) break;
            const double* hs = s.seg + static_cast<size_t>(head) * 18;
            const double ax = hs[0], ay = hs[1], bx = hs[2], by = hs[3], nx = hs[4], ny = hs[5];
            if (dadd(dmul(dsub(sx, ax), nx), dmul(dsub(sy, ay), ny)) <= kEps) break;
            const double dx = dsub(bx, ax), dy = dsub(by, ay);
            auto vis_at = [&](double u) {
                const double uc = u < 0.0 ? 0.0 : (1.0 < u ? 1.0 : u);   // std::clamp(u, 0, 1)
                return plan_clear_warp(s, sx, sy, dadd(ax, dmul(dx, uc)), dadd(ay, dmul(dy, uc)), head);
            };
            unsigned long long vis = 0;
            bool vis64 = false;
            for (int i = 0; i < 65; ++i) {
                const bool v = vis_at(__ddiv_rn(static_cast<double>(i), 64.0));
                if (i < 64) vis |= static_cast<unsigned long long>(v) << i;
                else vis64 = v;
            }
            auto V = [&](int i) { return i == 64 ? vis64 : ((vis >> i) & 1ull) != 0; };
            auto refine = [&](double lo, double hi, bool lo_vis) {
                for (int it = 0; it < 50 && dsub(hi, lo) > 1e-15; ++it) {
                    const double mid = dmul(0.5, dadd(lo, hi));
                    if (vis_at(mid) == lo_vis) lo = mid;
                    else hi = mid;
                }
                return dmul(0.5, dadd(lo, hi));
            };
            const double step = __ddiv_rn(1.0, 64.0);
            bool have = false;
            double b0 = 0, b1 = 0;
            int i = 0;
            while (i < 65) {
                if (!V(i)) {
                    ++i;
                    continue;
                }
                double start = __ddiv_rn(static_cast<double>(i), 64.0);
                if (i > 0) start = refine(dsub(start, step), start, false);
                int j = i;
                while (j + 1 < 65 && V(j + 1)) ++j;
                double end = __ddiv_rn(static_cast<double>(j), 64.0);
                if (j + 1 < 65) end = refine(end, dadd(end, step), true);
                // std::max_element by width: the first widest interval
                if (!have || dsub(b1, b0) < dsub(end, start)) {
                    b0 = start;
                    b1 = end;
                    have = true;
                }
                i = j + 1;
            }
            if (!have) break;
            double wax = dadd(ax, dmul(dx, b0)), way = dadd(ay, dmul(dy, b0));
            double wbx = dadd(ax, dmul(dx, b1)), wby = dadd(ay, dmul(dy, b1));
            double apx, apy;
            mirror2(sx, sy, ax, ay, bx, by, apx, apy);
            double ox = nx, oy = ny;
            bool ok = true;
            for (int c = 1; c < 4 && ok; ++c) {
                const int g = chain[4 * q + c];
                if (g < 0) break;
                if (!s.seg_ok[3 * g]) {
                    ok = false;
                    break;
                }
                const double* gs = s.seg + static_cast<size_t>(g) * 18;
                const Cov cv = beam_coverage(apx, apy, wax, way, wbx, wby, ox, oy, gs[0], gs[1], gs[2], gs[3]);
                if (cv.verdict == 2) {
                    ok = false;
                    break;
                }
                const double qx = dsub(gs[2], gs[0]), qy = dsub(gs[3], gs[1]);
                wax = dadd(gs[0], dmul(qx, cv.lo));
                way = dadd(gs[1], dmul(qy, cv.lo));
                wbx = dadd(gs[0], dmul(qx, cv.hi));
                wby = dadd(gs[1], dmul(qy, cv.hi));
                double mx, my;
                mirror2(apx, apy, gs[0], gs[1], gs[2], gs[3], mx, my);
                apx = mx;
                apy = my;
                ox = gs[4];
                oy = gs[5];
            }
            member = ok;
        } while (false);
        if (lane == 0) out[q] = member ? 1 : 0;
    }
}

// segment_blockers / probe_blockers (src/vistable.cpp:48-67): every face (but
// `skip`) the open segment hits, as a bitset over face indices. Warp per
// segment, exact predicate on every face (these run once per boundary).
template <int MAXV>
__global__ void __launch_bounds__(256) k_seg_hits(DevScene s, int nseg, const double* A, const double* B,
                                                  const int32_t* skip, uint32_t* hits, int words) {
    constexpr int STRIDE = RecLayout<MAXV>::kStride;
    const int lane = threadIdx.x & 31;
    for (int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < nseg; q += (gridDim.x * blockDim.x) >> 5) {
        const double ax = A[3 * q], ay = A[3 * q + 1], az = A[3 * q + 2];
        const double bx = B[3 * q], by = B[3 * q + 1], bz = B[3 * q + 2];
        // every hit, culled: tile boxes, then the members of candidate tiles
        // (a true hit lies in its face's dilated box: sweep.h)
        const SegF g = make_segf(s, ax, ay, az, bx, by, bz);
        for (int t0 = 0; t0 < s.ntiles; t0 += 32) {
            const int t = t0 + lane;
            unsigned cand = __ballot_sync(kFull, t < s.ntiles && sat_maybe(s.tbox + static_cast<size_t>(t) * 8, g));
            while (cand) {
                const int base = (t0 + __ffs(cand) - 1) * 64;
                cand &= cand - 1;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int m = base + lane + 32 * h;
                    if (m >= s.n || !sat_maybe(s.sbox + static_cast<size_t>(m) * 8, g)) continue;
                    const int f = s.perm[m];
                    if (f == skip[q]) continue;
                    if (seg_hits<MAXV>(s.srec + static_cast<size_t>(m) * STRIDE, ax, ay, az, bx, by, bz))
                        atomicOr(hits + static_cast<size_t>(q) * words + (f >> 5), 1u << (f & 31));
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Host: batched GPU rounds.
// ---------------------------------------------------------------------------

struct Gpu {
    const visrt_scene* sc;
    const DevScene& ds;
    int device;
    cudaStream_t st;
    float ms = 0.f;
    int64_t tests = 0, launches = 0;

    template <class T>
    T* up(const std::vector<T>& v, std::vector<void*>& tmp) {
        T* d = dalloc<T>(v.size(), tmp);
        if (!v.empty()) ck(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st), "H2D");
        return d;
    }
    template <class T>
    void down(std::vector<T>& v, const T* d) {
        if (!v.empty()) ck(cudaMemcpyAsync(v.data(), d, v.size() * sizeof(T), cudaMemcpyDeviceToHost, st), "D2H");
    }
    struct Timed {
        Gpu& g;
        cudaEvent_t e0, e1;
        explicit Timed(Gpu& gg) : g(gg) {
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0, g.st);
        }
        void done() {
            cudaEventRecord(e1, g.st);
            ck(cudaStreamSynchronize(g.st), "sync");
            float t = 0.f;
            cudaEventElapsedTime(&t, e0, e1);
            g.ms += t;
        }
        ~Timed() {
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
        }
    };
    static int warp_grid(long long nq) { return static_cast<int>(std::min<long long>((nq + 7) / 8, 148 * 16)); }

    // TableBuilder::reach(chain) != nullopt for query list (src[q], chain q):
    // K4 region of the chain head (paired task mode) + K5 cascade.
    // presence: order-1 queries only need whether the head has a region (K4w
    // presence mode: the scan stops at the first visible column)
    std::vector<uint8_t> reach_paired(const std::vector<double>& src, const std::vector<visrt_entry>& q,
                                      std::vector<uint8_t>* full = nullptr, bool presence = false) {
        const long long nq = static_cast<long long>(q.size());
        std::vector<uint8_t> out(q.size(), 0);
        if (full) full->assign(q.size(), 0);
        if (nq == 0) return out;
        std::vector<void*> tmp;
        FreeGuard guard{tmp};
        std::vector<int32_t> face(q.size());
        for (size_t k = 0; k < q.size(); ++k) face[k] = q[k].chain[0];
        const int words = static_cast<int>((nq + 31) / 32);
        double* d_src = up(src, tmp);
        int32_t* d_face = up(face, tmp);
        visrt_entry* d_ent = up(q, tmp);
        visrt_region* d_reg = dalloc<visrt_region>(q.size(), tmp);
        uint32_t* d_rows = dalloc<uint32_t>(words, tmp);
        uint32_t* d_full = dalloc<uint32_t>(words, tmp);
        unsigned long long* d_ctr = dalloc<unsigned long long>(4, tmp);
        ck(cudaMemsetAsync(d_rows, 0, words * 4, st), "memset");
        ck(cudaMemsetAsync(d_full, 0, words * 4, st), "memset");
        ck(cudaMemsetAsync(d_ctr, 0, 32, st), "memset");
        Timed t(*this);
        RegionArgs ra{ds, nq, d_src, d_reg, d_ctr, d_face, 0, 1};
        if (presence) {
            std::vector<uint8_t> pres(q.size());
            for (size_t k = 0; k < q.size(); ++k) pres[k] = q[k].order == 1 ? 1 : 0;
            ra.presence_of = up(pres, tmp);
        }
        ck(launch_point_regions(ra, device, st), "k_point_regions");
        BeamArgs ba{ds, 1, nq, d_src, d_reg, d_ent, d_rows, d_full, words, nullptr, 0, 1};
        ck(launch_beam_rows(ba, st), "k_beam_rows");
        launches += 2;
        std::vector<uint32_t> rows(words), fb(words);
        unsigned long long ctr[4];
        down(rows, d_rows);
        down(fb, d_full);
        ck(cudaMemcpyAsync(ctr, d_ctr, sizeof(ctr), cudaMemcpyDeviceToHost, st), "D2H");
        t.done();
        tests += static_cast<int64_t>(ctr[1]);
        for (long long k = 0; k < nq; ++k) {
            out[k] = (rows[k >> 5] >> (k & 31)) & 1u;
            if (full) (*full)[k] = (fb[k >> 5] >> (k & 31)) & 1u;
        }
        return out;
    }

    // Dense sampling pass: reach bits of every (source k, chain u); the
    // regions are computed only for the chain heads (face-list task mode).
    std::vector<uint32_t> reach_dense(const std::vector<double>& src, const std::vector<visrt_entry>& chains,
                                      int& words) {
        const long long ns = static_cast<long long>(src.size() / 3);
        const long long nc = static_cast<long long>(chains.size());
        words = static_cast<int>((nc + 31) / 32);
        std::vector<uint32_t> bits(static_cast<size_t>(ns) * words, 0u);
        if (ns == 0 || nc == 0) return bits;
        std::vector<int32_t> slot(ds.n, -1), heads;
        for (const visrt_entry& e : chains)
            if (slot[e.chain[0]] < 0) {
                slot[e.chain[0]] = static_cast<int32_t>(heads.size());
                heads.push_back(e.chain[0]);
            }
        const long long m = static_cast<long long>(heads.size());
        // heads whose chains are all single reflectors only need presence
        std::vector<uint8_t> pres(heads.size(), 1);
        for (const visrt_entry& e : chains)
            if (e.order >= 2) pres[slot[e.chain[0]]] = 0;
        const long long batch = std::max<long long>(1, (1ll << 24) / m);   // <= 16.8 M regions (0.9 GB) per batch
        std::vector<void*> tmp;
        FreeGuard guard{tmp};
        int32_t* d_heads = up(heads, tmp);
        uint8_t* d_pres = up(pres, tmp);
        int32_t* d_slot = up(slot, tmp);
        visrt_entry* d_ent = up(chains, tmp);
        const long long bs = std::min(batch, ns);
        double* d_src = dalloc<double>(static_cast<size_t>(bs) * 3, tmp);
        visrt_region* d_reg = dalloc<visrt_region>(static_cast<size_t>(bs * m), tmp);
        uint32_t* d_rows = dalloc<uint32_t>(static_cast<size_t>(bs) * words, tmp);
        uint32_t* d_full = dalloc<uint32_t>(static_cast<size_t>(bs) * words, tmp);
        unsigned long long* d_ctr = dalloc<unsigned long long>(4, tmp);
        for (long long k0 = 0; k0 < ns; k0 += bs) {
            const long long nb = std::min(bs, ns - k0);
            ck(cudaMemcpyAsync(d_src, src.data() + 3 * k0, nb * 24, cudaMemcpyHostToDevice, st), "H2D");
            ck(cudaMemsetAsync(d_rows, 0, static_cast<size_t>(nb) * words * 4, st), "memset");
            ck(cudaMemsetAsync(d_full, 0, static_cast<size_t>(nb) * words * 4, st), "memset");
            ck(cudaMemsetAsync(d_ctr, 0, 32, st), "memset");
            Timed t(*this);
            RegionArgs ra{ds, nb * m, d_src, d_reg, d_ctr, d_heads, static_cast<int>(m), 0};
            ra.presence_of = d_pres;
            ck(launch_point_regions(ra, device, st), "k_point_regions");
            BeamArgs ba{ds, nb, nc, d_src, d_reg, d_ent, d_rows, d_full, words, d_slot, static_cast<int>(m), 0};
            ck(launch_beam_rows(ba, st), "k_beam_rows");
            launches += 2;
            unsigned long long ctr[4];
            ck(cudaMemcpyAsync(bits.data() + static_cast<size_t>(k0) * words, d_rows,
                               static_cast<size_t>(nb) * words * 4, cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaMemcpyAsync(ctr, d_ctr, sizeof(ctr), cudaMemcpyDeviceToHost, st), "D2H");
            t.done();
            tests += static_cast<int64_t>(ctr[1]);
        }
        return bits;
    }

    // sightline_clear(a, b, scene, -1) per segment (culled any-hit sweep).
    std::vector<uint8_t> segs_clear(const std::vector<double>& A, const std::vector<double>& B) {
        const long long nseg = static_cast<long long>(A.size() / 3);
        std::vector<uint8_t> out(static_cast<size_t>(nseg), 0);
        if (nseg == 0) return out;
        std::vector<void*> tmp;
        FreeGuard guard{tmp};
        double* dA = up(A, tmp);
        double* dB = up(B, tmp);
        uint8_t* dC = dalloc<uint8_t>(out.size(), tmp);
        unsigned long long* d_ctr = dalloc<unsigned long long>(2, tmp);
        ck(cudaMemsetAsync(d_ctr, 0, 16, st), "memset");
        Timed t(*this);
        ck(launch_segments_clear(ds, nseg, dA, dB, dC, d_ctr, device, st), "k_segments_clear");
        ++launches;
        unsigned long long ctr[2];
        down(out, dC);
        ck(cudaMemcpyAsync(ctr, d_ctr, sizeof(ctr), cudaMemcpyDeviceToHost, st), "D2H");
        t.done();
        tests += static_cast<int64_t>(ctr[1]);
        return out;
    }

    std::vector<uint8_t> plan_clear(const std::vector<double>& P, const std::vector<double>& Q) {
        const int nq = static_cast<int>(P.size() / 2);
        std::vector<uint8_t> out(static_cast<size_t>(nq), 0);
        if (nq == 0) return out;
        std::vector<void*> tmp;
        FreeGuard guard{tmp};
        double* dP = up(P, tmp);
        double* dQ = up(Q, tmp);
        uint8_t* dO = dalloc<uint8_t>(out.size(), tmp);
        Timed t(*this);
        k_plan_clear<<<warp_grid(nq), 256, 0, st>>>(ds, nq, dP, dQ, dO);
        ck(cudaGetLastError(), "k_plan_clear");
        ++launches;
        down(out, dO);
        t.done();
        return out;
    }

    std::vector<uint8_t> plan_member(const std::vector<double>& S2, const std::vector<int32_t>& chain2) {
        const int nq = static_cast<int>(S2.size() / 2);
        std::vector<uint8_t> out(static_cast<size_t>(nq), 0);
        if (nq == 0) return out;
        std::vector<void*> tmp;
        FreeGuard guard{tmp};
        double* dS = up(S2, tmp);
        int32_t* dC = up(chain2, tmp);
        uint8_t* dO = dalloc<uint8_t>(out.size(), tmp);
        Timed t(*this);
        k_plan_member<<<warp_grid(nq), 256, 0, st>>>(ds, nq, dS, dC, dO);
        ck(cudaGetLastError(), "k_plan_member");
        ++launches;
        down(out, dO);
        t.done();
        return out;
    }

    // hit bitsets [nseg][words] over face indices
    std::vector<uint32_t> seg_hits(const std::vector<double>& A, const std::vector<double>& B,
                                   const std::vector<int32_t>& skip, int& words) {
        const int nseg = static_cast<int>(A.size() / 3);
        words = (ds.n + 31) / 32;
        std::vector<uint32_t> out(static_cast<size_t>(nseg) * words, 0u);
        if (nseg == 0) return out;
        std::vector<void*> tmp;
        FreeGuard guard{tmp};
        double* dA = up(A, tmp);
        double* dB = up(B, tmp);
        int32_t* dS = up(skip, tmp);
        uint32_t* dH = dalloc<uint32_t>(out.size(), tmp);
        ck(cudaMemsetAsync(dH, 0, out.size() * 4, st), "memset");
        Timed t(*this);
        if (ds.maxv <= 4) k_seg_hits<4><<<warp_grid(nseg), 256, 0, st>>>(ds, nseg, dA, dB, dS, dH, words);
        else k_seg_hits<8><<<warp_grid(nseg), 256, 0, st>>>(ds, nseg, dA, dB, dS, dH, words);
        ck(cudaGetLastError(), "k_seg_hits");
        ++launches;
        down(out, dH);
        t.done();
        return out;
    }
};

// ---------------------------------------------------------------------------
// Host: the reference's trajectory arithmetic (src/scene.cpp:443-469).
// ---------------------------------------------------------------------------

struct Route {
    std::vector<double> w;   // [nwp][3]
    int nwp = 0;
    double seg_len(int i) const {   // norm(w[i+1] - w[i])
        const double dx = w[3 * i + 3] - w[3 * i], dy = w[3 * i + 4] - w[3 * i + 1], dz = w[3 * i + 5] - w[3 * i + 2];
        return std::sqrt(dx * dx + dy * dy + dz * dz);
    }
    double total_length() const {
        double len = 0;
        for (int i = 0; i + 1 < nwp; ++i) len += seg_len(i);
        return len;
    }
    void position_at(double s, double* p) const {
        if (s <= 0) {
            p[0] = w[0]; p[1] = w[1]; p[2] = w[2];
            return;
        }
        for (int i = 0; i + 1 < nwp; ++i) {
            const double seg = seg_len(i);
            if (s <= seg) {
                const double t = s / seg;
                for (int c = 0; c < 3; ++c) p[c] = w[3 * i + c] + (w[3 * i + 3 + c] - w[3 * i + c]) * t;
                return;
            }
            s -= seg;
        }
        const int l = 3 * (nwp - 1);
        p[0] = w[l]; p[1] = w[l + 1]; p[2] = w[l + 2];
    }
};

struct KeyDef {
    int order, parent, node, vertex;   // parent -1 = "transmitter"; vertex -1 = face node
};

struct Event {
    double s = 0.0, lo = 0.0, hi = 0.0;
    int key = 0;
    bool before = false, appearing = false, vertical = false;
    int blockage = -1;
    int label = 0;
};

std::vector<visrt_mobile_row> trajectory_table(Gpu& gpu, const HostScene& hs, const Route& route,
                                               const visrt_entry* entries, int64_t nent, int max_order,
                                               const visrt_names& nm, visrt_stats& stats) {
    const int n = hs.n;
    // VISRT_TRAJ_PROFILE=1: host wall time per phase on stderr (development aid)
    static const bool prof = [] {
        const char* e = std::getenv("VISRT_TRAJ_PROFILE");
        return e && e[0] == '1';
    }();
    auto t_last = std::chrono::steady_clock::now();
    auto phase = [&](const char* name) {
        if (!prof) return;
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[traj] %-10s %8.2f ms\n", name,
                     std::chrono::duration<double, std::milli>(t - t_last).count());
        t_last = t;
    };
    const double length = route.total_length();
    auto pos = [&](double s, std::vector<double>& out) {
        double p[3];
        route.position_at(s, p);
        out.insert(out.end(), p, p + 3);
    };
    auto corner = [&](int f, int k, std::vector<double>& out) {
        const double* P = &hs.pts[(static_cast<size_t>(f) * VISRT_MAX_VERTS + k) * 3];
        out.insert(out.end(), P, P + 3);
    };

    // ---- MobileSampler ctor (src/vistable.cpp:699-716): keys and chains ----
    // hash maps on packed 16-bit face slots (faces < 65536 is checked by the caller)
    std::unordered_map<uint64_t, int> chain_id;   // reflectors (-1 padded) -> id
    std::vector<visrt_entry> chains;              // as K5 entries (order = #reflectors)
    std::vector<KeyDef> keys;
    std::unordered_map<uint64_t, int> face_key;   // (order, parent, node) -> keys index
    std::vector<std::vector<int>> key_chains;
    auto slot16 = [](int f) { return static_cast<uint64_t>(static_cast<uint16_t>(f)); };   // -1 -> 0xFFFF
    uint64_t last_refl = ~0ull;
    int last_c = -1, last_k = -1;
    for (int64_t q = 0; q < nent; ++q) {   // the caller's matrix entries, read in place
        const visrt_entry& e = entries[q];
        if (e.order < 1 || e.order > max_order) continue;
        const int L = e.order;   // reflectors chain[0..L-1]
        uint64_t rk = 0;
        for (int w = 0; w < 4; ++w) rk = (rk << 16) | slot16(w < L ? e.chain[w] : -1);
        int c, k;
        if (rk == last_refl) {   // consecutive entries of one chain (planes, aims): no lookups
            c = last_c;
            k = last_k;
        } else {
            auto ci = chain_id.find(rk);
            if (ci == chain_id.end()) {
                c = static_cast<int>(chains.size());
                chain_id.emplace(rk, c);
                visrt_entry ce = e;   // the K5 query: same reflectors (the aim and plane are not read for reach)
                ce.plane = 0;
                chains.push_back(ce);
            } else {
                c = ci->second;
            }
            const KeyDef kd{L, L >= 2 ? e.chain[L - 2] : -1, e.chain[L - 1], -1};
            const uint64_t kk = (static_cast<uint64_t>(L) << 32) | (slot16(kd.parent) << 16) | slot16(kd.node);
            auto it = face_key.find(kk);
            if (it == face_key.end()) {
                k = static_cast<int>(keys.size());
                face_key.emplace(kk, k);
                keys.push_back(kd);
                key_chains.emplace_back();
            } else {
                k = it->second;
            }
            last_refl = rk;
            last_c = c;
            last_k = k;
            if (std::find(key_chains[k].begin(), key_chains[k].end(), c) == key_chains[k].end())
                key_chains[k].push_back(c);
        }
    }
    const int nface_keys = static_cast<int>(keys.size());
    std::vector<int> vkey_base(nface_keys, -1);   // order-1 face key -> first vertex key
    for (int k = 0; k < nface_keys; ++k) {
        if (keys[k].order != 1) continue;
        vkey_base[k] = static_cast<int>(keys.size());
        for (int v = 0; v < hs.nv[keys[k].node]; ++v) {
            keys.push_back({1, -1, keys[k].node, v});
            key_chains.emplace_back();
        }
    }
    // SigKey order (order, parent, node, vertex) from the caller's string ranks
    const int nk = static_cast<int>(keys.size());
    auto prank = [&](int p) { return p < 0 ? nm.key_rank[9 * n] : nm.key_rank[p]; };
    auto nrank = [&](const KeyDef& k) {
        return k.vertex < 0 ? nm.key_rank[k.node] : nm.key_rank[n + VISRT_MAX_VERTS * k.node + k.vertex];
    };
    auto key_less = [&](const KeyDef& a, const KeyDef& b) {
        if (a.order != b.order) return a.order < b.order;
        if (prank(a.parent) != prank(b.parent)) return prank(a.parent) < prank(b.parent);
        if (nrank(a) != nrank(b)) return nrank(a) < nrank(b);
        return (a.vertex >= 0) < (b.vertex >= 0);
    };
    std::vector<int> order_of(nk), by_rank(nk);
    for (int k = 0; k < nk; ++k) by_rank[k] = k;
    std::stable_sort(by_rank.begin(), by_rank.end(), [&](int a, int b) { return key_less(keys[a], keys[b]); });
    for (int r = 0; r < nk; ++r) order_of[by_rank[r]] = r;   // key -> position in SigKey order

    phase("keys");
    // ---- sampling pass (src/vistable.cpp:846-866) --------------------------
    std::vector<double> samples;
    for (double s = 0.0; s < length; s += kStep) samples.push_back(s);
    samples.push_back(length);
    const int ns = static_cast<int>(samples.size());
    std::vector<double> P;
    P.reserve(3 * static_cast<size_t>(ns));
    for (double s : samples) pos(s, P);
    int words = 0;
    const std::vector<uint32_t> rbits = gpu.reach_dense(P, chains, words);
    std::vector<std::vector<int>> snaps(ns);   // SigKey-ordered positions
    std::vector<double> VA, VB;
    std::vector<std::pair<int, int>> vseg;     // (sample, key)
    std::vector<int> key_of_chain(chains.size(), -1);   // a chain's reflectors fix its key
    for (int k = 0; k < nface_keys; ++k)
        for (int c : key_chains[k]) key_of_chain[c] = k;
    std::vector<int> ks;
    for (int i = 0; i < ns; ++i) {
        ks.clear();
        for (int w = 0; w < words; ++w)
            for (uint32_t b = rbits[static_cast<size_t>(i) * words + w]; b; b &= b - 1)
                ks.push_back(key_of_chain[32 * w + __builtin_ctz(b)]);
        std::sort(ks.begin(), ks.end());
        ks.erase(std::unique(ks.begin(), ks.end()), ks.end());
        for (int k : ks) {
            snaps[i].push_back(order_of[k]);
            if (keys[k].order == 1)
                for (int v = 0; v < hs.nv[keys[k].node]; ++v) {
                    VA.insert(VA.end(), &P[3 * static_cast<size_t>(i)], &P[3 * static_cast<size_t>(i)] + 3);
                    corner(keys[k].node, v, VB);
                    vseg.push_back({i, vkey_base[k] + v});
                }
        }
    }
    const std::vector<uint8_t> vclear = gpu.segs_clear(VA, VB);
    for (size_t q = 0; q < vseg.size(); ++q)
        if (vclear[q]) snaps[vseg[q].first].push_back(order_of[vseg[q].second]);
    for (auto& sn : snaps) std::sort(sn.begin(), sn.end());

    phase("sampling");
    // ---- boundaries: lockstep bisection (src/vistable.cpp:868-885) -------
    std::vector<Event> events;
    for (int i = 0; i + 1 < ns; ++i) {
        std::vector<int> changed;
        std::set_symmetric_difference(snaps[i].begin(), snaps[i].end(), snaps[i + 1].begin(), snaps[i + 1].end(),
                                      std::back_inserter(changed));
        for (int r : changed) {
            Event ev;
            ev.key = by_rank[r];
            ev.before = std::binary_search(snaps[i].begin(), snaps[i].end(), r);
            ev.lo = samples[i];
            ev.hi = samples[i + 1];
            events.push_back(ev);
        }
    }
    // member(position, key) for a batch of (event, position) probes
    auto members = [&](const std::vector<std::pair<int, const double*>>& probes) {
        std::vector<double> SA, SB, RS;
        std::vector<visrt_entry> RQ;
        std::vector<int> seg_of(probes.size(), -1), rq0(probes.size(), -1);
        for (size_t q = 0; q < probes.size(); ++q) {
            const KeyDef& kd = keys[events[probes[q].first].key];
            const double* p = probes[q].second;
            if (kd.vertex >= 0) {
                seg_of[q] = static_cast<int>(SA.size() / 3);
                SA.insert(SA.end(), p, p + 3);
                corner(kd.node, kd.vertex, SB);
            } else {
                rq0[q] = static_cast<int>(RQ.size());
                for (int c : key_chains[events[probes[q].first].key]) {
                    RQ.push_back(chains[c]);
                    RS.insert(RS.end(), p, p + 3);
                }
            }
        }
        const std::vector<uint8_t> sc = gpu.segs_clear(SA, SB);
        const std::vector<uint8_t> rc = gpu.reach_paired(RS, RQ, nullptr, true);
        std::vector<uint8_t> out(probes.size(), 0);
        for (size_t q = 0; q < probes.size(); ++q) {
            if (seg_of[q] >= 0) {
                out[q] = sc[seg_of[q]];
            } else {
                const int nc = static_cast<int>(key_chains[events[probes[q].first].key].size());
                for (int c = 0; c < nc; ++c) out[q] |= rc[rq0[q] + c];
            }
        }
        return out;
    };
    for (;;) {
        std::vector<int> act;
        for (int e = 0; e < static_cast<int>(events.size()); ++e)
            if (events[e].hi - events[e].lo > kBoundTol) act.push_back(e);
        if (act.empty()) break;
        std::vector<double> mids(act.size()), mp;
        mp.reserve(3 * act.size());
        for (size_t q = 0; q < act.size(); ++q) {
            mids[q] = 0.5 * (events[act[q]].lo + events[act[q]].hi);
            pos(mids[q], mp);
        }
        std::vector<std::pair<int, const double*>> probes(act.size());
        for (size_t q = 0; q < act.size(); ++q) probes[q] = {act[q], &mp[3 * q]};
        const std::vector<uint8_t> m = members(probes);
        for (size_t q = 0; q < act.size(); ++q) {
            Event& ev = events[act[q]];
            if ((m[q] != 0) == ev.before) ev.lo = mids[q];
            else ev.hi = mids[q];
        }
    }

    phase("bisection");
    // ---- classify (src/vistable.cpp:770-812), batched ----------------------
    const size_t ne = events.size();
    std::vector<double> pm(3 * ne), po(3 * ne);   // p_member, p_other
    for (size_t e = 0; e < ne; ++e) {
        Event& ev = events[e];
        ev.s = 0.5 * (ev.lo + ev.hi);
        ev.appearing = !ev.before;
        const double delta = 2.0 * kBoundTol;
        const double sb = std::max(0.0, ev.s - delta);
        const double sa = std::min(length, ev.s + delta);
        double pb[3], pa[3];
        route.position_at(sb, pb);
        route.position_at(sa, pa);
        for (int c = 0; c < 3; ++c) {
            pm[3 * e + c] = ev.before ? pb[c] : pa[c];
            po[3 * e + c] = ev.before ? pa[c] : pb[c];
        }
    }
    // (a) chain reach at both probes, for the flipped chain of face keys
    std::vector<double> RS;
    std::vector<visrt_entry> RQ;
    std::vector<int> rq0(ne, -1);
    for (size_t e = 0; e < ne; ++e) {
        const KeyDef& kd = keys[events[e].key];
        if (kd.vertex >= 0) continue;
        rq0[e] = static_cast<int>(RQ.size());
        for (int c : key_chains[events[e].key]) {
            RQ.push_back(chains[c]);
            RS.insert(RS.end(), &pm[3 * e], &pm[3 * e] + 3);
            RQ.push_back(chains[c]);
            RS.insert(RS.end(), &po[3 * e], &po[3 * e] + 3);
        }
    }
    const std::vector<uint8_t> rc = gpu.reach_paired(RS, RQ, nullptr, true);
    // (b) plan-view membership + blocker segments
    std::vector<double> CP, CQ, MS;
    std::vector<int32_t> MC, skip;
    std::vector<double> HA, HB;
    std::vector<int> plan0(ne), hit0(ne), hitn(ne);
    for (size_t e = 0; e < ne; ++e) {
        const KeyDef& kd = keys[events[e].key];
        const double m2[2] = {pm[3 * e], pm[3 * e + 1]}, o2[2] = {po[3 * e], po[3 * e + 1]};
        hit0[e] = static_cast<int>(skip.size());
        if (kd.vertex >= 0) {
            plan0[e] = static_cast<int>(CP.size() / 2);
            std::vector<double> c3;
            corner(kd.node, kd.vertex, c3);
            CP.insert(CP.end(), m2, m2 + 2);
            CQ.insert(CQ.end(), c3.begin(), c3.begin() + 2);
            CP.insert(CP.end(), o2, o2 + 2);
            CQ.insert(CQ.end(), c3.begin(), c3.begin() + 2);
            // segment_blockers(p_member, corner) / (p_other, corner)
            HA.insert(HA.end(), &pm[3 * e], &pm[3 * e] + 3);
            HB.insert(HB.end(), c3.begin(), c3.end());
            skip.push_back(-1);
            HA.insert(HA.end(), &po[3 * e], &po[3 * e] + 3);
            HB.insert(HB.end(), c3.begin(), c3.end());
            skip.push_back(-1);
            hitn[e] = 1;
        } else {
            const std::vector<int>& kc = key_chains[events[e].key];
            int flipped = kc.front();
            for (size_t c = 0; c < kc.size(); ++c)
                if (rc[rq0[e] + 2 * c] != rc[rq0[e] + 2 * c + 1]) {
                    flipped = kc[c];
                    break;
                }
            const visrt_entry& ch = chains[flipped];
            plan0[e] = static_cast<int>(MS.size() / 2);
            int32_t c4[4] = {-1, -1, -1, -1};
            for (int q = 0; q < ch.order && q < 4; ++q) c4[q] = ch.chain[q];
            MS.insert(MS.end(), m2, m2 + 2);
            MC.insert(MC.end(), c4, c4 + 4);
            MS.insert(MS.end(), o2, o2 + 2);
            MC.insert(MC.end(), c4, c4 + 4);
            // probe_blockers(p, head): head vertices + centroid, head skipped
            const int head = ch.chain[0];
            const int nv = hs.nv[head];
            for (int side = 0; side < 2; ++side) {
                const double* p = side == 0 ? &pm[3 * e] : &po[3 * e];
                for (int v = 0; v <= nv; ++v) {
                    HA.insert(HA.end(), p, p + 3);
                    const double* q = &hs.samples[(static_cast<size_t>(head) * kMaxSamples + v) * 3];   // v == nv: centroid
                    HB.insert(HB.end(), q, q + 3);
                    skip.push_back(head);
                }
            }
            hitn[e] = nv + 1;
        }
    }
    const std::vector<uint8_t> pc = gpu.plan_clear(CP, CQ);
    const std::vector<uint8_t> pmm = gpu.plan_member(MS, MC);
    int hw = 0;
    const std::vector<uint32_t> hits = gpu.seg_hits(HA, HB, skip, hw);
    for (size_t e = 0; e < ne; ++e) {
        Event& ev = events[e];
        const KeyDef& kd = keys[ev.key];
        const std::vector<uint8_t>& pv = kd.vertex >= 0 ? pc : pmm;
        ev.vertical = pv[plan0[e]] == pv[plan0[e] + 1];
        std::vector<int> mb, ob;   // building ranks hit from p_member / p_other
        for (int side = 0; side < 2; ++side) {
            std::vector<int>& dst = side == 0 ? mb : ob;
            for (int q = 0; q < hitn[e]; ++q) {
                const uint32_t* row = &hits[static_cast<size_t>(hit0[e] + side * hitn[e] + q) * hw];
                for (int w = 0; w < hw; ++w)
                    for (uint32_t b = row[w]; b; b &= b - 1) dst.push_back(nm.building_rank[32 * w + __builtin_ctz(b)]);
            }
            std::sort(dst.begin(), dst.end());
            dst.erase(std::unique(dst.begin(), dst.end()), dst.end());
        }
        std::vector<int> fresh;
        std::set_difference(ob.begin(), ob.end(), mb.begin(), mb.end(), std::back_inserter(fresh));
        ev.blockage = fresh.empty() ? -1 : fresh.front();
    }

    phase("classify");
    // ---- labels (src/vistable.cpp:887-898) --------------------------------
    std::stable_sort(events.begin(), events.end(), [](const Event& a, const Event& b) {
        if (a.vertical != b.vertical) return a.vertical > b.vertical;
        return a.s < b.s;
    });
    int counter = 0;
    for (Event& ev : events) ev.label = ++counter;
    std::sort(events.begin(), events.end(), [](const Event& a, const Event& b) { return a.s < b.s; });

    // ---- per-node ranges (900-940) ------------------------------------------
    std::vector<char> seen(static_cast<size_t>(nk), 0);   // all_keys as a mark per SigKey position
    for (const auto& sn : snaps)
        for (int r : sn) seen[r] = 1;
    for (const Event& ev : events) seen[order_of[ev.key]] = 1;
    std::vector<int> all;   // SigKey positions, ascending
    for (int r = 0; r < nk; ++r)
        if (seen[r]) all.push_back(r);
    // each key's events in s order (the reference scans all events per key)
    std::vector<int> ev_first(keys.size() + 1, 0), ev_list(events.size());
    for (const Event& ev : events) ++ev_first[ev.key + 1];
    for (size_t k = 0; k < keys.size(); ++k) ev_first[k + 1] += ev_first[k];
    {
        std::vector<int> fill(ev_first.begin(), ev_first.end() - 1);
        for (int e = 0; e < static_cast<int>(events.size()); ++e) ev_list[fill[events[e].key]++] = e;
    }
    std::vector<visrt_mobile_row> table;
    for (int r : all) {
        const int k = by_rank[r];
        const KeyDef& kd = keys[k];
        bool open = std::binary_search(snaps.front().begin(), snaps.front().end(), r);
        double open_s = 0.0;
        int open_label = 0, open_prime = 0, open_block = -1;
        auto close_range = [&](double s_end, int end_label, int end_prime, int end_block) {
            visrt_mobile_row row{};
            row.order = kd.order;
            row.node = kd.node;
            row.vertex = kd.vertex;
            row.parent = kd.parent;
            row.s_start = open_s;
            row.s_end = s_end;
            row.label_start = open_label;
            row.prime_start = open_prime;
            row.label_end = end_label;
            row.prime_end = end_prime;
            row.blockage = open_block != -1 ? open_block : end_block;
            table.push_back(row);
        };
        for (int qi = ev_first[k]; qi < ev_first[k + 1]; ++qi) {
            const Event& ev = events[ev_list[qi]];
            if (ev.appearing) {
                if (!open) {
                    open = true;
                    open_s = ev.s;
                    open_label = ev.label;
                    open_prime = ev.vertical ? 1 : 0;
                    open_block = ev.blockage;
                }
            } else if (open) {
                close_range(ev.s, ev.label, ev.vertical ? 1 : 0, ev.blockage);
                open = false;
            }
        }
        if (open) close_range(length, 0, 0, -1);
    }

    phase("ranges");
    // ---- merge touching ranges (942-960) ------------------------------------
    auto par = [&](const visrt_mobile_row& r) { return r.parent < 0 ? nm.parent_rank[n] : nm.parent_rank[r.parent]; };
    auto nod = [&](const visrt_mobile_row& r) {
        return r.vertex < 0 ? nm.key_rank[r.node] : nm.key_rank[n + VISRT_MAX_VERTS * r.node + r.vertex];
    };
    std::sort(table.begin(), table.end(), [&](const visrt_mobile_row& a, const visrt_mobile_row& b) {
        if (a.order != b.order) return a.order < b.order;
        if (par(a) != par(b)) return par(a) < par(b);
        if (nod(a) != nod(b)) return nod(a) < nod(b);
        return a.s_start < b.s_start;
    });
    std::vector<visrt_mobile_row> merged;
    for (const visrt_mobile_row& row : table) {
        if (!merged.empty()) {
            visrt_mobile_row& last = merged.back();
            if (last.order == row.order && nod(last) == nod(row) && par(last) == par(row) &&
                last.blockage == row.blockage && row.s_start - last.s_end <= kBoundTol) {
                last.s_end = row.s_end;
                last.label_end = row.label_end;
                last.prime_end = row.prime_end;
                continue;
            }
        }
        merged.push_back(row);
    }
    phase("merge");
    stats.pairs = ns;
    stats.candidates = static_cast<int64_t>(events.size());
    stats.admitted = static_cast<int64_t>(merged.size());
    stats.tests_exec = gpu.tests;
    stats.sweeps = gpu.launches;
    stats.ms = gpu.ms;
    return merged;
}

}  // namespace
}  // namespace visrt

extern "C" int visrt_chain_reach(visrt_scene* sc, int64_t nq, const double* src_xyz, const visrt_entry* chains,
                                 uint8_t* reach, uint8_t* full, visrt_stats* stats, void* stream) {
    return visrt::capi_guard([&] {
        visrt::ScopedDevice dev(sc);
        const visrt::DevScene& ds = visrt::scene_dev(sc);
        for (int64_t q = 0; q < nq; ++q) {
            if (chains[q].order < 1 || chains[q].order > 4)
                throw visrt::UsageError("chain reach covers reflector chains of length 1..4");
            for (int c = 0; c <= chains[q].order; ++c)
                if (chains[q].chain[c] < 0 || chains[q].chain[c] >= ds.n) throw visrt::UsageError("bad face index");
            if (chains[q].plane < 0 || chains[q].plane > 2) throw visrt::UsageError("bad plane tag");
        }
        visrt::Gpu gpu{sc, ds, visrt::scene_device(sc), static_cast<cudaStream_t>(stream)};
        std::vector<double> src(src_xyz, src_xyz + 3 * nq);
        std::vector<visrt_entry> q(chains, chains + nq);
        std::vector<uint8_t> f;
        const std::vector<uint8_t> r = gpu.reach_paired(src, q, &f);
        std::copy(r.begin(), r.end(), reach);
        if (full) std::copy(f.begin(), f.end(), full);
        if (stats) {
            *stats = visrt_stats{};
            stats->pairs = nq;
            stats->tests_exec = gpu.tests;
            stats->ms = gpu.ms;
        }
    });
}

extern "C" int visrt_trajectory_table(visrt_scene* sc, int32_t nwp, const double* waypoints, int64_t nent,
                                      const visrt_entry* entries, int32_t max_order, const visrt_names* names,
                                      visrt_mobile_table** out, visrt_stats* stats, void* stream) {
    return visrt::capi_guard([&] {
        if (!out) throw visrt::UsageError("null output handle");
        *out = nullptr;
        visrt::ScopedDevice dev(sc);
        const visrt::DevScene& ds = visrt::scene_dev(sc);
        if (!names || !names->key_rank || !names->parent_rank || !names->building_rank)
            throw visrt::UsageError("visrt_names: every rank array is required");
        if (max_order < 1 || max_order > 4)
            throw visrt::UsageError("trajectory tables cover max_order 1..4");
        if (ds.n >= 65535) throw visrt::UsageError("trajectory tables index faces in 16 bits");
        for (int64_t e = 0; e < nent; ++e) {
            if (entries[e].order < 1 || entries[e].order > 4) continue;
            for (int c = 0; c <= entries[e].order; ++c)
                if (entries[e].chain[c] < 0 || entries[e].chain[c] >= ds.n) throw visrt::UsageError("bad face index");
        }
        visrt::Route route;
        route.nwp = nwp;
        route.w.assign(waypoints, waypoints + 3 * std::max(nwp, 0));
        // src/vistable.cpp:825-828
        if (nwp < 2 || route.total_length() <= visrt::kEps)
            throw visrt::VisError("trajectory must contain at least two distinct waypoints");
        visrt::Gpu gpu{sc, ds, visrt::scene_device(sc), static_cast<cudaStream_t>(stream)};
        visrt_stats st{};
        auto* t = new visrt_mobile_table;
        try {
            t->rows = visrt::trajectory_table(gpu, visrt::scene_host(sc), route, entries, nent, max_order, *names, st);
        } catch (...) {
            delete t;
            throw;
        }
        *out = t;
        if (stats) *stats = st;
    });
}

extern "C" int64_t visrt_mobile_table_rows(const visrt_mobile_table* t, visrt_mobile_row* rows, int64_t cap) {
    if (!t) return -1;
    const int64_t n = static_cast<int64_t>(t->rows.size());
    if (rows)
        for (int64_t k = 0; k < n && k < cap; ++k) rows[k] = t->rows[static_cast<size_t>(k)];
    return n;
}

extern "C" void visrt_mobile_table_destroy(visrt_mobile_table* t) { delete t; }
