// Culled any-hit occluder sweep shared by the matrix (K2), region (K4) and
// tree (K6) kernels.
//
// Two-level culling hierarchy (built once per scene by the host ingest):
//   * faces are Morton-ordered by the xy centre of their AABB and grouped in
//     tiles of 64 consecutive faces; every tile has a union culling box;
//   * level 1: 64 tile boxes per 64-bit candidate mask (a "chunk");
//   * level 2: the 64 member boxes of each candidate tile -> survivor mask;
//   * survivors run the exact FP64 predicate (device.h seg_hits) on records
//     stored in the same Morton order.
// Two traversals: per LANE (sweep_batch: every lane runs its own sweep, each
// warp iteration one 64-box fp32 SAT batch for every active lane) and per
// WARP (coop_any_hit: the 32 lanes split one segment's tile boxes, member
// boxes and exact survivors — used by K2w, K4w and the segment kernels,
// converged and with a short per-segment critical path). Tile boxes always
// live in shared memory; member boxes too when they fit (RESIDENT,
// N <= kResidentMaxBoxes), else they are read through L1/L2. No block barrier
// after the one-time TMA staging.
#pragma once

#include "device.h"

namespace visrt {

constexpr int kTile = 64;       // faces per tile / tiles per chunk (64-bit masks)
constexpr int kThreads = 256;   // 8 warps
constexpr unsigned kFull = 0xffffffffu;
constexpr int kResidentMaxBoxes = 6144;   // 192 KB of fp32 member boxes

// 64-box SAT batch -> mask (bit kk: box kk may meet the segment).
__device__ __forceinline__ unsigned long long sat64(const float* __restrict__ B, int cnt, const SegF& g) {
    unsigned long long mask = 0;
#pragma unroll 4
    for (int kk = 0; kk < cnt; ++kk)
        if (sat_maybe(B + kk * 8, g)) mask |= 1ull << kk;
    return mask;
}

#ifndef VISRT_CHUNK_BOXES
#define VISRT_CHUNK_BOXES 1   // 1: warp sweeps skip 4096-face chunks whose union box the segment misses
#endif
#ifndef VISRT_GROUPS
#define VISRT_GROUPS 1   // 1: non-resident sweeps cull 16-face groups (boxes in shared memory) before member boxes
#endif

struct SweepCtx {
    const float* tbox;   // [ntiles][8] (shared memory)
    const float* mbox;   // [n][8] member boxes (shared or global)
    const float* gbox;   // [ngroups][8] group boxes (shared memory; non-resident path only, else nullptr)
    const float* cbox;   // [nchunks][8] chunk boxes (shared memory): a chunk whose box the segment misses is skipped
    const float* tframe; // QRES: [ntiles][8] tile quantisation frames (shared memory), else nullptr
    const uint2* qbox;   // QRES: [n] 8-bit member boxes (shared memory), else nullptr
    int n, ntiles, nchunks, ngroups;
};

// Residency modes of the member boxes (template argument RES of the sweeping kernels).
constexpr int kStreamed = 0;   // member boxes read through L1/L2 (group level in shared memory)
constexpr int kResident = 1;   // fp32 member boxes in shared memory (N <= kResidentMaxBoxes)
constexpr int kQuantised = 2;  // 8-byte quantised member boxes + tile frames in shared memory
constexpr int kQuantisedMaxBoxes = 24576;   // 8 B/box + 64 B/tile: <= 200 KB, one CTA per SM
constexpr int kQThreads = 768;              // threads of a QUANTISED CTA (24 warps: the SM's only CTA)

// A segment in one tile's quantisation frame, coordinates doubled: M = 2 (m - o) inv,
// E = 2 e inv (ingest.cpp quantise_members). Against a quantised member box
// (lo, hi) the SAT reads D = M - (lo + hi), H = hi - lo: the same six axes as
// sat_maybe, all quantities scaled by 2 inv per axis (an affine map preserves
// intersection, so separating axes map to separating axes).
struct QSeg {
    float mx, my, mz, ex, ey, ez, ax, ay, az;
};

__device__ __forceinline__ QSeg make_qseg(const SegF& g, const float* __restrict__ F) {
    QSeg q;
    const float ix = 2.0f * F[4], iy = 2.0f * F[5], iz = 2.0f * F[6];
    q.mx = (g.mx - F[0]) * ix;
    q.my = (g.my - F[1]) * iy;
    q.mz = (g.mz - F[2]) * iz;
    q.ex = g.ex * ix;
    q.ey = g.ey * iy;
    q.ez = g.ez * iz;
    q.ax = fabsf(q.ex);
    q.ay = fabsf(q.ey);
    q.az = fabsf(q.ez);
    return q;
}

__device__ __forceinline__ bool qsat(uint2 b, const QSeg& g) {
    const float lx = static_cast<float>(b.x & 255u), ly = static_cast<float>((b.x >> 8) & 255u),
                lz = static_cast<float>((b.x >> 16) & 255u);
    const float ux = static_cast<float>(b.x >> 24), uy = static_cast<float>(b.y & 255u),
                uz = static_cast<float>((b.y >> 8) & 255u);
    const float dx = g.mx - (lx + ux), dy = g.my - (ly + uy), dz = g.mz - (lz + uz);
    const float hx = ux - lx, hy = uy - ly, hz = uz - lz;
    bool ok = fabsf(dx) <= hx + g.ax;
    ok &= fabsf(dy) <= hy + g.ay;
    ok &= fabsf(dz) <= hz + g.az;
    ok &= fabsf(__fmaf_rn(dy, g.ez, -dz * g.ey)) <= __fmaf_rn(hy, g.az, hz * g.ay);
    ok &= fabsf(__fmaf_rn(dz, g.ex, -dx * g.ez)) <= __fmaf_rn(hx, g.az, hz * g.ax);
    ok &= fabsf(__fmaf_rn(dx, g.ey, -dy * g.ex)) <= __fmaf_rn(hx, g.ay, hy * g.ax);
    return ok;
}

// Residency of a sweep: compile-time (RES >= 0, the kernel's template
// argument: dead paths drop out and the code stays i-cache sized) or read
// from the context (RES = -1).
template <int RES>
__device__ __forceinline__ bool use_groups(const SweepCtx& c) {
    return RES == kStreamed ? VISRT_GROUPS != 0 : (RES < 0 ? c.gbox != nullptr : false);
}
template <int RES>
__device__ __forceinline__ bool use_qbox(const SweepCtx& c) {
    return RES == kQuantised ? true : (RES < 0 ? c.qbox != nullptr : false);
}

// Member box k (Morton index) may meet segment g — any residency mode.
template <int RES = -1>
__device__ __forceinline__ bool member_maybe(const SweepCtx& c, int k, const SegF& g) {
    if (use_qbox<RES>(c)) return qsat(c.qbox[k], make_qseg(g, c.tframe + static_cast<size_t>(k >> 6) * 8));
    return sat_maybe(c.mbox + static_cast<size_t>(k) * 8, g);
}

// Per-lane state of one segment sweep.
struct Sweep {
    SegF g;
    int skip0, skip1;           // Morton-order indices never tested (the pair's own faces)
    int chunk, left;            // level-1 cursor (cyclic) and chunks still to scan
    int cbase;                  // first tile of the current candidate mask
    unsigned long long cand;    // candidate tiles of the current chunk

    __device__ void start(const SegF& seg, int s0, int s1, int start_chunk, int nchunks) {
        g = seg;
        skip0 = s0;
        skip1 = s1;
        chunk = start_chunk;
        left = nchunks;
        cand = 0;
        cbase = 0;
    }
    __device__ bool done() const { return cand == 0 && left == 0; }
};

// One 64-box batch of the lane's sweep. Returns the survivor mask of a
// level-2 tile (faces base..base+63 in Morton order, own faces removed) or 0
// after a level-1 chunk. `base` receives the tile's first face index.
__device__ __forceinline__ unsigned long long sweep_batch(Sweep& sw, const SweepCtx& c, int& base) {
    const float* ptr;
    int cnt;
    bool level1;
    if (sw.cand == 0) {
        level1 = true;
        const int t0 = sw.chunk * kTile;
        cnt = min(kTile, c.ntiles - t0);
        ptr = c.tbox + static_cast<size_t>(t0) * 8;
        base = t0;
    } else {
        level1 = false;
        const int t = sw.cbase + __ffsll(static_cast<long long>(sw.cand)) - 1;
        sw.cand &= sw.cand - 1;
        base = t * kTile;
        cnt = min(kTile, c.n - base);
        ptr = c.mbox + static_cast<size_t>(base) * 8;
    }
    unsigned long long mask = sat64(ptr, cnt, sw.g);
    if (level1) {
        sw.cand = mask;
        sw.cbase = base;
        sw.chunk = sw.chunk + 1 == c.nchunks ? 0 : sw.chunk + 1;
        --sw.left;
        return 0;
    }
    if (sw.skip0 >= base && sw.skip0 < base + kTile) mask &= ~(1ull << (sw.skip0 - base));
    if (sw.skip1 >= base && sw.skip1 < base + kTile) mask &= ~(1ull << (sw.skip1 - base));
    return mask;
}

// Warp-cooperative exact phase. Every lane holds the survivor mask of its own
// level-2 tile (Morton faces base..base+63) for its own segment a->b; the
// warp pools all survivors and deals them out 32 at a time, so each round
// issues 32 independent record loads and runs dense FP64 work instead of a
// divergent per-lane loop. Each lane's smallest hit (Morton index) comes back
// through `slot` (per-warp shared memory, 32 ints); with `all` every hit is
// also handed to on_hit(k, owner's payload) (blocker sets). Returns the lane's own
// first hit or -1. Must be called by all 32 lanes (inactive lanes: mask 0).
template <int MAXV, class OnHit>
__device__ __forceinline__ int coop_exact(const double* __restrict__ srec, unsigned long long mask, int base,
                                          double ax, double ay, double az, double bx, double by, double bz,
                                          int* slot, unsigned long long& tests, unsigned long long payload,
                                          OnHit&& on_hit) {
    constexpr int STRIDE = RecLayout<MAXV>::kStride;
    const int lane = threadIdx.x & 31;
    const int cnt = __popcll(mask);
    int pre = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(kFull, pre, o);
        if (lane >= o) pre += v;
    }
    const int total = __shfl_sync(kFull, pre, 31);
    if (total == 0) return -1;
    const int excl = pre - cnt;
    slot[lane] = 0x7fffffff;
    __syncwarp();
    for (int r = 0; r < total; r += 32) {
        const int gi = r + lane;
        // owner lane: the last lane whose exclusive prefix is <= gi
        int o = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
            const int e = __shfl_sync(kFull, excl, (o + step) & 31);
            if (o + step < 32 && e <= gi) o += step;
        }
        const unsigned long long om = __shfl_sync(kFull, mask, o);
        const int oexcl = __shfl_sync(kFull, excl, o);
        const int obase = __shfl_sync(kFull, base, o);
        const double oax = __shfl_sync(kFull, ax, o), oay = __shfl_sync(kFull, ay, o),
                     oaz = __shfl_sync(kFull, az, o);
        const double obx = __shfl_sync(kFull, bx, o), oby = __shfl_sync(kFull, by, o),
                     obz = __shfl_sync(kFull, bz, o);
        const unsigned long long opay = __shfl_sync(kFull, payload, o);
        if (gi < total) {
            // the (gi - oexcl)-th set bit of the owner's mask
            unsigned long long m = om;
            for (int q = gi - oexcl; q > 0; --q) m &= m - 1;
            const int k = obase + __ffsll(static_cast<long long>(m)) - 1;
            ++tests;
            if (seg_hits<MAXV>(srec + static_cast<size_t>(k) * STRIDE, oax, oay, oaz, obx, oby, obz)) {
                atomicMin(slot + o, k);
                on_hit(k, opay);
            }
        }
    }
    __syncwarp();
    const int h = slot[lane];
    return h == 0x7fffffff ? -1 : h;
}

// Warp-cooperative any-hit sweep of ONE segment (warp-uniform g / a->b):
// lanes split the 64 tile boxes of a chunk, then the 64 member boxes of each
// candidate tile; the survivors are compacted through the per-warp byte
// buffer `sv` (64 entries) and run the exact predicate 32 at a time. The
// sweep starts at the tile holding Morton face `home` (its neighbourhood is
// the likeliest blocker) and wraps around. Returns the Morton index of a
// blocking face (skip0 / skip1 never tested) or -1 when the segment is clear.
// Must be called by all 32 lanes with identical arguments.
// Non-resident any-hit sweep with the group level: per chunk the 64 tile
// boxes (2 per lane), then up to 8 candidate tiles at once — lane = (tile
// slot, group) tests one of the tile's 4 group boxes (shared memory) — then 2
// candidate groups at a time, a lane per member box (L1/L2) whose survivors
// run the exact test in place (at most 32 per round: no compaction needed).
// Same contract as coop_any_hit; which blocker is found first may differ.
// With `more` (2 ints), the round's second and third blockers of the segment
// come back too (-1 when none): K2w settles sibling sightlines with them.
template <int MAXV>
__device__ __forceinline__ int coop_any_hit_grouped(const SweepCtx& ctx, const double* __restrict__ srec,
                                                    const SegF& g, double ax, double ay, double az, double bx,
                                                    double by, double bz, int skip0, int skip1, int home,
                                                    unsigned long long& tests, unsigned long long& batches,
                                                    int* more = nullptr, int prio = -1) {
    constexpr int STRIDE = RecLayout<MAXV>::kStride;
    constexpr int GPT = kTile / kGroup;   // groups per tile (4)
    const int lane = threadIdx.x & 31;
    const int home_tile = home < 0 ? 0 : home / kTile;
    const int hc = home_tile / kTile;
    for (int cc = 0; cc < ctx.nchunks; ++cc) {
        const int c = hc + cc < ctx.nchunks ? hc + cc : hc + cc - ctx.nchunks;
        const int t0 = c * kTile;
        const int tc = min(kTile, ctx.ntiles - t0);
        if (VISRT_CHUNK_BOXES && ctx.nchunks > 1 && !sat_maybe(ctx.cbox + static_cast<size_t>(c) * 8, g)) continue;
        const bool h0 = lane < tc && sat_maybe(ctx.tbox + static_cast<size_t>(t0 + lane) * 8, g);
        const bool h1 = lane + 32 < tc && sat_maybe(ctx.tbox + static_cast<size_t>(t0 + lane + 32) * 8, g);
        unsigned long long cand = static_cast<unsigned long long>(__ballot_sync(kFull, h0)) |
                                  (static_cast<unsigned long long>(__ballot_sync(kFull, h1)) << 32);
        if (cc == 0) {   // the home tile first: rotate the mask so it starts there
            const int r = home_tile - t0;
            cand = r ? ((cand >> r) | (cand << (64 - r))) : cand;
        }
        const int rot = cc == 0 ? home_tile - t0 : 0;
        // `prio`'s tile joins the first batch (second slot)
        int ptile = -1;
        if (prio >= 0) {
            const int pt = prio / kTile - t0;
            if (pt >= 0 && pt < 64 && pt != home_tile - t0) {
                int pb = pt - rot;
                if (pb < 0) pb += 64;
                if ((cand >> pb) & 1ull) {
                    cand &= ~(1ull << pb);
                    ptile = t0 + pt;
                }
            }
        }
        ++batches;
        while (cand || ptile >= 0) {
            // up to 8 candidate tiles -> lane (slot = lane / 4, group = lane % 4)
            int my_tile = -1;
#pragma unroll
            for (int q = 0; q < 32 / GPT; ++q) {
                int t_abs;
                if (ptile >= 0 && (q == 1 || !cand)) {
                    t_abs = ptile;
                    ptile = -1;
                } else {
                    if (!cand) break;
                    const int b = __ffsll(static_cast<long long>(cand)) - 1;
                    cand &= cand - 1;
                    int t = b + rot;
                    if (t >= 64) t -= 64;
                    t_abs = t0 + t;
                }
                if (q == lane / GPT) my_tile = t_abs;
            }
            const int grp = my_tile * GPT + (lane % GPT);
            const bool gv = my_tile >= 0 && grp < ctx.ngroups && sat_maybe(ctx.gbox + static_cast<size_t>(grp) * 8, g);
            unsigned gm = __ballot_sync(kFull, gv);
            ++batches;
            while (gm) {
                // two candidate groups per round: lanes 0-15 / 16-31
                const int la = __ffs(gm) - 1;
                gm &= gm - 1;
                const int lb = gm ? __ffs(gm) - 1 : -1;
                if (lb >= 0) gm &= gm - 1;
                const int ga = __shfl_sync(kFull, grp, la);
                const int gb = __shfl_sync(kFull, grp, lb < 0 ? la : lb);
                const int mg = lane < kGroup ? ga : (lb < 0 ? -1 : gb);
                const int m = mg * kGroup + (lane & (kGroup - 1));
                bool v = mg >= 0 && m < ctx.n && m != skip0 && m != skip1 &&
                         sat_maybe(ctx.mbox + static_cast<size_t>(m) * 8, g);
                if (v) {
                    ++tests;
                    v = seg_hits<MAXV>(srec + static_cast<size_t>(m) * STRIDE, ax, ay, az, bx, by, bz);
                }
                const unsigned hb = __ballot_sync(kFull, v);
                ++batches;
                if (hb) {
                    if (more) {
                        const unsigned r1 = hb & (hb - 1), r2 = r1 & (r1 - 1);
                        more[0] = r1 ? __shfl_sync(kFull, m, __ffs(r1) - 1) : -1;
                        more[1] = r2 ? __shfl_sync(kFull, m, __ffs(r2) - 1) : -1;
                    }
                    return __shfl_sync(kFull, m, __ffs(hb) - 1);
                }
            }
        }
    }
    return -1;
}

template <int MAXV, int FIRST = 0, int RES = -1>
__device__ __forceinline__ int coop_any_hit(const SweepCtx& ctx, const double* __restrict__ srec, const SegF& g,
                                            double ax, double ay, double az, double bx, double by, double bz,
                                            int skip0, int skip1, int home, unsigned char* sv,
                                            unsigned long long& tests, unsigned long long& batches) {
    if (use_groups<RES>(ctx)) return coop_any_hit_grouped<MAXV>(ctx, srec, g, ax, ay, az, bx, by, bz, skip0, skip1, home, tests,
                                                   batches);
    constexpr int STRIDE = RecLayout<MAXV>::kStride;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int home_tile = home < 0 ? 0 : home / kTile;
    const int hc = home_tile / kTile;
    int hit = -1;
    for (int cc = 0; cc < ctx.nchunks && hit < 0; ++cc) {
        const int c = hc + cc < ctx.nchunks ? hc + cc : hc + cc - ctx.nchunks;
        const int t0 = c * kTile;
        const int tc = min(kTile, ctx.ntiles - t0);
        if (VISRT_CHUNK_BOXES && ctx.nchunks > 1 && !sat_maybe(ctx.cbox + static_cast<size_t>(c) * 8, g)) continue;
        const bool h0 = lane < tc && sat_maybe(ctx.tbox + static_cast<size_t>(t0 + lane) * 8, g);
        const bool h1 = lane + 32 < tc && sat_maybe(ctx.tbox + static_cast<size_t>(t0 + lane + 32) * 8, g);
        unsigned long long cand = static_cast<unsigned long long>(__ballot_sync(kFull, h0)) |
                                  (static_cast<unsigned long long>(__ballot_sync(kFull, h1)) << 32);
        unsigned long long later = 0;
        if (cc == 0) {   // the home tile first, wrap around after
            const unsigned long long below = (1ull << (home_tile - t0)) - 1ull;
            later = cand & below;
            cand &= ~below;
        }
        ++batches;
        while ((cand | later) && hit < 0) {
            if (!cand) {
                cand = later;
                later = 0;
            }
            const int base = (t0 + __ffsll(static_cast<long long>(cand)) - 1) * kTile;
            cand &= cand - 1;
            const int mc = min(kTile, ctx.n - base);
            const int m0 = base + lane, m1 = base + lane + 32;
            bool v0, v1;
            if (use_qbox<RES>(ctx)) {
                const QSeg qs = make_qseg(g, ctx.tframe + static_cast<size_t>(base >> 6) * 8);
                v0 = lane < mc && m0 != skip0 && m0 != skip1 && qsat(ctx.qbox[m0], qs);
                v1 = lane + 32 < mc && m1 != skip0 && m1 != skip1 && qsat(ctx.qbox[m1], qs);
            } else {
                v0 = lane < mc && m0 != skip0 && m0 != skip1 && sat_maybe(ctx.mbox + static_cast<size_t>(m0) * 8, g);
                v1 = lane + 32 < mc && m1 != skip0 && m1 != skip1 &&
                     sat_maybe(ctx.mbox + static_cast<size_t>(m1) * 8, g);
            }
            const unsigned lo = __ballot_sync(kFull, v0), hi = __ballot_sync(kFull, v1);
            ++batches;
            const int clo = __popc(lo), tot = clo + __popc(hi);
            if (tot == 0) continue;
            if (v0) sv[__popc(lo & lt)] = static_cast<unsigned char>(lane);
            if (v1) sv[clo + __popc(hi & lt)] = static_cast<unsigned char>(32 + lane);
            __syncwarp();
            // FIRST > 0: a narrow first round (the home-ordered first survivors
            // are the likeliest blockers), then rounds of 32
            for (int r = 0; r < tot && hit < 0; r += (FIRST > 0 && r == 0) ? FIRST : 32) {
                const int width = (FIRST > 0 && r == 0) ? FIRST : 32;
                const int idx = (lane < width && r + lane < tot) ? sv[r + lane] : -1;
                bool h = false;
                if (idx >= 0) {
                    ++tests;
                    h = seg_hits<MAXV>(srec + static_cast<size_t>(base + idx) * STRIDE, ax, ay, az, bx, by, bz);
                }
                const unsigned hb = __ballot_sync(kFull, h);
                if (hb) hit = __shfl_sync(kFull, base + idx, __ffs(hb) - 1);
            }
            __syncwarp();
        }
    }
    return hit;
}

// sat_maybe against the box dilated by R on every axis (conservative for any
// segment within distance R of g: the box grown by R contains the box's
// Minkowski sum with the R-ball).
__device__ __forceinline__ bool sat_maybe_dil(const float* __restrict__ B, const SegF& g, float R) {
    const float dx = g.mx - B[0], dy = g.my - B[1], dz = g.mz - B[2];
    const float hx = B[4] + R, hy = B[5] + R, hz = B[6] + R;
    bool ok = fabsf(dx) <= hx + g.ax;
    ok &= fabsf(dy) <= hy + g.ay;
    ok &= fabsf(dz) <= hz + g.az;
    ok &= fabsf(__fmaf_rn(dy, g.ez, -dz * g.ey)) <= __fmaf_rn(hy, g.az, hz * g.ay);
    ok &= fabsf(__fmaf_rn(dz, g.ex, -dx * g.ez)) <= __fmaf_rn(hx, g.az, hz * g.ax);
    ok &= fabsf(__fmaf_rn(dx, g.ey, -dy * g.ex)) <= __fmaf_rn(hx, g.ay, hy * g.ax);
    return ok;
}

// Collecting sweep of a FAN: every face (Morton index, `skip` excluded) whose
// culling box, dilated by R, meets the axis segment g — i.e. every face that
// could meet ANY segment within distance R of g. No exact tests, no early
// exit. The indices go to `list` (per-warp shared memory, `cap` entries) in
// traversal order; returns their count, or -1 when more than `cap` faces
// qualify or the member boxes are quantised (the caller falls back to
// per-sightline sweeps). Warp-uniform arguments; all 32 lanes.
template <int RES = -1>
__device__ __forceinline__ int coop_collect(const SweepCtx& ctx, const SegF& g, float R, int skip, int* list,
                                            int cap, unsigned long long& batches) {
    if (use_qbox<RES>(ctx)) return -1;
    constexpr int GPT = kTile / kGroup;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    int cnt = 0;
    auto append = [&](bool v, int m) -> bool {   // false: overflow
        const unsigned b = __ballot_sync(kFull, v);
        if (v && cnt + __popc(b & lt) < cap) list[cnt + __popc(b & lt)] = m;
        cnt += __popc(b);
        return cnt <= cap;
    };
    for (int c = 0; c < ctx.nchunks; ++c) {
        const int t0 = c * kTile;
        const int tc = min(kTile, ctx.ntiles - t0);
        if (VISRT_CHUNK_BOXES && ctx.nchunks > 1 && !sat_maybe_dil(ctx.cbox + static_cast<size_t>(c) * 8, g, R))
            continue;
        const bool h0 = lane < tc && sat_maybe_dil(ctx.tbox + static_cast<size_t>(t0 + lane) * 8, g, R);
        const bool h1 = lane + 32 < tc && sat_maybe_dil(ctx.tbox + static_cast<size_t>(t0 + lane + 32) * 8, g, R);
        unsigned long long cand = static_cast<unsigned long long>(__ballot_sync(kFull, h0)) |
                                  (static_cast<unsigned long long>(__ballot_sync(kFull, h1)) << 32);
        ++batches;
        if (use_groups<RES>(ctx)) {   // streamed: 8 candidate tiles x 4 groups per round, then 2 groups of members
            while (cand) {
                int my_tile = -1;
#pragma unroll
                for (int q = 0; q < 32 / GPT; ++q) {
                    if (!cand) break;
                    const int t = t0 + __ffsll(static_cast<long long>(cand)) - 1;
                    cand &= cand - 1;
                    if (q == lane / GPT) my_tile = t;
                }
                const int grp = my_tile * GPT + (lane % GPT);
                const bool gv = my_tile >= 0 && grp < ctx.ngroups &&
                                sat_maybe_dil(ctx.gbox + static_cast<size_t>(grp) * 8, g, R);
                unsigned gm = __ballot_sync(kFull, gv);
                ++batches;
                while (gm) {
                    const int la = __ffs(gm) - 1;
                    gm &= gm - 1;
                    const int lb = gm ? __ffs(gm) - 1 : -1;
                    if (lb >= 0) gm &= gm - 1;
                    const int ga = __shfl_sync(kFull, grp, la);
                    const int gb = __shfl_sync(kFull, grp, lb < 0 ? la : lb);
                    const int mg = lane < kGroup ? ga : (lb < 0 ? -1 : gb);
                    const int m = mg * kGroup + (lane & (kGroup - 1));
                    const bool v = mg >= 0 && m < ctx.n && m != skip &&
                                   sat_maybe_dil(ctx.mbox + static_cast<size_t>(m) * 8, g, R);
                    ++batches;
                    if (!append(v, m)) return -1;
                }
            }
        } else {   // member boxes in shared memory: 64 per candidate tile
            while (cand) {
                const int base = (t0 + __ffsll(static_cast<long long>(cand)) - 1) * kTile;
                cand &= cand - 1;
                const int mc = min(kTile, ctx.n - base);
                const int m0 = base + lane, m1 = base + lane + 32;
                const bool v0 = lane < mc && m0 != skip && sat_maybe_dil(ctx.mbox + static_cast<size_t>(m0) * 8, g, R);
                const bool v1 =
                    lane + 32 < mc && m1 != skip && sat_maybe_dil(ctx.mbox + static_cast<size_t>(m1) * 8, g, R);
                ++batches;
                if (!append(v0, m0) || !append(v1, m1)) return -1;
            }
        }
    }
    return cnt;
}

// A CONE: every segment from the apex S to a point of a target face F lies in
// the pyramid hull(S, F). A point at parameter t of such a segment is within
// t * r of the axis point S + t (c - S) (c the centre of F's box, r its
// half-diagonal), so the pyramid lies inside the union of three tapered
// pieces: axis t in [0, 1/2] dilated by r/2, [1/2, 3/4] by 3r/4, [3/4, 1] by r.
// A box that misses all three pieces (sat_maybe_dil) cannot meet any segment
// S -> F: its face can block none of them.
struct ConeF {
    SegF g[3];
    float R[3];
};

__device__ __forceinline__ bool cone_maybe(const float* __restrict__ B, const ConeF& c) {
    return sat_maybe_dil(B, c.g[0], c.R[0]) | sat_maybe_dil(B, c.g[1], c.R[1]) | sat_maybe_dil(B, c.g[2], c.R[2]);
}

// A warp's cone list: up to cap entries in its slice of a global buffer (L1
// resident while the warp scans it; a shared-memory head was measured slower:
// it shrinks the L1 the streamed member boxes live in).
struct ConeBuf {
    float4* g;
    int cap;
    __device__ __forceinline__ float4* at(int c) const { return g + 2 * c; }
};

// Collecting sweep of a cone: every face (Morton index, `skip` excluded) whose
// culling box may meet the cone, written to `out` (global, per warp: entry e =
// out[2e] {cx, cy, cz, index as int bits}, out[2e + 1] {hx, hy, hz, 0} — the
// member box with its face) in traversal order. Returns the count, or -1 when
// more than `cap` faces qualify or the member boxes are quantised. No exact
// tests, no early exit. Warp-uniform arguments; all 32 lanes.
template <int RES = -1>
__device__ __forceinline__ int coop_collect_cone(const SweepCtx& ctx, const ConeF& cone, int skip, ConeBuf out,
                                                 unsigned long long& batches) {
    const int cap = out.cap;
    if (use_qbox<RES>(ctx)) return -1;
    constexpr int GPT = kTile / kGroup;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    int cnt = 0;
    auto append = [&](bool v, int m) -> bool {   // false: overflow
        const unsigned b = __ballot_sync(kFull, v);
        const int at = cnt + __popc(b & lt);
        if (v && at < cap) {
            const float4* B = reinterpret_cast<const float4*>(ctx.mbox + static_cast<size_t>(m) * 8);
            float4 b0 = B[0];
            b0.w = __int_as_float(m);
            float4* e = out.at(at);
            e[0] = b0;
            e[1] = B[1];
        }
        cnt += __popc(b);
        return cnt <= cap;
    };
    for (int c = 0; c < ctx.nchunks; ++c) {
        const int t0 = c * kTile;
        const int tc = min(kTile, ctx.ntiles - t0);
        if (VISRT_CHUNK_BOXES && ctx.nchunks > 1 && !cone_maybe(ctx.cbox + static_cast<size_t>(c) * 8, cone)) continue;
        const bool h0 = lane < tc && cone_maybe(ctx.tbox + static_cast<size_t>(t0 + lane) * 8, cone);
        const bool h1 = lane + 32 < tc && cone_maybe(ctx.tbox + static_cast<size_t>(t0 + lane + 32) * 8, cone);
        unsigned long long cand = static_cast<unsigned long long>(__ballot_sync(kFull, h0)) |
                                  (static_cast<unsigned long long>(__ballot_sync(kFull, h1)) << 32);
        ++batches;
        if (use_groups<RES>(ctx)) {   // streamed: 8 candidate tiles x 4 groups per round, then 2 groups of members
            while (cand) {
                int my_tile = -1;
#pragma unroll
                for (int q = 0; q < 32 / GPT; ++q) {
                    if (!cand) break;
                    const int t = t0 + __ffsll(static_cast<long long>(cand)) - 1;
                    cand &= cand - 1;
                    if (q == lane / GPT) my_tile = t;
                }
                const int grp = my_tile * GPT + (lane % GPT);
                const bool gv = my_tile >= 0 && grp < ctx.ngroups &&
                                cone_maybe(ctx.gbox + static_cast<size_t>(grp) * 8, cone);
                unsigned gm = __ballot_sync(kFull, gv);
                ++batches;
                while (gm) {
                    const int la = __ffs(gm) - 1;
                    gm &= gm - 1;
                    const int lb = gm ? __ffs(gm) - 1 : -1;
                    if (lb >= 0) gm &= gm - 1;
                    const int ga = __shfl_sync(kFull, grp, la);
                    const int gb = __shfl_sync(kFull, grp, lb < 0 ? la : lb);
                    const int mg = lane < kGroup ? ga : (lb < 0 ? -1 : gb);
                    const int m = mg * kGroup + (lane & (kGroup - 1));
                    const bool v = mg >= 0 && m < ctx.n && m != skip &&
                                   cone_maybe(ctx.mbox + static_cast<size_t>(m) * 8, cone);
                    ++batches;
                    if (!append(v, m)) return -1;
                }
            }
        } else {   // member boxes in shared memory: 64 per candidate tile
            while (cand) {
                const int base = (t0 + __ffsll(static_cast<long long>(cand)) - 1) * kTile;
                cand &= cand - 1;
                const int mc = min(kTile, ctx.n - base);
                const int m0 = base + lane, m1 = base + lane + 32;
                const bool v0 = lane < mc && m0 != skip && cone_maybe(ctx.mbox + static_cast<size_t>(m0) * 8, cone);
                const bool v1 = lane + 32 < mc && m1 != skip && cone_maybe(ctx.mbox + static_cast<size_t>(m1) * 8, cone);
                ++batches;
                if (!append(v0, m0) || !append(v1, m1)) return -1;
            }
        }
    }
    return cnt;
}

// sat_maybe on a cone-list entry (two float4: centre, half extent)
__device__ __forceinline__ bool sat_maybe4(const float4& c, const float4& h, const SegF& g) {
    const float dx = g.mx - c.x, dy = g.my - c.y, dz = g.mz - c.z;
    bool ok = fabsf(dx) <= h.x + g.ax;
    ok &= fabsf(dy) <= h.y + g.ay;
    ok &= fabsf(dz) <= h.z + g.az;
    ok &= fabsf(__fmaf_rn(dy, g.ez, -dz * g.ey)) <= __fmaf_rn(h.y, g.az, h.z * g.ay);
    ok &= fabsf(__fmaf_rn(dz, g.ex, -dx * g.ez)) <= __fmaf_rn(h.x, g.az, h.z * g.ax);
    ok &= fabsf(__fmaf_rn(dx, g.ey, -dy * g.ex)) <= __fmaf_rn(h.x, g.ay, h.y * g.ax);
    return ok;
}

// Block setup: stage the tile boxes (and the member boxes when resident,
// fp32 or quantised) in shared memory with TMA bulk copies (cp.async.bulk,
// one mbarrier). Shared layout: tile boxes | members (fp32 [n][8] RESIDENT,
// group boxes STREAMED, tile frames + quantised boxes QUANTISED) | chunk boxes.
template <int RES>
__device__ __forceinline__ SweepCtx sweep_setup(const DevScene& s, float* smem, uint64_t* bar) {
    SweepCtx c;
    c.n = s.n;
    c.ntiles = s.ntiles;
    c.nchunks = s.nchunks;
    float* st = smem;
    float* sm = smem + static_cast<size_t>(s.ntiles) * 8;   // member boxes (RESIDENT) or group boxes
    constexpr bool kGroups = RES == kStreamed && VISRT_GROUPS;
    c.ngroups = s.ngroups;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    const uint32_t tb = static_cast<uint32_t>(s.ntiles) * 32u;
    const uint32_t qb = static_cast<uint32_t>((s.n + 1) / 2) * 16u;
    const uint32_t mb = RES == kResident ? static_cast<uint32_t>(s.n) * 32u
                      : RES == kQuantised ? tb + qb
                                         : (kGroups ? static_cast<uint32_t>(s.ngroups) * 32u : 0u);
    if (threadIdx.x == 0) {
        const uint32_t cb = static_cast<uint32_t>(s.nchunks) * 32u;
        mbar_expect_tx(bar, tb + mb + cb);
        for (uint32_t off = 0; off < tb; off += 32768u)
            bulk_g2s(reinterpret_cast<char*>(st) + off, reinterpret_cast<const char*>(s.tbox) + off,
                     min(32768u, tb - off), bar);
        if (RES == kQuantised) {
            for (uint32_t off = 0; off < tb; off += 32768u)
                bulk_g2s(reinterpret_cast<char*>(sm) + off, reinterpret_cast<const char*>(s.tframe) + off,
                         min(32768u, tb - off), bar);
            for (uint32_t off = 0; off < qb; off += 32768u)
                bulk_g2s(reinterpret_cast<char*>(sm) + tb + off, reinterpret_cast<const char*>(s.qbox) + off,
                         min(32768u, qb - off), bar);
        } else {
            const char* msrc = reinterpret_cast<const char*>(RES == kResident ? s.sbox : s.gbox);
            for (uint32_t off = 0; off < mb; off += 32768u)
                bulk_g2s(reinterpret_cast<char*>(sm) + off, msrc + off, min(32768u, mb - off), bar);
        }
        bulk_g2s(reinterpret_cast<char*>(sm) + mb, reinterpret_cast<const char*>(s.cbox), cb, bar);
    }
    mbar_wait(bar, 0);
    c.tbox = st;
    c.mbox = RES == kResident ? sm : s.sbox;
    c.gbox = kGroups ? sm : nullptr;
    c.tframe = RES == kQuantised ? sm : nullptr;
    c.qbox = RES == kQuantised ? reinterpret_cast<const uint2*>(reinterpret_cast<const char*>(sm) + tb) : nullptr;
    c.cbox = reinterpret_cast<const float*>(reinterpret_cast<const char*>(sm) + mb);
    return c;
}

inline size_t sweep_smem_bytes(int n, int ntiles, int res) {
    const size_t groups = VISRT_GROUPS ? static_cast<size_t>((n + kGroup - 1) / kGroup) : 0;
    const size_t chunks = (static_cast<size_t>(ntiles) + kTile - 1) / kTile;
    const size_t members = res == kResident ? static_cast<size_t>(n) * 32
                         : res == kQuantised ? static_cast<size_t>(ntiles) * 32 + static_cast<size_t>((n + 1) / 2) * 16
                                            : groups * 32;
    return static_cast<size_t>(ntiles) * 32 + members + chunks * 32 + 128;
}

// Morton chunk holding original face f (a sweep starting there meets the
// face's own neighbourhood — the likeliest blockers — first).
__device__ __forceinline__ int home_chunk(const DevScene& s, int f) {
    return f < 0 ? 0 : (s.inv[f] / kTile) / kTile;
}

}  // namespace visrt
