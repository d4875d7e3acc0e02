// (1) Inter-visibility matrix kernels for sm_100a.
//
//   K1 k-prefilter   first_order_pair's gate (src/vismatrix.cpp:597-604:
//                    non-oblique, mutually_front 160-169, required_planes
//                    171-181) over all i<j, ordered prefix-sum compaction
//                    (cub::DeviceSelect) into a candidate list.
//   K2w k_pair_bits_warp (default) occlusion_judgment's Occluded verdict
//                    (253-302) with early exit, one WARP per pair: warp blocker
//                    cache tested on all sightlines at once, then one
//                    warp-cooperative culled sweep (sweep.h hierarchy: tile
//                    boxes, member boxes, exact survivors) per unresolved
//                    sightline; a found blocker settles every other sightline
//                    it blocks. A pair stops at its first clear (or degenerate)
//                    sightline.
//   K2 k_pair_bits   the same bit with one LANE per pair state machine and
//                    per-lane culled sweeps (VISRT_K2_WARP=0; kept for A/B).
//   K2d k_pair_detail Visible / Partial / Occluded + blocker sets (no early exit).
//
// All geometry is the reference's FP64 predicate with explicit _rn intrinsics
// (device.h), so every decision is bit-identical to the CPU oracle.
#include <algorithm>
#include <cstdlib>

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "device.h"
#include "sweep.h"

namespace visrt {




// Sightline `ord` of pair (i, j) in the kernel's exploration order: the
// centroid pair first, then the diagonal grid pairs, then the vertex pairs
// (any order is valid: the verdict counts blocked sightlines, and the bit only
// needs one unblocked one). Returns the reference endpoint pair.
__device__ __forceinline__ void sightline_endpoints(const DevScene& s, int i, int j, int nr, int na,
                                                    int grid, int ord, double& ax, double& ay,
                                                    double& az, double& bx, double& by, double& bz) {
    int ri, ai;
    if (ord == 0) {
        ri = nr;
        ai = na;
    } else if (ord <= grid) {
        ri = nr + ord;
        ai = na + ord;
    } else {
        const int v = ord - 1 - grid;
        ri = v / na;
        ai = v % na;
    }
    const double* P = s.samples + (static_cast<size_t>(i) * kMaxSamples + ri) * 3;
    const double* Q = s.samples + (static_cast<size_t>(j) * kMaxSamples + ai) * 3;
    ax = P[0]; ay = P[1]; az = P[2];
    bx = Q[0]; by = Q[1]; bz = Q[2];
}

// norm(q - p) <= kEps (src/vismatrix.cpp:278-280): never blocked.
__device__ __forceinline__ bool degenerate(double ax, double ay, double az, double bx, double by,
                                           double bz) {
    const double dx = dsub(bx, ax), dy = dsub(by, ay), dz = dsub(bz, az);
    return __dsqrt_rn(dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz))) <= kEps;
}

__device__ __forceinline__ void set_pair_bit(unsigned long long* bits, int words, int i, int j) {
    atomicOr(bits + static_cast<size_t>(i) * words + (j >> 6), 1ull << (j & 63));
    atomicOr(bits + static_cast<size_t>(j) * words + (i >> 6), 1ull << (i & 63));
}

// Faces whose (exact) AABBs are more than 1e-6 m apart have no coincident
// samples, hence no degenerate sightline (samples lie in the face AABB up to
// ~1e-11 m of rounding).
__device__ __forceinline__ bool may_touch(const DevScene& s, int i, int j) {
    const double* A = s.aabb + 6 * static_cast<size_t>(i);
    const double* B = s.aabb + 6 * static_cast<size_t>(j);
    bool sep = false;
#pragma unroll
    for (int d = 0; d < 3; ++d) sep |= (B[d] > A[3 + d] + 1e-6) | (A[d] > B[3 + d] + 1e-6);
    return !sep;
}

#ifndef VISRT_K2_MINB
#define VISRT_K2_MINB 3   // CTAs per SM the register budget targets (80 regs at 3)
#endif
#ifndef VISRT_K2_BC
#define VISRT_K2_BC 4     // blocker-cache entries per lane (4 measured best: r01 k2sweep)
#endif

template <int MAXV, bool RESIDENT>
__global__ void __launch_bounds__(kThreads, VISRT_K2_MINB) k_pair_bits(PairArgs a) {
    constexpr int STRIDE = RecLayout<MAXV>::kStride;
    constexpr int BC = VISRT_K2_BC;
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t bar[1];
    const DevScene& s = a.s;
    const int n = s.n;
    const int lane = threadIdx.x & 31;
    const SweepCtx ctx = sweep_setup<RESIDENT>(s, smem, bar);

    bool active = false, exhausted = false;
    long long pidx = 0;
    int pi = 0, pj = 0, si = 0, sj = 0, nr = 0, na = 0, grid = 0, S = 0, ord = 0;
    int bc[BC];               // blocker cache (Morton indices of the last blockers, most recent first)
#pragma unroll
    for (int q = 0; q < BC; ++q) bc[q] = -1;
    double ax = 0, ay = 0, az = 0, bx = 0, by = 0, bz = 0;
    Sweep sw{};
    unsigned long long tests = 0, sweeps = 0, batches = 0;

    auto finish = [&](bool occluded) {
        if (!occluded) set_pair_bit(a.bits, s.words, pi, pj);
        if (a.cbit) a.cbit[pidx] = occluded ? 0 : 1;
        active = false;
    };
    auto exact = [&](int k) {
        ++tests;
        return seg_hits<MAXV>(s.srec + static_cast<size_t>(k) * STRIDE, ax, ay, az, bx, by, bz);
    };
    // Next sightline of the current pair. Sightlines a cached blocker already
    // blocks are settled on the spot (one exact test each); the first one the
    // cache does not block starts a culled sweep over every other face.
    auto advance = [&]() {
        for (;;) {
            if (++ord == S) {
                finish(true);   // every sightline blocked: Occluded
                return;
            }
            sightline_endpoints(s, pi, pj, nr, na, grid, ord, ax, ay, az, bx, by, bz);
            const SegF g = make_segf(s, ax, ay, az, bx, by, bz);
            int hitc = -1;
#pragma unroll
            for (int q = 0; q < BC; ++q)
                if (hitc < 0 && bc[q] >= 0 && bc[q] != si && bc[q] != sj &&
                    sat_maybe(ctx.mbox + static_cast<size_t>(bc[q]) * 8, g) && exact(bc[q]))
                    hitc = q;
            if (hitc >= 0) {
#pragma unroll
                for (int q = 1; q < BC; ++q)
                    if (q == hitc) {   // move to front
                        const int t = bc[0];
                        bc[0] = bc[q];
                        bc[q] = t;
                    }
                continue;
            }
            sw.start(g, si, sj, home_chunk(s, pi), ctx.nchunks);
            ++sweeps;
            return;
        }
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
                if (my >= a.npairs) {
                    exhausted = true;
                } else {
                    pidx = my;
                    if (a.ci) {
                        pi = a.ci[my];
                        pj = a.cj[my];
                    } else {
                        pair_from_index(my, n, pi, pj);
                    }
                    si = s.inv[pi];
                    sj = s.inv[pj];
                    nr = s.nv[pi];
                    na = s.nv[pj];
                    grid = min(s.ns[pi] - nr - 1, s.ns[pj] - na - 1);
                    S = nr * na + 1 + grid;
                    bool degen = false;
                    if (may_touch(s, pi, pj)) {
                        for (int o = 0; o < S && !degen; ++o) {
                            sightline_endpoints(s, pi, pj, nr, na, grid, o, ax, ay, az, bx, by, bz);
                            degen = degenerate(ax, ay, az, bx, by, bz);
                        }
                    }
                    active = true;
                    if (degen) {
                        finish(false);   // a degenerate sightline is never blocked
                    } else {
                        ord = -1;
                        advance();
                    }
                }
            }
            need = __ballot_sync(kFull, !active && !exhausted);
        }
    };

    refill();
    for (;;) {
        if (active) {
            ++batches;
            int base;
            unsigned long long mask = sweep_batch(sw, ctx, base);
            int hk = -1;
            while (mask) {
                const int kk = __ffsll(static_cast<long long>(mask)) - 1;
                mask &= mask - 1;
                if (exact(base + kk)) {
                    hk = base + kk;
                    break;
                }
            }
            if (hk >= 0) {
                if (hk != bc[0]) {
#pragma unroll
                    for (int q = BC - 1; q > 0; --q) bc[q] = bc[q - 1];
                    bc[0] = hk;
                }
                advance();
            } else if (sw.done()) {
                finish(false);   // a sightline clear of every occluder
            }
        }
        refill();
        if (!__any_sync(kFull, active || !exhausted)) break;
    }
    for (int o = 16; o > 0; o >>= 1) {
        tests += __shfl_down_sync(kFull, tests, o);
        sweeps += __shfl_down_sync(kFull, sweeps, o);
        batches += __shfl_down_sync(kFull, batches, o);
    }
    if (lane == 0) {
        atomicAdd(&a.counter[1], tests);
        atomicAdd(&a.counter[2], sweeps);
        atomicAdd(&a.counter[3], batches);
    }
}

// K2w: the same verdict bit with a WARP per pair. Lane l owns sightlines
// l, l+32, l+64 (S <= 89). A warp-uniform cache of the last kWC blockers is
// tested on every sightline at once; each still-unresolved sightline then gets
// ONE warp-cooperative culled sweep (lanes split the 64 tile boxes of a chunk,
// then the 64 member boxes of each candidate tile, then the survivors' exact
// tests), and the blocker it finds is immediately tested on every other
// unresolved sightline of the pair. The pair ends at the first clear sightline
// (bit = 1) or when every sightline is blocked — the same bit as the lane
// kernel, with converged SAT/exact work instead of 32 divergent state machines.
#ifndef VISRT_K2W_MINB
#define VISRT_K2W_MINB 3
#endif
#ifndef VISRT_K2W_WC
#define VISRT_K2W_WC 4      // warp blocker-cache entries (with 16-pair grabs; 2/3/4/5/6/8 swept: 4 best)
#endif
#ifndef VISRT_K2W_RSAT
#define VISRT_K2W_RSAT 1    // fp32 SAT before the exact test when settling sightlines with a known blocker
#endif
#ifndef VISRT_K2W_CHUNK
#define VISRT_K2W_CHUNK 16  // consecutive pairs per warp grab (r01 sweep 1/4/8/12/16/32: 16 best)
#endif
#ifndef VISRT_K2W_HISLOT
#define VISRT_K2W_HISLOT 0  // 1: sweep the highest-slot unresolved sightline first (r01: -1 % config 2, +4 % config 3)
#endif
// Large all-pairs launches grab tr x tc tiles of the pair matrix (PairArgs::tr, tc, tmorton); the
// launcher picks the shape by scene (launch_bits_t). VISRT_K2W_TR / VISRT_K2W_TC / VISRT_K2W_TMORTON /
// VISRT_K2W_WCT (6 | 8) override at run time (tests force every shape on small scenes).
#ifndef VISRT_K2W_TMORTON
#define VISRT_K2W_TMORTON 0
#endif
#ifndef VISRT_K2W_TR
#define VISRT_K2W_TR 2      // default tile shape of the resident scenes
#endif
#ifndef VISRT_K2W_TC
#define VISRT_K2W_TC 16
#endif
#ifndef VISRT_K2W_CHUNK_CAND
#define VISRT_K2W_CHUNK_CAND 2
#endif
#ifndef VISRT_K2W_PRI
#define VISRT_K2W_PRI 0     // 1: the aim face's tile is swept second (r01: more sweeps, 4-9% slower)
#endif
#ifndef VISRT_K2W_ROT
#define VISRT_K2W_ROT 1     // candidate tiles of the home chunk start at the pair's own tile
#endif
#ifndef VISRT_K2W_MULTI
#define VISRT_K2W_MULTI 2     // extra blockers of the swept sightline used to settle its siblings (1 or 2)
#endif
#ifndef VISRT_K2W_NOSAT
#define VISRT_K2W_NOSAT 0   // 1: member boxes not culled, every member of a candidate tile runs the exact test
#endif
#ifndef VISRT_K2W_MORTON
#define VISRT_K2W_MORTON 0
#endif
#ifndef VISRT_K1_ROWS
#define VISRT_K1_ROWS 1   // 1: K1 as row tiles + sort (k_prefilter_rows) for >= 2^25 pairs; 0: always the cub selection
#endif
#ifndef VISRT_K2W_PRELOAD
#define VISRT_K2W_PRELOAD 1   // settling passes load the (warp-uniform) blocker's plane words once per blocker
#endif
#ifndef VISRT_K2W_RLOOP
#define VISRT_K2W_RLOOP 1     // the round's blockers settle through one loop (one inlined resolve site)
#endif
#ifndef VISRT_K2W_WC_TILED
#define VISRT_K2W_WC_TILED 6   // warp-cache entries of tiled launches (configs 3-5: r01 config 4 822 -> 803 ms)
#endif

// Development aid (-DVISRT_K2W_PROF): per-phase cycles of K2w (lane 0 of each warp).
#ifdef VISRT_K2W_PROF
__device__ unsigned long long g_k2w_prof[16];
#define K2P(i, v)                                                                                   \
    do {                                                                                            \
        if (lane == 0) atomicAdd(&g_k2w_prof[i], static_cast<unsigned long long>(v));               \
    } while (0)
#define K2CLK() clock64()
#else
#define K2P(i, v) \
    do {          \
    } while (0)
#define K2CLK() 0ll
#endif

template <int MAXV, int RES, int MINB, int NT = kThreads, int kWC = VISRT_K2W_WC>
__global__ void __launch_bounds__(NT, MINB) k_pair_bits_warp(PairArgs a) {
    constexpr int STRIDE = RecLayout<MAXV>::kStride;
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t bar[1];
    const DevScene& s = a.s;
    const int n = s.n;
    const int lane = threadIdx.x & 31;
    const SweepCtx ctx = sweep_setup<RES>(s, smem, bar);
    int wc = -1;        // lane q < kWC holds warp cache entry q (Morton index)
    int wc_next = 0;    // warp-uniform insertion cursor
    unsigned long long tests = 0, sweeps = 0, batches = 0;
    __shared__ unsigned char surv_buf[NT / 32][64];   // per warp: surviving members of a tile, in order
    unsigned char* sv = surv_buf[threadIdx.x >> 5];
    const unsigned lt = (1u << lane) - 1u;

    long long pnext = 0, pend = 0;
    int tI = 0, tJ = 0, tl = 0, tl_end = 0;   // tiled grabs: current tile origin and cursor
    const bool tiled = a.tiled != 0;
    const int TR = a.tr, TC = a.tc;
    const int ntc = tiled ? (n + TC - 1) / TC : 1;
    const long long ntiles_all = !tiled ? 0 : a.tile_end ? a.tile_end : static_cast<long long>((n + TR - 1) / TR) * ntc;
    const int row_end = a.row1 ? a.row1 : n;
    for (;;) {
        long long p = 0;
        int pi = 0, pj = 0;
        if (tiled) {
            // a warp takes a TR x TC tile of the pair matrix
            // (neighbouring reference AND aim faces: the warp cache stays warm)
            bool got = false, done = false;
            while (!got) {
                if (tl == tl_end) {
                    unsigned long long tw = 0;
                    if (lane == 0) tw = atomicAdd(&a.counter[0], 1ull);
                    const long long T = static_cast<long long>(__shfl_sync(kFull, tw, 0));
                    if (T >= ntiles_all) {
                        done = true;
                        break;
                    }
                    tI = static_cast<int>(T / ntc) * TR;
                    tJ = static_cast<int>(T % ntc) * TC;
                    tl = 0;
                    tl_end = tJ + TC - 1 > tI ? TR * TC : 0;   // skip tiles below the diagonal
                    continue;
                }
                const int l = tl++;
                pi = tI + l / TC;
                pj = tJ + l % TC;
                if (a.serp && ((l / TC) & 1)) pj = tJ + TC - 1 - l % TC;
                got = pi >= a.row0 && pi < row_end && pj < n && pj > pi;
            }
            if (done) break;
            if (a.tmorton) {
                // the tile is a block of Morton positions: its reference and aim faces
                // are spatial neighbours (index neighbours are only building-mates);
                // every unordered pair still comes up once, oriented lower index first
                const int oi = s.perm[pi], oj = s.perm[pj];
                pi = oi < oj ? oi : oj;
                pj = oi < oj ? oj : oi;
            }
        } else {
        // a warp takes VISRT_K2W_CHUNK consecutive pairs at a time: row-major
        // neighbours share the reference face (and its blockers: warp cache)
        if (pnext == pend) {
            unsigned long long pw = 0;
            if (lane == 0) pw = atomicAdd(&a.counter[0], static_cast<unsigned long long>(a.chunk));
            pnext = static_cast<long long>(__shfl_sync(kFull, pw, 0));
            if (pnext >= a.npairs) break;
            pend = min(pnext + a.chunk, a.npairs);
        }
        p = pnext++;
        if (a.ci) {
            pi = a.ci[p];
            pj = a.cj[p];
        } else {
            pair_from_index(p * a.stride, n, pi, pj);
#if VISRT_K2W_MORTON
            // walk the pair space in Morton order (spatially coherent pairs keep
            // the warp blocker cache warm); the verdict keeps the reference's
            // lower-index orientation
            {
                const int oi = s.perm[pi], oj = s.perm[pj];
                pi = oi < oj ? oi : oj;
                pj = oi < oj ? oj : oi;
            }
#endif
        }
        }
        const int si = s.inv[pi], sj = s.inv[pj];
        const int nr = s.nv[pi], na = s.nv[pj];
        const int grid = min(s.ns[pi] - nr - 1, s.ns[pj] - na - 1);
        const int S = nr * na + 1 + grid;
        unsigned unres = 0;
#pragma unroll
        for (int r = 0; r < 3; ++r)
            if (lane + 32 * r < S) unres |= 1u << r;
        double ax, ay, az, bx, by, bz;
        // sightline_endpoints without the integer division: v / na = (v * mg) >> 16 for v < 64
        const unsigned mg = (65536u + na - 1) / na;
        auto ends = [&](int ord) {
            int ri, ai;
            if (ord == 0) {
                ri = nr;
                ai = na;
            } else if (ord <= grid) {
                ri = nr + ord;
                ai = na + ord;
            } else {
                const unsigned v = static_cast<unsigned>(ord - 1 - grid);
                ri = static_cast<int>((v * mg) >> 16);
                ai = static_cast<int>(v) - ri * na;
            }
            const double* P = s.samples + (static_cast<size_t>(pi) * kMaxSamples + ri) * 3;
            const double* Q = s.samples + (static_cast<size_t>(pj) * kMaxSamples + ai) * 3;
            ax = P[0]; ay = P[1]; az = P[2];
            bx = Q[0]; by = Q[1]; bz = Q[2];
        };
        auto exact = [&](int k) {
            ++tests;
            return seg_hits<MAXV>(s.srec + static_cast<size_t>(k) * STRIDE, ax, ay, az, bx, by, bz);
        };
        // settle every unresolved sightline blocked by occluder k (Morton index)
        auto resolve = [&](int k) {
#if VISRT_K2W_PRELOAD && VISRT_SEG_V2
            // k is warp-uniform: its plane words are loaded once, ahead of the
            // sightlines' own loads, not once per sightline behind them
            const double2* V = reinterpret_cast<const double2*>(s.srec + static_cast<size_t>(k) * STRIDE);
            const double2 v0 = V[0], v1 = V[1], v2 = V[2];
#endif
            for (unsigned m = unres; m; m &= m - 1) {
                const int r = __ffs(m) - 1;
                ends(lane + 32 * r);
                if (!(!VISRT_K2W_RSAT || a.nocull || member_maybe(ctx, k, make_segf(s, ax, ay, az, bx, by, bz))))
                    continue;
#if VISRT_K2W_PRELOAD && VISRT_SEG_V2
                ++tests;
                if (seg_hits_pn<MAXV>(V, v0, v1, v2, ax, ay, az, bx, by, bz)) unres &= ~(1u << r);
#else
                if (exact(k)) unres &= ~(1u << r);
#endif
            }
        };

        bool clear = false;
        const long long pclk0 = K2CLK();
        if (may_touch(s, pi, pj)) {   // a degenerate sightline is never blocked
            bool degen = false;
            for (unsigned m = unres; m && !degen; m &= m - 1) {
                ends(lane + 32 * (__ffs(m) - 1));
                degen = degenerate(ax, ay, az, bx, by, bz);
            }
            clear = __any_sync(kFull, degen);
        }
        const long long cclk0 = K2CLK();
        if (!clear) {
            for (int i = 0; i < kWC; ++i) {   // most recent blocker first
                const int q = (wc_next + kWC - 1 - i) % kWC;
                const int k = __shfl_sync(kFull, wc, q);
                if (k < 0 || k == si || k == sj) continue;
                resolve(k);
                if (!__any_sync(kFull, unres != 0)) break;
            }
        }
        K2P(1, K2CLK() - cclk0);
        {
            const bool left = __any_sync(kFull, unres != 0);
            K2P(9, left ? 0 : 1);   // pairs settled by the cache alone
            (void)left;
        }
        while (!clear) {
            const unsigned who = __ballot_sync(kFull, unres != 0);
            if (!who) break;   // every sightline blocked: Occluded
            int L = __ffs(who) - 1;
            int r0 = __ffs(__shfl_sync(kFull, unres, L)) - 1;
#if VISRT_K2W_HISLOT
            // sweep a sightline of the highest occupied slot first (lane 0's
            // 33rd sightline of a quad pair): once it is settled, every resolve
            // pass over the pair is a single lane iteration
            for (int r = 2; r > 0; --r) {
                const unsigned wr = __ballot_sync(kFull, (unres >> r) & 1u);
                if (wr) {
                    L = __ffs(wr) - 1;
                    r0 = r;
                    break;
                }
            }
#endif
            ends(L + 32 * r0);   // the swept sightline, uniform across the warp
            const SegF g = make_segf(s, ax, ay, az, bx, by, bz);
            ++sweeps;
            const long long sclk0 = K2CLK();
            int hit = -1;
#if VISRT_K2W_MULTI
            int hit2 = -1, hit3 = -1;
#endif
            const int home = home_chunk(s, pi);
            if (RES == kStreamed && ctx.gbox && !a.flat && !a.nocull) {
                // non-resident scenes (config 4/5): tile -> group (shared memory) -> member (L1/L2)
                int more[2];
                hit = coop_any_hit_grouped<MAXV>(ctx, s.srec, g, ax, ay, az, bx, by, bz, si, sj, si, tests, batches,
                                                 more, VISRT_K2W_PRI ? sj : -1);
#if VISRT_K2W_MULTI
                if (hit >= 0) {
                    hit2 = more[0];
                    hit3 = VISRT_K2W_MULTI > 1 ? more[1] : -1;
                }
#endif
            }
            for (int cc = 0; cc < ctx.nchunks && hit < 0 && (RES != kStreamed || !ctx.gbox || a.flat || a.nocull); ++cc) {
                const int c = home + cc < ctx.nchunks ? home + cc : home + cc - ctx.nchunks;
                const int t0 = c * kTile;
                const int tc = min(kTile, ctx.ntiles - t0);
                if (VISRT_CHUNK_BOXES && ctx.nchunks > 1 && !a.nocull &&
                    !sat_maybe(ctx.cbox + static_cast<size_t>(c) * 8, g))
                    continue;
                const bool h0 = lane < tc && (a.nocull || sat_maybe(ctx.tbox + static_cast<size_t>(t0 + lane) * 8, g));
                const bool h1 = lane + 32 < tc &&
                                (a.nocull || sat_maybe(ctx.tbox + static_cast<size_t>(t0 + lane + 32) * 8, g));
                unsigned long long cand = static_cast<unsigned long long>(__ballot_sync(kFull, h0)) |
                                          (static_cast<unsigned long long>(__ballot_sync(kFull, h1)) << 32);
                unsigned long long later = 0;
                const int ti = (si >> 6) - t0;   // the reference face's tile (in range when cc == 0)
                if (VISRT_K2W_ROT && cc == 0) {   // the pair's own tile first, wrap around after
                    const unsigned long long below = (1ull << ti) - 1ull;
                    later = cand & below;
                    cand &= ~below;
                }
                // the aim face's tile right after the reference face's: a back-facing
                // end is blocked by its own building (Morton neighbours)
                unsigned long long pri = 0;
                {
                    const int tj = (sj >> 6) - t0;
                    if (VISRT_K2W_PRI && tj >= 0 && tj < 64 && (((cand | later) >> tj) & 1ull)) {
                        pri = 1ull << tj;
                        cand &= ~pri;
                        later &= ~pri;
                    }
                }
                bool first_done = false;
                ++batches;
                while ((cand | later | pri) && hit < 0) {
                    int tb;
                    if (pri && (first_done || cc != 0 || !((cand >> ti) & 1ull))) {
                        tb = __ffsll(static_cast<long long>(pri)) - 1;
                        pri = 0;
                    } else {
                        if (!cand) {
                            cand = later;
                            later = 0;
                        }
                        tb = __ffsll(static_cast<long long>(cand)) - 1;
                        cand &= cand - 1;
                    }
                    first_done = true;
                    const int base = (t0 + tb) * kTile;
                    const int mc = min(kTile, n - base);
                    const int m0 = base + lane, m1 = base + lane + 32;
                    bool v0, v1;
                    if (RES == kQuantised) {
                        const QSeg qs = make_qseg(g, ctx.tframe + static_cast<size_t>(t0 + tb) * 8);
                        v0 = lane < mc && m0 != si && m0 != sj && (VISRT_K2W_NOSAT || a.nocull || qsat(ctx.qbox[m0], qs));
                        v1 = lane + 32 < mc && m1 != si && m1 != sj &&
                             (VISRT_K2W_NOSAT || a.nocull || qsat(ctx.qbox[m1], qs));
                    } else {
                        v0 = lane < mc && m0 != si && m0 != sj &&
                             (VISRT_K2W_NOSAT || a.nocull || sat_maybe(ctx.mbox + static_cast<size_t>(m0) * 8, g));
                        v1 = lane + 32 < mc && m1 != si && m1 != sj &&
                             (VISRT_K2W_NOSAT || a.nocull || sat_maybe(ctx.mbox + static_cast<size_t>(m1) * 8, g));
                    }
                    const unsigned lo = __ballot_sync(kFull, v0), hi = __ballot_sync(kFull, v1);
                    ++batches;
                    const int clo = __popc(lo), tot = clo + __popc(hi);
                    if (tot == 0) continue;
                    // compact the survivors (member order) through shared memory
                    if (v0) sv[__popc(lo & lt)] = static_cast<unsigned char>(lane);
                    if (v1) sv[clo + __popc(hi & lt)] = static_cast<unsigned char>(32 + lane);
                    __syncwarp();
                    for (int r = 0; r < tot && hit < 0; r += 32) {
                        const int idx = r + lane < tot ? sv[r + lane] : -1;
                        const bool h = idx >= 0 && exact(base + idx);
                        const unsigned hb = __ballot_sync(kFull, h);
                        if (hb) {
                            hit = __shfl_sync(kFull, base + idx, __ffs(hb) - 1);
#if VISRT_K2W_MULTI
                            // the round's other blockers of this sightline are likely
                            // blockers of its siblings too: settle with them as well
                            const unsigned rest = hb & (hb - 1);
                            hit2 = rest ? __shfl_sync(kFull, base + idx, __ffs(rest) - 1) : -1;
                            const unsigned rest2 = rest & (rest - 1);
                            hit3 = (VISRT_K2W_MULTI > 1 && rest2) ? __shfl_sync(kFull, base + idx, __ffs(rest2) - 1) : -1;
#endif
                        }
                    }
                    __syncwarp();
                }
            }
            K2P(2, K2CLK() - sclk0);
            K2P(3, 1);
            if (hit < 0) {
                K2P(4, K2CLK() - sclk0);
                K2P(5, 1);
                clear = true;   // a sightline clear of every occluder
                break;
            }
            const long long rclk0 = K2CLK();
            if (lane == L) unres &= ~(1u << r0);   // the swept sightline: its sweep found `hit` blocking it
            if (lane == wc_next) wc = hit;
            wc_next = wc_next + 1 == kWC ? 0 : wc_next + 1;
#if VISRT_K2W_MULTI && VISRT_K2W_RLOOP
            // one resolve site for the round's blockers (code size: the predicate
            // and the sightline set-up are inlined once, not three times)
            for (int hq = 0; hq < 3; ++hq) {
                const int hk = hq == 0 ? hit : (hq == 1 ? hit2 : hit3);
                if (hk < 0) break;   // hit3 is only set after hit2
                if (hq > 0 && !__any_sync(kFull, unres != 0)) break;
                resolve(hk);
            }
#else
            resolve(hit);
#if VISRT_K2W_MULTI
            if (hit2 >= 0 && __any_sync(kFull, unres != 0)) resolve(hit2);
            if (hit3 >= 0 && __any_sync(kFull, unres != 0)) resolve(hit3);
#endif
#endif
            K2P(6, K2CLK() - rclk0);
        }
        K2P(0, K2CLK() - pclk0);
        K2P(7, 1);
        if (clear) {
            K2P(8, K2CLK() - pclk0);
            K2P(10, 1);
        }
        if (lane == 0) {
            if (clear) set_pair_bit(a.bits, s.words, pi, pj);
            if (a.cbit) a.cbit[p] = clear ? 1 : 0;
        }
    }
    for (int o = 16; o > 0; o >>= 1) tests += __shfl_down_sync(kFull, tests, o);
    if (lane == 0) {
        atomicAdd(&a.counter[1], tests);
        atomicAdd(&a.counter[2], sweeps);
        atomicAdd(&a.counter[3], batches);
    }
}

// Detail sweep: per pair every sightline against every occluder (no early
// exit), as occlusion_judgment does, recording the blocker set.
template <int MAXV, bool RESIDENT>
__global__ void __launch_bounds__(kThreads, 3) k_pair_detail(PairArgs a) {
    constexpr int STRIDE = RecLayout<MAXV>::kStride;
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t bar[1];
    const DevScene& s = a.s;
    const int lane = threadIdx.x & 31;
    const SweepCtx ctx = sweep_setup<RESIDENT>(s, smem, bar);

    bool active = false, exhausted = false, hit_any = false;
    long long pidx = 0;
    int pi = 0, pj = 0, si = 0, sj = 0, nr = 0, na = 0, grid = 0, S = 0, ord = 0, blocked = 0;
    double ax = 0, ay = 0, az = 0, bx = 0, by = 0, bz = 0;
    Sweep sw{};
    unsigned long long tests = 0;
    uint32_t* mask_out = nullptr;

    // next non-degenerate sightline (degenerate ones are never blocked)
    auto next_sightline = [&]() {
        while (ord < S) {
            sightline_endpoints(s, pi, pj, nr, na, grid, ord, ax, ay, az, bx, by, bz);
            if (!degenerate(ax, ay, az, bx, by, bz)) {
                sw.start(make_segf(s, ax, ay, az, bx, by, bz), si, sj, home_chunk(s, pi), ctx.nchunks);
                hit_any = false;
                return;
            }
            ++ord;
        }
        a.kind[pidx] = static_cast<int8_t>(blocked == 0 ? 0 : (blocked == S ? 2 : 1));
        active = false;
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
                if (my >= a.npairs) {
                    exhausted = true;
                } else {
                    pidx = my;
                    pi = a.ci[my];
                    pj = a.cj[my];
                    si = s.inv[pi];
                    sj = s.inv[pj];
                    nr = s.nv[pi];
                    na = s.nv[pj];
                    grid = min(s.ns[pi] - nr - 1, s.ns[pj] - na - 1);
                    S = nr * na + 1 + grid;
                    ord = 0;
                    blocked = 0;
                    mask_out = a.blk_mask + static_cast<size_t>(my) * a.blk_words;
                    active = true;
                    next_sightline();
                }
            }
            need = __ballot_sync(kFull, !active && !exhausted);
        }
    };

    refill();
    for (;;) {
        if (active) {
            int base;
            unsigned long long mask = sweep_batch(sw, ctx, base);
            while (mask) {
                const int kk = __ffsll(static_cast<long long>(mask)) - 1;
                mask &= mask - 1;
                ++tests;
                if (seg_hits<MAXV>(s.srec + static_cast<size_t>(base + kk) * STRIDE, ax, ay, az, bx, by, bz)) {
                    hit_any = true;
                    const int k = s.perm[base + kk];
                    atomicOr(mask_out + (k >> 5), 1u << (k & 31));
                }
            }
            if (sw.done()) {
                if (hit_any) ++blocked;
                ++ord;
                next_sightline();
            }
        }
        refill();
        if (!__any_sync(kFull, active || !exhausted)) break;
    }
    for (int o = 16; o > 0; o >>= 1) tests += __shfl_down_sync(kFull, tests, o);
    if (lane == 0) atomicAdd(&a.counter[1], tests);
}

// K1: first_order_pair's gate for one unordered pair index.
struct PrefilterOp {
    DevScene s;
    __device__ bool front(int of, int probe) const {
        const double* P = s.pts + static_cast<size_t>(of) * VISRT_MAX_VERTS * 3;
        const double* N = s.normal + 3 * static_cast<size_t>(of);
        const double* Q = s.pts + static_cast<size_t>(probe) * VISRT_MAX_VERTS * 3;
        const int nv = s.nv[probe];
        for (int k = 0; k < nv; ++k) {
            if (dot_rel(Q[3 * k], Q[3 * k + 1], Q[3 * k + 2], P[0], P[1], P[2], N[0], N[1], N[2]) > kEps)
                return true;
        }
        return false;
    }
    __device__ bool operator()(long long p) const {
        int i, j;
        pair_from_index(p, s.n, i, j);
        if (s.orient[i] == 2 || s.orient[j] == 2) return false;
        if (!front(i, j) || !front(j, i)) return false;
        for (int pl = 0; pl < 3; ++pl) {
            if (!s.seg_ok[3 * i + pl] || !s.seg_ok[3 * j + pl]) continue;
            const double* a = s.seg + (static_cast<size_t>(i) * 3 + pl) * 6;
            const double* b = s.seg + (static_cast<size_t>(j) * 3 + pl) * 6;
            const double d = fabs(dadd(dmul(a[4], b[4]), dmul(a[5], b[5])));
            if (d >= 1.0 - 1e-9 || d <= 1e-9) return true;
        }
        return false;
    }
};

__global__ void k_split_pairs(const long long* sel, long long m, int n, int32_t* ci, int32_t* cj) {
    for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < m;
         k += static_cast<long long>(gridDim.x) * blockDim.x) {
        int i, j;
        pair_from_index(sel[k], n, i, j);
        ci[k] = i;
        cj[k] = j;
    }
}

__global__ void k_clear_pairs(unsigned long long* bits, int words, const int32_t* ci, const int32_t* cj,
                              long long m) {
    for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < m;
         k += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int i = ci[k], j = cj[k];
        atomicAnd(bits + static_cast<size_t>(i) * words + (j >> 6), ~(1ull << (j & 63)));
        atomicAnd(bits + static_cast<size_t>(j) * words + (i >> 6), ~(1ull << (i & 63)));
    }
}

// ---------------------------------------------------------------------------
// Host launchers
// ---------------------------------------------------------------------------

static int persistent_grid(const void* fn, size_t smem, int device, int threads = kThreads) {
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, smem);
    if (per < 1) per = 1;
    return sms * per;
}

template <class K>
static cudaError_t launch_persistent(K fn, size_t smem, const PairArgs& a, int device, cudaStream_t st,
                                     int threads = kThreads) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const int grid = persistent_grid(reinterpret_cast<const void*>(fn), smem, device, threads);
    fn<<<grid, threads, smem, st>>>(a);
    return cudaGetLastError();
}

// VISRT_FORCE_STREAM=1 keeps the member boxes in global memory (L1/L2) even
// when they fit in shared memory (tests cover both paths on small scenes).
static bool use_resident(int n) {
    static const bool force_stream = [] {
        const char* e = std::getenv("VISRT_FORCE_STREAM");
        return e && e[0] == '1';
    }();
    return !force_stream && n <= kResidentMaxBoxes;
}

static size_t sweep_smem(const DevScene& s, int res) { return sweep_smem_bytes(s.n, s.ntiles, res); }

// Quantised shared-memory member boxes (sweep.h QSeg/qsat, one CTA of
// kQThreads per SM) are an opt-in residency: VISRT_QUANT=1 uses them where the
// fp32 boxes do not fit (6,144 < N <= 24,576), VISRT_QUANT=2 everywhere (tests).
// Off by default — measured r02 on config 4 (B): 982 ms quantised vs 822 ms
// streamed; the 200 KB of shared memory leave L1 too small for the occluder
// records and the 8-bit boxes pass 18 % more exact tests.
static int quant_mode() {
    static const int m = [] {
        const char* e = std::getenv("VISRT_QUANT");
        return e ? std::atoi(e) : 0;   // off by default: measured slower
    }();
    return m;
}

static bool use_quantised(int n, bool resident_ok) {
    const int m = quant_mode();
    return m != 0 && n <= kQuantisedMaxBoxes && (m == 2 || !resident_ok);
}

// The warp-per-pair kernel is the default (r01: config 2 8.05 -> 6.31 ms,
// config 3 40.8 -> 34.1 ms); VISRT_K2_WARP=0 selects the lane-per-pair kernel.
static bool use_warp_k2() {
    static const bool w = [] {
        const char* e = std::getenv("VISRT_K2_WARP");
        return !(e && e[0] == '0');
    }();
    return w;
}

template <int MAXV>
static cudaError_t launch_bits_t(const PairArgs& a0, int device, cudaStream_t st) {
    static const int flat = [] {
        const char* e = std::getenv("VISRT_K2W_GROUPED");
        return e && e[0] == '0' ? 1 : 0;
    }();
    static const int stride = [] {
        const char* e = std::getenv("VISRT_K2_STRIDE");
        return e ? std::max(1, std::atoi(e)) : 1;
    }();
    PairArgs a = a0;
    a.flat = flat;
    // VISRT_NOCULL=1: every fp32 culling test (chunk, tile, member boxes, cache
    // pre-checks) passes, so every occluder runs the exact predicate — the
    // brute-force reference for the culled builds (tools/nocull_check.py)
    static const int nocull = [] {
        const char* e = std::getenv("VISRT_NOCULL");
        return e && e[0] == '1' ? 1 : 0;
    }();
    a.nocull = nocull;
    int smem_sm = 0;
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
    a.stride = (a.ci || a.row1) ? 1 : stride;   // the profiling stride walks whole all-pairs matrices only
    // all-pairs rows share the reference face over long runs; candidate lists are
    // short and sparse, where big grabs only unbalance the tail
    a.chunk = a.ci ? VISRT_K2W_CHUNK_CAND : VISRT_K2W_CHUNK;
    // all-pairs launches with >= 512 pairs per resident warp (configs 3-5) grab
    // 2 x 16 tiles of the pair matrix (r01: config 4 915 -> 831 ms, config 3
    // 12.9 -> 12.3 ms); smaller ones keep 16-pair rows (config 2: tiles of 32
    // pairs unbalance the tail)
    {   // keep >= 8 grabs per resident warp (small scenes: config 1 has 6,670 pairs)
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        const long long warps = static_cast<long long>(sms) * 3 * (kThreads / 32);
        const long long work = a.npairs - a.pbegin;   // pairs this launch decides
        a.chunk = static_cast<int>(std::max<long long>(1, std::min<long long>(a.chunk, work / (8 * warps))));
        // VISRT_K2W_TILED=0/1 forces the grab shape (tests run the tiled walk on small scenes)
        static const int tiled_env = [] {
            const char* e = std::getenv("VISRT_K2W_TILED");
            return e ? std::atoi(e) : -1;
        }();
        // Grab shape by scene (r02 sweeps, tools/r02_t9/t11..t15.sh; every shape gives the same bits):
        //  * streamed big scenes (config 4/5): 48 x 4 tiles of face INDICES — a long run of
        //    reference faces against four aim faces — walked boustrophedon (consecutive pairs
        //    always share a face), with an 8-entry cache (config 4: 2 x 16 804 ms, 16 x 8 760,
        //    32 x 4 736, 64 x 2 733, 128 x 1 833; Morton tiles 749-778; boustrophedon 64 x 2 733,
        //    64 x 4 723, 48 x 4 722, 64 x 6 735);
        //  * resident scenes (configs 2/3): rows of MORTON positions, 1 x tc with tc = pairs per
        //    warp / 14 in [8, 48] (config 3: index 2 x 16 12.2 ms -> Morton 1 x 48 11.0 ms;
        //    config 2: 16-pair index rows 3.75 ms -> Morton 1 x 16 3.45 ms).
        static const int tr_env = [] { const char* e = std::getenv("VISRT_K2W_TR"); return e ? std::atoi(e) : 0; }();
        static const int tc_env = [] { const char* e = std::getenv("VISRT_K2W_TC"); return e ? std::atoi(e) : 0; }();
        static const int tmorton_env = [] { const char* e = std::getenv("VISRT_K2W_TMORTON"); return e ? std::atoi(e) : -1; }();
        const bool big_scene = a.s.n > kResidentMaxBoxes;
        const long long per_warp = work / warps;
        const bool big = tiled_env >= 0 ? tiled_env == 1 : (big_scene ? per_warp >= 512 : per_warp >= 8 * 14);
        a.tiled = (!a.ci && a.stride == 1 && big) ? 1 : 0;
        a.tr = tr_env > 0 ? tr_env : (big_scene ? 48 : 1);
        a.tc = tc_env > 0 ? tc_env
                          : (big_scene ? 4 : static_cast<int>(std::min<long long>(48, std::max<long long>(8, per_warp / 14))));
        static const int serp_env = [] { const char* e = std::getenv("VISRT_K2W_SERP"); return e ? std::atoi(e) : -1; }();
        a.serp = serp_env >= 0 ? serp_env : (big_scene ? 1 : 0);
        a.tmorton = (tmorton_env >= 0 ? tmorton_env == 1 : !big_scene) && !a.row1 ? 1 : 0;   // row blocks cut face rows
        // the cursor's start value: the block's first tile (tiled) or first pair
        const int ntc = (a.s.n + a.tc - 1) / a.tc;
        long long start = a.pbegin;
        if (a.tiled && a.row1) {
            start = static_cast<long long>(a.row0 / a.tr) * ntc;
            a.tile_end = static_cast<long long>((a.row1 + a.tr - 1) / a.tr) * ntc;
        }
        if (start) {
            const unsigned long long s0 = static_cast<unsigned long long>(start);
            cudaError_t e = cudaMemcpyAsync(a.counter, &s0, sizeof(s0), cudaMemcpyHostToDevice, st);   // pageable: staged before return
            if (e != cudaSuccess) return e;
        }
    }
    if (a.stride > 1) a.npairs = (a.npairs + a.stride - 1) / a.stride;
    // K2w keeps the member boxes resident only while 3 CTAs still fit per SM:
    // occupancy beats residency (r01: config 3 resident 14.8 ms at 2 CTAs,
    // streamed with the group level 12.9 ms at 3 CTAs)
    bool res = use_resident(a.s.n);
    if (res && use_warp_k2() && 3 * (sweep_smem(a.s, kResident) + 3 * 1024) > static_cast<size_t>(smem_sm)) res = false;
    if (use_warp_k2() && use_quantised(a.s.n, res)) {
        // one CTA of kQThreads per SM holds the quantised member boxes
        const size_t qsm = sweep_smem(a.s, kQuantised);
        if (qsm + (kQThreads / 32) * 64 + 1024 <= static_cast<size_t>(smem_sm))
            return launch_persistent(k_pair_bits_warp<MAXV, kQuantised, 1, kQThreads>, qsm, a, device, st, kQThreads);
    }
    const size_t smem = sweep_smem(a.s, res);
    if (use_warp_k2()) {
        // register budget by occupancy: when shared memory already limits the
        // SM to <= 2 CTAs, take the 2-CTA register budget
        const bool two = smem + 1024 > static_cast<size_t>(smem_sm) / 3;
        // tiled launches (large all-pairs builds) keep VISRT_K2W_WC_TILED cached
        // blockers, row grabs VISRT_K2W_WC (a larger cache costs config 2 ~3 %)
        constexpr int WT = VISRT_K2W_WC_TILED;
        // streamed big scenes (config 4/5): 16 x 8 tiles with an 8-entry cache
        static const int wct_env = [] { const char* e = std::getenv("VISRT_K2W_WCT"); return e ? std::atoi(e) : 0; }();
        const int wct = wct_env > 0 ? wct_env : (a.s.n > kResidentMaxBoxes ? 8 : WT);
        if (a.tiled && !two && !res && wct == 8)
            return launch_persistent(k_pair_bits_warp<MAXV, false, VISRT_K2W_MINB, kThreads, 8>, smem, a, device, st);
        if (two) {
            if (a.tiled)
                return res ? launch_persistent(k_pair_bits_warp<MAXV, true, 2, kThreads, WT>, smem, a, device, st)
                           : launch_persistent(k_pair_bits_warp<MAXV, false, 2, kThreads, WT>, smem, a, device, st);
            return res ? launch_persistent(k_pair_bits_warp<MAXV, true, 2>, smem, a, device, st)
                       : launch_persistent(k_pair_bits_warp<MAXV, false, 2>, smem, a, device, st);
        }
        if (a.tiled)
            return res ? launch_persistent(k_pair_bits_warp<MAXV, true, VISRT_K2W_MINB, kThreads, WT>, smem, a, device, st)
                       : launch_persistent(k_pair_bits_warp<MAXV, false, VISRT_K2W_MINB, kThreads, WT>, smem, a, device,
                                           st);
        return res ? launch_persistent(k_pair_bits_warp<MAXV, true, VISRT_K2W_MINB>, smem, a, device, st)
                   : launch_persistent(k_pair_bits_warp<MAXV, false, VISRT_K2W_MINB>, smem, a, device, st);
    }
    return res ? launch_persistent(k_pair_bits<MAXV, true>, smem, a, device, st)
               : launch_persistent(k_pair_bits<MAXV, false>, smem, a, device, st);
}

template <int MAXV>
static cudaError_t launch_detail_t(const PairArgs& a, int device, cudaStream_t st) {
    const bool res = use_resident(a.s.n);
    const size_t smem = sweep_smem(a.s, res);
    return res ? launch_persistent(k_pair_detail<MAXV, true>, smem, a, device, st)
               : launch_persistent(k_pair_detail<MAXV, false>, smem, a, device, st);
}

cudaError_t launch_pair_bits(const PairArgs& a, int device, cudaStream_t st) {
    return a.s.maxv <= 4 ? launch_bits_t<4>(a, device, st) : launch_bits_t<8>(a, device, st);
}

cudaError_t launch_pair_detail(const PairArgs& a, int device, cudaStream_t st) {
    return a.s.maxv <= 4 ? launch_detail_t<4>(a, device, st) : launch_detail_t<8>(a, device, st);
}

// K1 row tiles: the same gate as PrefilterOp with the pair loop reorganised
// for the GPU — a block takes 8 consecutive reference faces (a warp each) and
// walks their aim faces j > i in chunks of 32 staged once in shared memory
// (first vertex + normal, the vertices, orientation, the plane segments'
// directions): the chunk's face data is read from L2 once per 8 rows instead
// of once per pair, and no pair index is ever decoded. Survivors are appended
// with one atomic per warp (the caller sorts them into row-major order).
constexpr int kK1Rows = 8;
template <int MAXV>
struct K1Face {
    double pn[6];           // first vertex, normal
    double v[MAXV * 3];     // vertices
    double sd[3][2];        // plane segment directions (seg[4], seg[5]) per plane
    int orient, nv, ok[3];
};
template <int MAXV>
__global__ void __launch_bounds__(256) k_prefilter_rows(DevScene s, unsigned long long* out, unsigned long long* count,
                                                         unsigned long long* cursor) {
    __shared__ K1Face<MAXV> chunk[32];
    __shared__ K1Face<MAXV> rowf[kK1Rows];
    __shared__ long long tile_s;
    const int n = s.n;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int ntile = (n + kK1Rows - 1) / kK1Rows;
    auto load = [&](K1Face<MAXV>& F, int f, int part) {   // part: one of 8 slices of the face, by lane group
        const double* P = s.pts + static_cast<size_t>(f) * VISRT_MAX_VERTS * 3;
        if (part == 0) {
            for (int d = 0; d < 3; ++d) F.pn[d] = P[d];
            for (int d = 0; d < 3; ++d) F.pn[3 + d] = s.normal[3 * static_cast<size_t>(f) + d];
            F.orient = s.orient[f];
            F.nv = s.nv[f];
        } else if (part == 1) {
            for (int q = 0; q < MAXV * 3; ++q) F.v[q] = q < s.nv[f] * 3 ? P[q] : 0.0;
        } else if (part == 2) {
            for (int pl = 0; pl < 3; ++pl) {
                F.ok[pl] = s.seg_ok[3 * f + pl];
                F.sd[pl][0] = s.seg[(static_cast<size_t>(f) * 3 + pl) * 6 + 4];
                F.sd[pl][1] = s.seg[(static_cast<size_t>(f) * 3 + pl) * 6 + 5];
            }
        }
    };
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) tile_s = static_cast<long long>(atomicAdd(cursor, 1ull));
        __syncthreads();
        const long long tile = tile_s;
        if (tile >= ntile) break;
        const int i0 = static_cast<int>(tile) * kK1Rows;
        // the block's 8 reference faces (3 slices each)
        if (threadIdx.x < kK1Rows * 3) {
            const int r = threadIdx.x / 3;
            if (i0 + r < n) load(rowf[r], i0 + r, threadIdx.x % 3);
        }
        const int i = i0 + w;
        for (int j0 = i0 + 1; j0 < n; j0 += 32) {
            __syncthreads();
            if (threadIdx.x < 96) {
                const int c = threadIdx.x / 3;
                if (j0 + c < n) load(chunk[c], j0 + c, threadIdx.x % 3);
            }
            __syncthreads();
            const int j = j0 + lane;
            bool keep = false;
            if (i < n && j < n && j > i) {
                const K1Face<MAXV>& A = rowf[w];
                const K1Face<MAXV>& B = chunk[lane];
                if (A.orient != 2 && B.orient != 2) {
                    // mutually_front (src/vismatrix.cpp:160-169): a vertex of each strictly in front of the other
                    bool fij = false, fji = false;
                    for (int k = 0; k < B.nv && !fij; ++k)
                        fij = dot_rel(B.v[3 * k], B.v[3 * k + 1], B.v[3 * k + 2], A.pn[0], A.pn[1], A.pn[2], A.pn[3],
                                      A.pn[4], A.pn[5]) > kEps;
                    if (fij)
                        for (int k = 0; k < A.nv && !fji; ++k)
                            fji = dot_rel(A.v[3 * k], A.v[3 * k + 1], A.v[3 * k + 2], B.pn[0], B.pn[1], B.pn[2],
                                          B.pn[3], B.pn[4], B.pn[5]) > kEps;
                    if (fij && fji)
                        for (int pl = 0; pl < 3 && !keep; ++pl) {   // required_planes (171-181) non-empty
                            if (!A.ok[pl] || !B.ok[pl]) continue;
                            const double d = fabs(dadd(dmul(A.sd[pl][0], B.sd[pl][0]), dmul(A.sd[pl][1], B.sd[pl][1])));
                            keep = d >= 1.0 - 1e-9 || d <= 1e-9;
                        }
                }
            }
            const unsigned b = __ballot_sync(kFull, keep);
            if (b) {
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd(count, static_cast<unsigned long long>(__popc(b)));
                base = __shfl_sync(kFull, base, 0);
                if (keep) {
                    const long long row = static_cast<long long>(i) * (2LL * n - i - 1) / 2;   // pairs before row i
                    out[base + __popc(b & ((1u << lane) - 1u))] = static_cast<unsigned long long>(row + (j - i - 1));
                }
            }
        }
    }
}

// Ordered compaction of the prefiltered pairs; returns the device count in *d_count.
cudaError_t launch_prefilter(const DevScene& s, long long npairs, long long* d_sel, long long* d_count,
                             void*& temp, size_t& temp_bytes, cudaStream_t st) {
    // row tiles pay off on big scenes (config 4: 10.6 -> 3.7 ms); below ~3e7
    // pairs the ordered selection is as fast and needs no sort
    if (VISRT_K1_ROWS && npairs >= (1LL << 25)) {
        // row tiles -> unordered survivors in d_sel, then a radix sort back into
        // the row-major (i, j) order PrefilterOp's ordered selection gives
        cudaError_t e = cudaMemsetAsync(d_count, 0, 2 * sizeof(long long), st);   // [0] count, [1] tile cursor
        if (e != cudaSuccess) return e;
        unsigned long long* cnt = reinterpret_cast<unsigned long long*>(d_count);
        int dev = 0, sms = 0, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (s.maxv <= 4) {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_prefilter_rows<4>, 256, 0);
            k_prefilter_rows<4><<<sms * std::max(per, 1), 256, 0, st>>>(s, reinterpret_cast<unsigned long long*>(d_sel),
                                                                      cnt, cnt + 1);
        } else {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_prefilter_rows<8>, 256, 0);
            k_prefilter_rows<8><<<sms * std::max(per, 1), 256, 0, st>>>(s, reinterpret_cast<unsigned long long*>(d_sel),
                                                                      cnt, cnt + 1);
        }
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        long long m = 0;
        e = cudaMemcpyAsync(&m, d_count, sizeof(long long), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess || m <= 1) return e;
        int bits = 1;
        while (bits < 63 && (1LL << bits) < npairs) ++bits;
        unsigned long long* keys = reinterpret_cast<unsigned long long*>(d_sel);
        unsigned long long* sorted = nullptr;
        e = cudaMallocAsync(&sorted, static_cast<size_t>(m) * sizeof(unsigned long long), st);
        if (e != cudaSuccess) return e;
        size_t need = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, need, keys, sorted, m, 0, bits, st);
        if (need > temp_bytes) {
            if (temp) cudaFree(temp);
            e = cudaMalloc(&temp, need);
            if (e != cudaSuccess) return e;
            temp_bytes = need;
        }
        e = cub::DeviceRadixSort::SortKeys(temp, temp_bytes, keys, sorted, m, 0, bits, st);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(keys, sorted, static_cast<size_t>(m) * sizeof(unsigned long long),
                                cudaMemcpyDeviceToDevice, st);
        cudaFreeAsync(sorted, st);
        return e;
    }
    thrust::counting_iterator<long long> in(0);
    PrefilterOp op{s};
    size_t need = 0;
    cudaError_t e = cub::DeviceSelect::If(nullptr, need, in, d_sel, d_count, npairs, op, st);
    if (e != cudaSuccess) return e;
    if (need > temp_bytes) {
        if (temp) cudaFree(temp);
        e = cudaMalloc(&temp, need);
        if (e != cudaSuccess) return e;
        temp_bytes = need;
    }
    return cub::DeviceSelect::If(temp, temp_bytes, in, d_sel, d_count, npairs, op, st);
}

cudaError_t launch_split_pairs(const long long* sel, long long m, int n, int32_t* ci, int32_t* cj,
                               cudaStream_t st) {
    if (m <= 0) return cudaSuccess;
    const int blocks = static_cast<int>(std::min<long long>((m + 255) / 256, 148 * 16));
    k_split_pairs<<<blocks, 256, 0, st>>>(sel, m, n, ci, cj);
    return cudaGetLastError();
}

cudaError_t launch_clear_pairs(unsigned long long* bits, int words, const int32_t* ci, const int32_t* cj,
                               long long m, cudaStream_t st) {
    if (m <= 0) return cudaSuccess;
    const int blocks = static_cast<int>(std::min<long long>((m + 255) / 256, 148 * 16));
    k_clear_pairs<<<blocks, 256, 0, st>>>(bits, words, ci, cj, m);
    return cudaGetLastError();
}

}  // namespace visrt

#ifdef VISRT_K2W_PROF
extern "C" int visrt_debug_k2w_prof(unsigned long long* out) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, visrt::g_k2w_prof, sizeof(visrt::g_k2w_prof));
    static const unsigned long long zero[16] = {};
    return static_cast<int>(cudaMemcpyToSymbol(visrt::g_k2w_prof, zero, sizeof(zero)));
}
#endif
#ifdef VISRT_SEG_STATS
extern "C" int visrt_debug_seg_stats(unsigned long long* out) {
    cudaDeviceSynchronize();
    return static_cast<int>(cudaMemcpyFromSymbol(out, visrt::g_seg_stats, sizeof(visrt::g_seg_stats)));
}
#endif
