// (3) Image-tree expansion for sm_100a (K6): TraceAccelerator::trace batched
// over snapshots, level by level.
//
// Reference: src/raytracer.cpp:400-430 (Engine::expand: level 1 over every
// face, deeper levels over the ChainFilter continuations + obliques, skip the
// immediate repeat, prune when the parent image is within kEps of / behind the
// candidate plane), 383-394 (attempt), 205-278 (resolve_sequence: forward
// images, backward unfolding with strict plane crossing + contains, legs
// longer than kEps, Occluder::clear per leg), 319-340 (build_chain_filter).
//
//   k_tree_expand  one warp per parent node: the warp walks the parent's
//                  candidate pool 32 at a time, prunes, and appends the
//                  surviving children with ballot/popc prefix sums + one
//                  atomic per warp (prefix-sum compaction into the next
//                  frontier).
//   k_tree_unfold  one thread per node of a level: forward images, backward
//                  unfolding, leg lengths; valid sequences are compacted
//                  into a candidate list.
//   k_tree_legs    one lane per candidate: each leg is a culled any-hit sweep
//                  (sweep.h) over all faces; candidates whose legs are all
//                  clear become paths.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <vector>

#include <cub/cub.cuh>

#include "capi_internal.h"
#include "device.h"
#include "sweep.h"
#include "tables.h"

namespace visrt {

struct TreeNode {
    int32_t snap, depth, f0, f1, f2, f3, rank, filtered;   // rank: continuation row of the last pair
    double ix, iy, iz;
};

struct Cand {
    int32_t snap, depth, f[4], edge;   // edge: diffraction edge index (-1: ends at the receiver)
    int32_t node;                      // keyed mode: index of the source node (result slot)
    double pts[21];                    // tx, reflections..., [diffraction point], rx
    double length;
};

struct TreeArgs {
    DevScene s;
    const int32_t* off1;      // conts1 CSR over faces (admitted aims, ascending)
    const int32_t* idx1;
    const long long* off2;    // conts2 CSR over directed admitted pairs (row-major rank)
    const int32_t* idx2;
    const int32_t* obl;
    int32_t nobl;
    const double* tx;
    const double* rx;
    int32_t rx_fixed;
    int32_t snap0, nsnap;     // batch
    int32_t max_refl;
    const TreeNode* in;       // nullptr: the batch's snapshot roots
    long long nin;
    TreeNode* out;
    unsigned long long* nout;
    long long cap;
    unsigned long long* nodes_per_snap;   // [total snapshots]
    Cand* cand;
    unsigned long long* ncand;
    long long cand_cap;
    visrt_path* paths;
    unsigned long long* npaths;
    long long path_cap;
    unsigned long long* counter;          // [0] cursor, [1] leg tests
    const int32_t* snap_edge;             // [total snapshots] closest diffraction edge or -1 (nullptr: none)
    const double* edge_ab;                // [nedges][6]
    int32_t brute;                        // brute_force_trace: no chain filter, no image prune
    // keyed mode (resolve_keys): every node is one fixed sequence; node.rank
    // holds its edge (-1: ends at the receiver); results go to per-node slots
    int32_t keyed;
    uint8_t* slot_ok;
    visrt_path* slot_paths;
};

__device__ __forceinline__ double sdist_face(const DevScene& s, int f, double x, double y, double z) {
    const double* P = s.pn + 6 * static_cast<size_t>(f);   // first vertex, then the normal (dense, 48 B)
    return dot_rel(x, y, z, P[0], P[1], P[2], P[3], P[4], P[5]);
}

// mirror_point (src/geom.cpp:122-124): p - n * (2 * signed_distance(p))
__device__ __forceinline__ void mirror_face(const DevScene& s, int f, double& x, double& y, double& z) {
    const double* N = s.pn + 6 * static_cast<size_t>(f) + 3;
    const double d2 = dmul(2.0, sdist_face(s, f, x, y, z));
    x = dsub(x, dmul(N[0], d2));
    y = dsub(y, dmul(N[1], d2));
    z = dsub(z, dmul(N[2], d2));
}

// ConvexPolygon::contains (src/geom.cpp:155-167) on an occluder record.
template <int MAXV>
__device__ __forceinline__ bool rec_contains(const double* __restrict__ R, double px, double py, double pz) {
    if (fabs(dot_rel(px, py, pz, R[0], R[1], R[2], R[3], R[4], R[5])) > kEps) return false;
    if (dot_rel(px, py, pz, R[0], R[1], R[2], R[6], R[7], R[8]) < -kEps) return false;
#pragma unroll
    for (int k = 1; k < MAXV; ++k) {
        const double* E = R + 9 + (k - 1) * 6;
        if (dot_rel(px, py, pz, E[0], E[1], E[2], E[3], E[4], E[5]) < -kEps) return false;
    }
    return true;
}

// Candidate pool of a parent node (Engine::expand, src/raytracer.cpp:400-430):
// all faces at the root or under an unfiltered prefix; else the chain
// continuations of the prefix, then the obliques.
struct Pool {
    const int32_t* list;
    long long lo, hi, npool;
    bool all;
    int d, last;
};

__device__ __forceinline__ TreeNode tree_parent(const TreeArgs& a, long long p) {
    if (a.in) return a.in[p];
    TreeNode par{};
    par.snap = a.snap0 + static_cast<int>(p);
    par.depth = 0;
    par.f0 = par.f1 = par.f2 = par.f3 = -1;
    par.rank = -1;
    par.filtered = a.brute ? 0 : 1;
    par.ix = a.tx[3 * static_cast<size_t>(par.snap)];
    par.iy = a.tx[3 * static_cast<size_t>(par.snap) + 1];
    par.iz = a.tx[3 * static_cast<size_t>(par.snap) + 2];
    return par;
}

__device__ __forceinline__ Pool tree_pool(const TreeArgs& a, const TreeNode& par, int n) {
    Pool q;
    q.d = par.depth;
    q.last = q.d == 0 ? -1 : (q.d == 1 ? par.f0 : (q.d == 2 ? par.f1 : (q.d == 3 ? par.f2 : par.f3)));
    q.list = nullptr;
    q.lo = 0;
    q.hi = n;
    q.all = q.d == 0 || !par.filtered;
    if (!q.all) {
        if (q.d == 1) {
            q.lo = a.off1[par.f0];
            q.hi = a.off1[par.f0 + 1];
            q.list = a.idx1;
        } else if ((q.d == 2 || q.d == 3) && par.rank >= 0) {
            // Markov-2 chains: the continuations of (..., p, t) are those of the
            // pair (p, t) (build_matrix growth, src/vismatrix.cpp:760-797)
            q.lo = a.off2[par.rank];
            q.hi = a.off2[par.rank + 1];
            q.list = a.idx2;
        } else {
            q.lo = q.hi = 0;
        }
    }
    q.npool = (q.hi - q.lo) + (q.all ? 0 : a.nobl);
    return q;
}

// candidate q of the pool: face c (+ its continuation rank at depth 1); ok =
// not the immediate repeat and the parent image strictly in front
__device__ __forceinline__ bool tree_child(const TreeArgs& a, const TreeNode& par, const Pool& P, long long q, int& c,
                                           int& rank) {
    rank = -1;
    if (q < P.hi - P.lo) {
        c = P.list ? P.list[P.lo + q] : static_cast<int>(P.lo + q);
        if (!P.all && P.d == 1) rank = static_cast<int>(P.lo + q);
    } else {
        c = a.obl[q - (P.hi - P.lo)];
    }
    return c != P.last && (a.brute || sdist_face(a.s, c, par.ix, par.iy, par.iz) > kEps);
}

// K6 level expansion, pass 1: children per parent (warp per parent).
__global__ void __launch_bounds__(256) k_tree_count(TreeArgs a, unsigned long long* cnt) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
    const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    const long long nparents = a.in ? a.nin : a.nsnap;
    for (long long p = warp; p < nparents; p += nwarps) {
        const TreeNode par = tree_parent(a, p);
        const Pool P = tree_pool(a, par, a.s.n);
        unsigned long long c_all = 0;
        for (long long q0 = 0; q0 < P.npool; q0 += 32) {
            const long long q = q0 + lane;
            int c, rank;
            const bool ok = q < P.npool && tree_child(a, par, P, q, c, rank);
            c_all += __popc(__ballot_sync(kFull, ok));
        }
        if (lane == 0) cnt[p] = c_all;
    }
}

// Per-snapshot node counts of one level: the level is ordered by snapshot
// (children are written in parent order, roots in snapshot order), so each
// snapshot's count is an upper_bound - lower_bound over the level.
__global__ void k_tree_snapcount(const TreeNode* lvl, long long nn, int snap0, int ns,
                                 unsigned long long* nodes_per_snap) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= ns) return;
    const int sn = snap0 + q;
    long long lo = 0, hi = nn;
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (lvl[mid].snap < sn) lo = mid + 1;
        else hi = mid;
    }
    long long lo2 = lo, hi2 = nn;
    while (lo2 < hi2) {
        const long long mid = (lo2 + hi2) >> 1;
        if (lvl[mid].snap <= sn) lo2 = mid + 1;
        else hi2 = mid;
    }
    nodes_per_snap[sn] += static_cast<unsigned long long>(lo2 - lo);
}

// Pass 2 (after an exclusive scan of the counts): each parent's children are
// written contiguously at off[p], in pool order — coalesced rows, no global
// append atomics, and a deterministic frontier order.
__global__ void __launch_bounds__(256) k_tree_expand(TreeArgs a, const unsigned long long* off) {
    const DevScene& s = a.s;
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
    const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    const long long nparents = a.in ? a.nin : a.nsnap;
    for (long long p = warp; p < nparents; p += nwarps) {
        const TreeNode par = tree_parent(a, p);
        const Pool P = tree_pool(a, par, s.n);
        unsigned long long w = off[p];
        for (long long q0 = 0; q0 < P.npool; q0 += 32) {
            const long long q = q0 + lane;
            int c = -1, rank = -1;
            const bool ok = q < P.npool && tree_child(a, par, P, q, c, rank);
            const unsigned m = __ballot_sync(kFull, ok);
            if (ok) {
                TreeNode ch;
                ch.snap = par.snap;
                ch.depth = P.d + 1;
                ch.f0 = P.d == 0 ? c : par.f0;
                ch.f1 = P.d == 1 ? c : par.f1;
                ch.f2 = P.d == 2 ? c : par.f2;
                ch.f3 = P.d == 3 ? c : par.f3;
                if (P.d == 1) {
                    ch.rank = rank;
                } else if (P.d == 2 && a.max_refl > 3) {
                    // rank of the admitted pair (f1, c): its row in idx1
                    int lo = a.off1[par.f1], hi = a.off1[par.f1 + 1];
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (a.idx1[mid] < c) lo = mid + 1;
                        else hi = mid;
                    }
                    ch.rank = (lo < a.off1[par.f1 + 1] && a.idx1[lo] == c) ? lo : -1;
                } else {
                    ch.rank = -1;
                }
                ch.filtered = par.filtered && s.orient[c] != 2;
                ch.ix = par.ix;
                ch.iy = par.iy;
                ch.iz = par.iz;
                mirror_face(s, c, ch.ix, ch.iy, ch.iz);
                a.out[w + __popc(m & ((1u << lane) - 1u))] = ch;
            }
            w += __popc(m);
        }
    }
}

// fermat_point_on_edge (src/raytracer.cpp:174-192)
__device__ void fermat_point(const double* E, const double* from, const double* to, double* p) {
    const double dx = dsub(E[3], E[0]), dy = dsub(E[4], E[1]), dz = dsub(E[5], E[2]);
    const double len = __dsqrt_rn(dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz)));
    if (len <= kEps) {
        p[0] = E[0]; p[1] = E[1]; p[2] = E[2];
        return;
    }
    const double il = __ddiv_rn(1.0, len);
    const double ux = dmul(dx, il), uy = dmul(dy, il), uz = dmul(dz, il);
    const double fx = dsub(from[0], E[0]), fy = dsub(from[1], E[1]), fz = dsub(from[2], E[2]);
    const double tx = dsub(to[0], E[0]), ty = dsub(to[1], E[1]), tz = dsub(to[2], E[2]);
    const double A = dadd(dadd(dmul(fx, ux), dmul(fy, uy)), dmul(fz, uz));
    const double B = dadd(dadd(dmul(tx, ux), dmul(ty, uy)), dmul(tz, uz));
    const double ax = dsub(fx, dmul(ux, A)), ay = dsub(fy, dmul(uy, A)), az = dsub(fz, dmul(uz, A));
    const double bx = dsub(tx, dmul(ux, B)), by = dsub(ty, dmul(uy, B)), bz = dsub(tz, dmul(uz, B));
    const double ra = __dsqrt_rn(dadd(dadd(dmul(ax, ax), dmul(ay, ay)), dmul(az, az)));
    const double rb = __dsqrt_rn(dadd(dadd(dmul(bx, bx), dmul(by, by)), dmul(bz, bz)));
    double t;
    if (dadd(ra, rb) <= kEps) t = dmul(0.5, dadd(A, B));
    else t = __ddiv_rn(dadd(dmul(A, rb), dmul(B, ra)), dadd(ra, rb));
    double c = __ddiv_rn(t, len);
    c = c < 0.0 ? 0.0 : (1.0 < c ? 1.0 : c);   // std::clamp(t / len, 0, 1)
    p[0] = dadd(E[0], dmul(dx, c));
    p[1] = dadd(E[1], dmul(dy, c));
    p[2] = dadd(E[2], dmul(dz, c));
}

__device__ __forceinline__ double dist3(const double* a, const double* b) {
    const double x = dsub(a[0], b[0]), y = dsub(a[1], b[1]), z = dsub(a[2], b[2]);
    return __dsqrt_rn(dadd(dadd(dmul(x, x), dmul(y, y)), dmul(z, z)));
}

// resolve_sequence up to the occlusion tests (src/raytracer.cpp:205-278): one
// thread per node (or per snapshot root for the line-of-sight sequence); with
// a diffraction edge for the snapshot, Engine::attempt's second sequence
// (ending at the edge's Fermat point) is unfolded too (383-394).
template <int MAXV>
__device__ void unfold_one(const TreeArgs& a, int snap, int d, const int* f, long long t, int kedge,
                           const double* pimg = nullptr) {
    constexpr int STRIDE = RecLayout<MAXV>::kStride;
    const DevScene& s = a.s;
    {
        const double* T = a.tx + 3 * static_cast<size_t>(snap);
        const double* Rx = a.rx_fixed ? a.rx : a.rx + 3 * static_cast<size_t>(snap);
        double img[5][3];
        img[0][0] = T[0];
        img[0][1] = T[1];
        img[0][2] = T[2];
        // The image chain img[k + 1] = mirror(img[k], f[k]) with the forward
        // test signed_distance(f[k], img[k]) > kEps. With pimg (the parent's
        // image = img[d - 1], the same mirror sequence: fused last level, not
        // brute) every forward test is known to hold — each prefix node and
        // this child passed it when created (tree_child's prune) — and only
        // img[d] is formed now; img[1 .. d-1] follow once the first backward
        // step (the most selective: it ends most sequences) has passed.
        int have = d;   // img[0 .. have] valid
        if (pimg) {
            img[d][0] = pimg[0];
            img[d][1] = pimg[1];
            img[d][2] = pimg[2];
            mirror_face(s, f[d - 1], img[d][0], img[d][1], img[d][2]);
            have = 0;
        } else {
            bool fwd = true;
            for (int k = 0; k < d && fwd; ++k) {
                if (sdist_face(s, f[k], img[k][0], img[k][1], img[k][2]) <= kEps) {
                    fwd = false;
                    break;
                }
                img[k + 1][0] = img[k][0];
                img[k + 1][1] = img[k][1];
                img[k + 1][2] = img[k][2];
                mirror_face(s, f[k], img[k + 1][0], img[k + 1][1], img[k + 1][2]);
            }
            if (!fwd) return;
        }
        auto complete_chain = [&]() {   // img[1 .. d-1] (img[d - 1] = the parent image)
            for (int k = 0; k + 1 < d - 1; ++k) {
                img[k + 1][0] = img[k][0];
                img[k + 1][1] = img[k][1];
                img[k + 1][2] = img[k][2];
                mirror_face(s, f[k], img[k + 1][0], img[k + 1][1], img[k + 1][2]);
            }
            if (d >= 2) {
                img[d - 1][0] = pimg[0];
                img[d - 1][1] = pimg[1];
                img[d - 1][2] = pimg[2];
            }
            have = d;
        };
        const int edge = a.keyed ? kedge : (a.snap_edge ? a.snap_edge[snap] : -1);
        for (int v = (a.keyed && kedge >= 0) ? 1 : 0; v < (edge >= 0 ? 2 : 1); ++v) {
            bool ok = true;
            double target[3] = {Rx[0], Rx[1], Rx[2]};
            if (v == 1) {
                double p[3];
                fermat_point(a.edge_ab + 6 * static_cast<size_t>(edge), img[d], Rx, p);
                if (dist3(p, Rx) <= kEps || dist3(p, img[d]) <= kEps) continue;
                target[0] = p[0];
                target[1] = p[1];
                target[2] = p[2];
            }
            double refl[4][3];
            double cx = target[0], cy = target[1], cz = target[2];
            for (int k = d - 1; k >= 0 && ok; --k) {
                if (k + 1 < d && have < d) complete_chain();
                const double da = sdist_face(s, f[k], cx, cy, cz);
                const double db = sdist_face(s, f[k], img[k + 1][0], img[k + 1][1], img[k + 1][2]);
                if (dmul(da, db) >= 0.0) {   // segment_plane_crossing, src/geom.cpp:182-189
                    ok = false;
                    break;
                }
                const double tt = __ddiv_rn(da, dsub(da, db));
                const double px = dadd(cx, dmul(dsub(img[k + 1][0], cx), tt));
                const double py = dadd(cy, dmul(dsub(img[k + 1][1], cy), tt));
                const double pz = dadd(cz, dmul(dsub(img[k + 1][2], cz), tt));
                if (!rec_contains<MAXV>(s.rec + static_cast<size_t>(f[k]) * STRIDE, px, py, pz)) {
                    ok = false;
                    break;
                }
                refl[k][0] = px;
                refl[k][1] = py;
                refl[k][2] = pz;
                cx = px;
                cy = py;
                cz = pz;
            }
            if (!ok) continue;
            Cand c;
            c.snap = snap;
            c.depth = d;
            c.f[0] = f[0];
            c.f[1] = f[1];
            c.f[2] = f[2];
            c.f[3] = f[3];
            c.edge = v ? edge : -1;
            c.node = static_cast<int32_t>(t);
            c.pts[0] = T[0];
            c.pts[1] = T[1];
            c.pts[2] = T[2];
            for (int k = 0; k < d; ++k) {
                c.pts[3 * (k + 1)] = refl[k][0];
                c.pts[3 * (k + 1) + 1] = refl[k][1];
                c.pts[3 * (k + 1) + 2] = refl[k][2];
            }
            int np = d + 1;
            if (v) {
                c.pts[3 * np] = target[0];
                c.pts[3 * np + 1] = target[1];
                c.pts[3 * np + 2] = target[2];
                ++np;
            }
            c.pts[3 * np] = Rx[0];
            c.pts[3 * np + 1] = Rx[1];
            c.pts[3 * np + 2] = Rx[2];
            double length = 0.0;
            for (int i = 0; i < np && ok; ++i) {
                const double seg = dist3(c.pts + 3 * i, c.pts + 3 * (i + 1));
                if (seg <= kEps) ok = false;
                length = dadd(length, seg);
            }
            if (!ok) continue;
            c.length = length;
            const unsigned long long slot = atomicAdd(a.ncand, 1ull);
            if (static_cast<long long>(slot) < a.cand_cap) a.cand[slot] = c;
        }
    }
}

template <int MAXV>
__global__ void __launch_bounds__(256) k_tree_unfold(TreeArgs a) {
    const long long nt = a.in ? a.nin : a.nsnap;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < nt; t += stride) {
        int snap, d;
        int f[4] = {-1, -1, -1, -1};
        if (a.in) {
            const TreeNode& nd = a.in[t];
            snap = nd.snap;
            d = nd.depth;
            f[0] = nd.f0;
            f[1] = nd.f1;
            f[2] = nd.f2;
            f[3] = nd.f3;
        } else {
            snap = a.snap0 + static_cast<int>(t);
            d = 0;
        }
        unfold_one<MAXV>(a, snap, d, f, t, a.keyed ? a.in[t].rank : -1);
    }
}

// The LAST level fused: per parent (warp) the children are counted (cnt[p])
// and unfolded on the spot instead of being written as a frontier level and
// read back — the deepest level is most of the tree (config 3 order 3: 4.3M of
// 4.3M nodes per snapshot), so this removes its node rows from HBM entirely.
#ifndef VISRT_K6L_COMPACT
#define VISRT_K6L_COMPACT 1   // 1: pruned-in children compacted before the unfold
#endif
#if VISRT_K6L_COMPACT
__shared__ int k6l_buf[8][64];   // per warp (256 threads): pending children of the current parent
#endif
#ifndef VISRT_K6L_GRAB
#define VISRT_K6L_GRAB 4   // parents per grab of the fused last level's work cursor
#endif
#ifndef VISRT_K6L_LAZY
#define VISRT_K6L_LAZY 1   // 1: fused last level forms the children's image chains lazily (unfold_one pimg)
#endif
#ifndef VISRT_K6L_MINB
#define VISRT_K6L_MINB 2   // CTAs per SM the fused last level's register budget targets (r02 final sweep, config 3 order 3 per 50 snapshots: 2 -> 16.5 ms, 3 -> 17.2, 4 -> 19.5)
#endif
template <int MAXV>
__global__ void __launch_bounds__(256, VISRT_K6L_MINB) k_tree_last(TreeArgs a, unsigned long long* cnt,
                                                                   unsigned long long* pcur) {
    const int lane = threadIdx.x & 31;
    const long long nparents = a.in ? a.nin : a.nsnap;
    long long pnext = 0, pend = 0;
    for (;;) {
        // parents grabbed dynamically (pool sizes vary widely between parents),
        // VISRT_K6L_GRAB at a time: one global atomic per grab, not per parent
        if (pnext == pend) {
            unsigned long long pw = 0;
            if (lane == 0) pw = atomicAdd(pcur, static_cast<unsigned long long>(VISRT_K6L_GRAB));
            pnext = static_cast<long long>(__shfl_sync(kFull, pw, 0));
            pend = min(pnext + VISRT_K6L_GRAB, nparents);
        }
        const long long p = pnext++;
        if (p >= nparents) break;
        const TreeNode par = tree_parent(a, p);
        const Pool P = tree_pool(a, par, a.s.n);
        const int fp[4] = {par.f0, par.f1, par.f2, par.f3};
        unsigned long long c_all = 0;
        // the parent image (= the children's img[d - 1]): lazy image chains
        // (unfold_one), not for brute_force_trace (no prune: forward tests live)
        const double pim[3] = {par.ix, par.iy, par.iz};
        const double* pimg = (VISRT_K6L_LAZY && !a.brute && !a.keyed) ? pim : nullptr;
#if VISRT_K6L_COMPACT
        // the children that pass the prune are compacted through shared memory
        // and unfolded 32 at a time (full lanes on the heavy unfold)
        int* buf = k6l_buf[threadIdx.x >> 5];
        int pend = 0;
        auto unfold_batch = [&](int m) {
            const int c = lane < m ? buf[lane] : -1;
            __syncwarp();
            if (c >= 0) {
                int f[4] = {fp[0], fp[1], fp[2], fp[3]};
                f[P.d] = c;
                unfold_one<MAXV>(a, par.snap, P.d + 1, f, -1, -1, pimg);
            }
        };
        for (long long q0 = 0; q0 < P.npool; q0 += 32) {
            const long long q = q0 + lane;
            int c = -1, rank;
            const bool ok = q < P.npool && tree_child(a, par, P, q, c, rank);
            const unsigned ob = __ballot_sync(kFull, ok);
            c_all += __popc(ob);
            if (ok) buf[pend + __popc(ob & ((1u << lane) - 1u))] = c;
            pend += __popc(ob);
            __syncwarp();
            if (pend >= 32) {
                unfold_batch(32);
                pend -= 32;
                if (lane < pend) buf[lane] = buf[32 + lane];
                __syncwarp();
            }
        }
        if (pend > 0) unfold_batch(pend);
        __syncwarp();
#else
        for (long long q0 = 0; q0 < P.npool; q0 += 32) {
            const long long q = q0 + lane;
            int c = -1, rank;
            const bool ok = q < P.npool && tree_child(a, par, P, q, c, rank);
            c_all += __popc(__ballot_sync(kFull, ok));
            if (ok) {
                int f[4] = {fp[0], fp[1], fp[2], fp[3]};
                f[P.d] = c;
                unfold_one<MAXV>(a, par.snap, P.d + 1, f, -1, -1, pimg);
            }
        }
#endif
        if (lane == 0) cnt[p] = c_all;
    }
}

// Per-snapshot node counts of a fused last level: the parents are in snapshot
// order, so snapshot sn's children are off[hi] - off[lo] over its parent range.
__global__ void k_tree_snapcount_parents(const TreeNode* par, long long np, const unsigned long long* off, int snap0,
                                         int ns, unsigned long long* nodes_per_snap) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= ns) return;
    const int sn = snap0 + q;
    long long lo = 0, hi = np;
    if (par) {
        long long l = 0, h = np;
        while (l < h) {
            const long long mid = (l + h) >> 1;
            if (par[mid].snap < sn) l = mid + 1;
            else h = mid;
        }
        lo = l;
        h = np;
        while (l < h) {
            const long long mid = (l + h) >> 1;
            if (par[mid].snap <= sn) l = mid + 1;
            else h = mid;
        }
        hi = l;
    } else {   // roots: parent q is snapshot snap0 + q
        lo = q;
        hi = q + 1;
    }
    nodes_per_snap[sn] += off[hi] - off[lo];
}

// Occluder::clear on every leg of every candidate (lane per candidate).
template <int MAXV, bool RESIDENT>
__global__ void __launch_bounds__(kThreads, 3) k_tree_legs(TreeArgs a) {
    constexpr int STRIDE = RecLayout<MAXV>::kStride;
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t bar[1];
    const DevScene& s = a.s;
    const int lane = threadIdx.x & 31;
    const SweepCtx ctx = sweep_setup<RESIDENT>(s, smem, bar);
    const long long ncand = static_cast<long long>(*a.ncand) < a.cand_cap ? static_cast<long long>(*a.ncand)
                                                                          : a.cand_cap;

    bool active = false, exhausted = false;
    long long cid = 0;
    int leg = 0, legs = 0, bc0 = -1, bc1 = -1;   // cache: Morton indices
    double ax = 0, ay = 0, az = 0, bx = 0, by = 0, bz = 0;
    Sweep sw{};
    unsigned long long tests = 0;

    auto emit = [&]() {
        const Cand& c = a.cand[cid];
        const unsigned long long slot = a.keyed ? static_cast<unsigned long long>(c.node) : atomicAdd(a.npaths, 1ull);
        if (a.keyed || static_cast<long long>(slot) < a.path_cap) {
            visrt_path p;
            p.nrefl = c.depth;
            p.faces[0] = c.f[0];
            p.faces[1] = c.f[1];
            p.faces[2] = c.f[2];
            p.faces[3] = c.f[3];
            p.edge = c.edge;
            p.snap = c.snap;
            p.pad = 0;
            const int npts = c.depth + 2 + (c.edge >= 0 ? 1 : 0);
            for (int i = 0; i < 21; ++i) p.points[i] = i < 3 * npts ? c.pts[i] : 0.0;
            p.length = c.length;
            if (a.keyed) {
                a.slot_paths[slot] = p;
                a.slot_ok[slot] = 1;
            } else {
                a.paths[slot] = p;
            }
        }
        active = false;
    };
    auto exact = [&](int k) {
        ++tests;
        return seg_hits<MAXV>(s.srec + static_cast<size_t>(k) * STRIDE, ax, ay, az, bx, by, bz);
    };
    // set up leg `leg`; legs a cached blocker already blocks end the candidate
    auto start_leg = [&]() {
        for (;;) {
            if (leg == legs) {
                emit();
                return;
            }
            const double* P = a.cand[cid].pts + 3 * leg;
            ax = P[0];
            ay = P[1];
            az = P[2];
            bx = P[3];
            by = P[4];
            bz = P[5];
            if ((bc0 >= 0 && exact(bc0)) || (bc1 >= 0 && exact(bc1))) {
                active = false;   // blocked leg: no path
                return;
            }
            const Cand& c = a.cand[cid];
            sw.start(make_segf(s, ax, ay, az, bx, by, bz), -1, -1,
                     home_chunk(s, leg == 0 ? (c.depth ? c.f[0] : -1) : (leg - 1 < c.depth ? c.f[leg - 1] : -1)),
                     ctx.nchunks);
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
                if (my >= ncand) {
                    exhausted = true;
                } else {
                    cid = my;
                    legs = a.cand[my].depth + 1 + (a.cand[my].edge >= 0 ? 1 : 0);
                    leg = 0;
                    active = true;
                    start_leg();
                }
            }
            need = __ballot_sync(kFull, !active && !exhausted);
        }
    };
    __shared__ int slots[kThreads];
    int* slot = slots + (threadIdx.x & ~31);
    auto step = [&]() {
        unsigned long long mask = 0;
        int base = 0;
        if (active) mask = sweep_batch(sw, ctx, base);
        const int hk = coop_exact<MAXV>(s.srec, mask, base, ax, ay, az, bx, by, bz, slot, tests, 0ull,
                                        [](int, unsigned long long) {});
        if (!active) return;
        if (hk >= 0) {
            if (hk != bc0) {
                bc1 = bc0;
                bc0 = hk;
            }
            active = false;   // blocked: the sequence supports no path
        } else if (sw.done()) {
            ++leg;
            start_leg();
        }
    };

    refill();
    for (;;) {
        step();
        refill();
        if (!__any_sync(kFull, active || !exhausted)) break;
    }
    for (int o = 16; o > 0; o >>= 1) tests += __shfl_down_sync(kFull, tests, o);
    if (lane == 0) atomicAdd(&a.counter[1], tests);
}

static int grid_of(const void* fn, int threads, size_t smem, int device) {
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, smem);
    return sms * std::max(per, 1);
}

template <int MAXV>
static void launch_legs_t(const TreeArgs& a, int device, cudaStream_t st) {
    const char* e = std::getenv("VISRT_FORCE_STREAM");
    const bool res = !(e && e[0] == '1') && a.s.n <= kResidentMaxBoxes;
    const size_t smem = sweep_smem_bytes(a.s.n, a.s.ntiles, res);
    if (res) {
        auto fn = k_tree_legs<MAXV, true>;
        ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)), "attr");
        fn<<<grid_of(reinterpret_cast<const void*>(fn), kThreads, smem, device), kThreads, smem, st>>>(a);
    } else {
        auto fn = k_tree_legs<MAXV, false>;
        ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)), "attr");
        fn<<<grid_of(reinterpret_cast<const void*>(fn), kThreads, smem, device), kThreads, smem, st>>>(a);
    }
    ck(cudaGetLastError(), "k_tree_legs");
}

}  // namespace visrt

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
using visrt::ck;

struct visrt_tracer {
    visrt_scene* scene = nullptr;
    int max_refl = 0;
    std::vector<void*> allocs;
    int32_t* off1 = nullptr;
    int32_t* idx1 = nullptr;
    long long* off2 = nullptr;
    int32_t* idx2 = nullptr;
    int32_t* obl = nullptr;
    int32_t nobl = 0;
    // diffraction edges (visrt_tracer_set_edges)
    std::vector<double> edge_ab;
    std::vector<int32_t> edge_rank;
    double* d_edge_ab = nullptr;
    // frontier / candidate / path buffers, allocated on the first trace
    visrt::TreeNode* lvl[2] = {nullptr, nullptr};
    unsigned long long* cnt = nullptr;   // per parent child counts (+1 for the scan total)
    unsigned long long* off = nullptr;
    void* scan_tmp = nullptr;
    size_t scan_bytes = 0;
    visrt::Cand* cand = nullptr;
    visrt_path* dpaths = nullptr;
    // results of the last trace
    int64_t nsnap = 0;
    std::vector<visrt_path> paths;
    std::vector<int64_t> path_off;
    std::vector<int64_t> nodes;
    std::vector<int32_t> snap_edge;   // per snapshot diffraction edge of the last trace (empty: none)
    ~visrt_tracer() {
        for (void* p : allocs) visrt::BlockCache::get().release(p);
    }
};

extern "C" int visrt_tracer_create(visrt_scene* sc, int max_refl, const uint64_t* admitted_bits, int64_t ntriples,
                                   const int32_t* triples, visrt_tracer** out) {
    return visrt::capi_guard([&] {
        visrt::ScopedDevice dev(sc);
        if (!out) throw visrt::UsageError("null out");
        *out = nullptr;
        if (max_refl < 0) throw visrt::VisError("reflection order must be non-negative");
        if (max_refl > 4) throw visrt::VisError("max reflection order must be between 1 and 4");
        if (max_refl >= 3 && !triples && ntriples > 0) throw visrt::UsageError("triples required");
        const visrt::HostScene& hs = visrt::scene_host(sc);
        const int n = hs.n;
        const int words = (n + 63) / 64;
        std::vector<uint64_t> bits(static_cast<size_t>(n) * words);
        if (admitted_bits) {
            std::memcpy(bits.data(), admitted_bits, bits.size() * 8);
        } else {
            ck(cudaMemcpy(bits.data(), visrt_matrix_bits_device(sc), bits.size() * 8, cudaMemcpyDeviceToHost),
               "D2H bits");
        }
        auto tr = std::make_unique<visrt_tracer>();
        tr->scene = sc;
        tr->max_refl = max_refl;
        // conts1: admitted aims per face, ascending (build_chain_filter sorts + uniques)
        std::vector<int32_t> off1(n + 1, 0), idx1;
        for (int p = 0; p < n; ++p) {
            for (int w = 0; w < words; ++w) {
                uint64_t m = bits[static_cast<size_t>(p) * words + w];
                while (m) {
                    const int b = __builtin_ctzll(m);
                    m &= m - 1;
                    idx1.push_back(w * 64 + b);
                }
            }
            off1[p + 1] = static_cast<int32_t>(idx1.size());
        }
        // conts2: per directed admitted pair (rank = position in idx1), sorted unique
        std::vector<long long> off2(idx1.size() + 1, 0);
        std::vector<int32_t> idx2;
        if (ntriples > 0) {
            std::vector<std::pair<long long, int32_t>> keyed;
            keyed.reserve(ntriples);
            for (int64_t k = 0; k < ntriples; ++k) {
                const int p = triples[3 * k], t = triples[3 * k + 1], c = triples[3 * k + 2];
                const int32_t* b = idx1.data() + off1[p];
                const int32_t* e = idx1.data() + off1[p + 1];
                const int32_t* it = std::lower_bound(b, e, t);
                if (it == e || *it != t) throw visrt::UsageError("triple prefix is not an admitted pair");
                keyed.push_back({static_cast<long long>(it - idx1.data()), c});
            }
            std::sort(keyed.begin(), keyed.end());
            keyed.erase(std::unique(keyed.begin(), keyed.end()), keyed.end());
            for (const auto& kv : keyed) {
                off2[kv.first + 1]++;
                idx2.push_back(kv.second);
            }
            for (size_t r = 0; r < idx1.size(); ++r) off2[r + 1] += off2[r];
        }
        std::vector<int32_t> obl;
        for (int f = 0; f < n; ++f)
            if (hs.orient[f] == 2) obl.push_back(f);
        auto up = [&](const void* src, size_t bytes) {
            void* p = nullptr;
            ck(cudaMalloc(&p, std::max<size_t>(bytes, 16)), "cudaMalloc");
            tr->allocs.push_back(p);
            if (bytes) ck(cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice), "H2D");
            return p;
        };
        tr->off1 = static_cast<int32_t*>(up(off1.data(), off1.size() * 4));
        tr->idx1 = static_cast<int32_t*>(up(idx1.data(), idx1.size() * 4));
        tr->off2 = static_cast<long long*>(up(off2.data(), off2.size() * 8));
        tr->idx2 = static_cast<int32_t*>(up(idx2.data(), idx2.size() * 4));
        tr->obl = static_cast<int32_t*>(up(obl.data(), obl.size() * 4));
        tr->nobl = static_cast<int32_t>(obl.size());
        *out = tr.release();
    });
}

extern "C" void visrt_tracer_destroy(visrt_tracer* t) { delete t; }

extern "C" int visrt_tracer_set_edges(visrt_tracer* tr, int32_t nedges, const double* edge_ab,
                                      const int32_t* edge_rank) {
    return visrt::capi_guard([&] {
        if (!tr) throw visrt::UsageError("null tracer");
        visrt::ScopedDevice dev(tr->scene);
        if (nedges > 0 && (!edge_ab || !edge_rank)) throw visrt::UsageError("null edge arrays");
        tr->edge_ab.assign(edge_ab, edge_ab + 6 * static_cast<size_t>(std::max(nedges, 0)));
        tr->edge_rank.assign(edge_rank, edge_rank + std::max(nedges, 0));
        tr->d_edge_ab = visrt::dalloc<double>(std::max<size_t>(tr->edge_ab.size(), 1), tr->allocs);
        if (nedges > 0)
            ck(cudaMemcpy(tr->d_edge_ab, tr->edge_ab.data(), tr->edge_ab.size() * 8, cudaMemcpyHostToDevice), "H2D");
    });
}

namespace {

// Scene::inside_building (src/scene.cpp:199-211) for closed-shell scenes.
bool inside_building(const visrt::HostScene& hs, const double* p) {
    int nb = 0;
    for (int f = 0; f < hs.n; ++f) nb = std::max(nb, hs.building[f] + 1);
    for (int b = 0; b < nb; ++b) {
        bool inside = true, any = false;
        for (int f = 0; f < hs.n && inside; ++f) {
            if (hs.building[f] != b) continue;
            any = true;
            const double* P = &hs.pts[static_cast<size_t>(f) * VISRT_MAX_VERTS * 3];
            const double* N = &hs.normal[3 * static_cast<size_t>(f)];
            const double d = (p[0] - P[0]) * N[0] + (p[1] - P[1]) * N[1] + (p[2] - P[2]) * N[2];
            if (d >= -visrt::kEps) inside = false;
        }
        if (any && inside) return true;
    }
    return false;
}

}  // namespace

extern "C" int visrt_trace(visrt_tracer* tr, int64_t nsnap, const double* tx, const double* rx, int flags,
                           visrt_trace_stats* stats, void* stream) {
    return visrt::capi_guard([&] {
        if (!tr) throw visrt::UsageError("null tracer");
        visrt::ScopedDevice dev(tr->scene);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const visrt::HostScene& hs = visrt::scene_host(tr->scene);
        const visrt::DevScene& ds = visrt::scene_dev(tr->scene);
        const int device = visrt::scene_device(tr->scene);
        const int rx_fixed = (flags & VISRT_TRACE_RX_FIXED) ? 1 : 0;
        const bool diffraction = (flags & VISRT_TRACE_DIFFRACTION) != 0;
        const bool brute = (flags & VISRT_TRACE_BRUTE_FORCE) != 0;
        // Engine ctor placement checks (src/raytracer.cpp:355-363)
        for (int64_t k = 0; k < nsnap; ++k) {
            const double* T = tx + 3 * k;
            const double* R = rx_fixed ? rx : rx + 3 * k;
            const double dx = T[0] - R[0], dy = T[1] - R[1], dz = T[2] - R[2];
            if (std::sqrt(dx * dx + dy * dy + dz * dz) <= visrt::kEps)
                throw visrt::PlaceError("transmitter and receiver coincide");
            if (inside_building(hs, T)) throw visrt::PlaceError("transmitter lies inside a building volume");
            if (inside_building(hs, R)) throw visrt::PlaceError("receiver lies inside a building volume");
        }
        std::vector<void*> tmp;
        visrt::FreeGuard guard{tmp};
        double* d_tx = visrt::dalloc<double>(static_cast<size_t>(nsnap) * 3, tmp);
        double* d_rx = visrt::dalloc<double>(static_cast<size_t>(rx_fixed ? 1 : nsnap) * 3, tmp);
        ck(cudaMemcpyAsync(d_tx, tx, nsnap * 24, cudaMemcpyHostToDevice, st), "H2D tx");
        ck(cudaMemcpyAsync(d_rx, rx, (rx_fixed ? 1 : nsnap) * 24, cudaMemcpyHostToDevice, st), "H2D rx");
        // Engine ctor: edge_ = closest_diffraction_edge(rx, scene) when allowed (src/raytracer.cpp:367)
        std::vector<int32_t> snap_edge;
        int32_t* d_snap_edge = nullptr;
        if (diffraction && !tr->edge_rank.empty()) {
            const int64_t nrx = rx_fixed ? 1 : nsnap;
            std::vector<int32_t> e(static_cast<size_t>(std::max<int64_t>(nrx, 1)), -1);
            visrt::closest_edges(tr->scene, nrx, rx, static_cast<int32_t>(tr->edge_rank.size()), tr->edge_ab.data(),
                                 tr->edge_rank.data(), e.data(), nullptr, nullptr, st);
            snap_edge.resize(static_cast<size_t>(nsnap));
            for (int64_t k = 0; k < nsnap; ++k) snap_edge[k] = rx_fixed ? e[0] : e[k];
            d_snap_edge = visrt::dalloc<int32_t>(snap_edge.size(), tmp);
            ck(cudaMemcpyAsync(d_snap_edge, snap_edge.data(), snap_edge.size() * 4, cudaMemcpyHostToDevice, st), "H2D");
        }
        unsigned long long* d_nodes = visrt::dalloc<unsigned long long>(std::max<int64_t>(nsnap, 1), tmp);
        ck(cudaMemsetAsync(d_nodes, 0, std::max<int64_t>(nsnap, 1) * 8, st), "memset");
        unsigned long long* d_ctr = visrt::dalloc<unsigned long long>(8, tmp);   // nout, ncand, npaths, cursor, tests
        // frontier / candidate / path buffers (capacity-bounded; batches adapt)
        const long long node_cap = 1ll << 25;   // 33.5M nodes per level per batch (1.9 GB per level buffer)
        const long long cand_cap = 1ll << 22;
        const long long path_cap = 1ll << 22;
        if (!tr->lvl[0]) {
            tr->cnt = visrt::dalloc<unsigned long long>(node_cap + 1, tr->allocs);
            tr->off = visrt::dalloc<unsigned long long>(node_cap + 1, tr->allocs);
            cub::DeviceScan::ExclusiveSum(nullptr, tr->scan_bytes, tr->cnt, tr->off, node_cap + 1);
            tr->scan_tmp = visrt::dalloc<char>(tr->scan_bytes, tr->allocs);
            tr->lvl[0] = visrt::dalloc<visrt::TreeNode>(node_cap, tr->allocs);
            tr->lvl[1] = visrt::dalloc<visrt::TreeNode>(node_cap, tr->allocs);
            tr->cand = visrt::dalloc<visrt::Cand>(cand_cap, tr->allocs);
            tr->dpaths = visrt::dalloc<visrt_path>(path_cap, tr->allocs);
        }
        visrt::TreeNode* lvl[2] = {tr->lvl[0], tr->lvl[1]};
        visrt::Cand* d_cand = tr->cand;
        visrt_path* d_paths = tr->dpaths;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);

        visrt::TreeArgs a{};
        a.s = ds;
        a.off1 = tr->off1;
        a.idx1 = tr->idx1;
        a.off2 = tr->off2;
        a.idx2 = tr->idx2;
        a.obl = tr->obl;
        a.nobl = tr->nobl;
        a.tx = d_tx;
        a.rx = d_rx;
        a.rx_fixed = rx_fixed;
        a.max_refl = tr->max_refl;
        a.nodes_per_snap = d_nodes;
        a.cand = d_cand;
        a.cand_cap = cand_cap;
        a.paths = d_paths;
        a.path_cap = path_cap;
        a.snap_edge = d_snap_edge;
        a.brute = brute ? 1 : 0;
        a.edge_ab = tr->d_edge_ab;
        std::vector<visrt_path> host_paths;
        int64_t total_nodes = 0, total_seq = 0, leg_tests = 0;
        unsigned long long* c_nout = d_ctr + 0;
        unsigned long long* c_ncand = d_ctr + 1;
        unsigned long long* c_npath = d_ctr + 2;
        const int eb = visrt::grid_of(reinterpret_cast<const void*>(visrt::k_tree_expand), 256, 0, device);
        const int ub = visrt::grid_of(reinterpret_cast<const void*>(ds.maxv <= 4 ? visrt::k_tree_unfold<4>
                                                                                  : visrt::k_tree_unfold<8>),
                                      256, 0, device);
        // One batch of snapshots: expand level by level; unfold + leg sweeps per
        // level; returns false when a level overflowed (caller halves the batch).
        auto run_batch = [&](int s0, int ns) -> bool {
            ck(cudaMemsetAsync(d_ctr, 0, 8 * 8, st), "memset");
            a.snap0 = s0;
            a.nsnap = ns;
            long long seqs = ns;   // line-of-sight sequences
            auto resolve_level = [&](const visrt::TreeNode* in, long long nin) -> bool {
                a.in = in;
                a.nin = nin;
                ck(cudaMemsetAsync(c_ncand, 0, 8, st), "memset");
                ck(cudaMemsetAsync(d_ctr + 3, 0, 8, st), "memset");
                if (ds.maxv <= 4) visrt::k_tree_unfold<4><<<ub, 256, 0, st>>>(a);
                else visrt::k_tree_unfold<8><<<ub, 256, 0, st>>>(a);
                ck(cudaGetLastError(), "k_tree_unfold");
                a.ncand = c_ncand;
                a.npaths = c_npath;
                a.counter = d_ctr + 3;
                if (ds.maxv <= 4) visrt::launch_legs_t<4>(a, device, st);
                else visrt::launch_legs_t<8>(a, device, st);
                unsigned long long nc = 0;
                ck(cudaMemcpyAsync(&nc, c_ncand, 8, cudaMemcpyDeviceToHost, st), "D2H");
                ck(cudaStreamSynchronize(st), "sync");
                return static_cast<long long>(nc) <= cand_cap;
            };
            a.ncand = c_ncand;
            if (!resolve_level(nullptr, ns)) return false;
            const visrt::TreeNode* in = nullptr;
            long long nin = ns;
            for (int depth = 0; depth < tr->max_refl; ++depth) {
                a.in = in;
                a.nin = nin;
                a.out = lvl[depth & 1];
                a.cap = node_cap;
                if (depth == tr->max_refl - 1) {
                    // deepest level: count + unfold fused, no frontier rows
                    const long long np = in ? nin : ns;
                    ck(cudaMemsetAsync(c_ncand, 0, 8, st), "memset");
                    ck(cudaMemsetAsync(d_ctr + 3, 0, 8, st), "memset");   // legs cursor
                    ck(cudaMemsetAsync(d_ctr + 5, 0, 8, st), "memset");   // k_tree_last parent cursor
                    // grid = the fused kernel's own residency on THIS device (one wave; per call, cheap)
                    if (ds.maxv <= 4) {
                        const int lb4 = visrt::grid_of(reinterpret_cast<const void*>(visrt::k_tree_last<4>),
                                                              256, 0, device);
                        visrt::k_tree_last<4><<<lb4, 256, 0, st>>>(a, tr->cnt, d_ctr + 5);
                    } else {
                        const int lb8 = visrt::grid_of(reinterpret_cast<const void*>(visrt::k_tree_last<8>),
                                                              256, 0, device);
                        visrt::k_tree_last<8><<<lb8, 256, 0, st>>>(a, tr->cnt, d_ctr + 5);
                    }
                    ck(cudaGetLastError(), "k_tree_last");
                    ck(cub::DeviceScan::ExclusiveSum(tr->scan_tmp, tr->scan_bytes, tr->cnt, tr->off, np + 1, st), "scan");
                    visrt::k_tree_snapcount_parents<<<(ns + 255) / 256, 256, 0, st>>>(in, np, tr->off, s0, ns, d_nodes);
                    ck(cudaGetLastError(), "k_tree_snapcount_parents");
                    a.ncand = c_ncand;
                    a.npaths = c_npath;
                    a.counter = d_ctr + 3;
                    if (ds.maxv <= 4) visrt::launch_legs_t<4>(a, device, st);
                    else visrt::launch_legs_t<8>(a, device, st);
                    unsigned long long no = 0, nc = 0;
                    ck(cudaMemcpyAsync(&no, tr->off + np, 8, cudaMemcpyDeviceToHost, st), "D2H");
                    ck(cudaMemcpyAsync(&nc, c_ncand, 8, cudaMemcpyDeviceToHost, st), "D2H");
                    ck(cudaStreamSynchronize(st), "sync");
                    if (static_cast<long long>(nc) > cand_cap) return false;
                    seqs += static_cast<long long>(no);
                    break;
                }
                // count -> exclusive scan -> fill (src/raytracer.cpp:400-430 per parent)
                const long long np = in ? nin : ns;
                visrt::k_tree_count<<<eb, 256, 0, st>>>(a, tr->cnt);
                ck(cudaGetLastError(), "k_tree_count");
                ck(cub::DeviceScan::ExclusiveSum(tr->scan_tmp, tr->scan_bytes, tr->cnt, tr->off, np + 1, st), "scan");
                unsigned long long no = 0;
                ck(cudaMemcpyAsync(&no, tr->off + np, 8, cudaMemcpyDeviceToHost, st), "D2H");
                ck(cudaStreamSynchronize(st), "sync");
                if (static_cast<long long>(no) > node_cap) return false;
                if (no) {
                    visrt::k_tree_expand<<<eb, 256, 0, st>>>(a, tr->off);
                    ck(cudaGetLastError(), "k_tree_expand");
                    visrt::k_tree_snapcount<<<(ns + 255) / 256, 256, 0, st>>>(lvl[depth & 1], static_cast<long long>(no),
                                                                             s0, ns, d_nodes);
                    ck(cudaGetLastError(), "k_tree_snapcount");
                }
                seqs += static_cast<long long>(no);
                if (no == 0) break;
                if (!resolve_level(lvl[depth & 1], static_cast<long long>(no))) return false;
                in = lvl[depth & 1];
                nin = static_cast<long long>(no);
            }
            unsigned long long np = 0, tests = 0;
            ck(cudaMemcpyAsync(&np, c_npath, 8, cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaMemcpyAsync(&tests, d_ctr + 4, 8, cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaStreamSynchronize(st), "sync");
            if (static_cast<long long>(np) > path_cap) return false;
            const size_t old = host_paths.size();
            host_paths.resize(old + np);
            if (np) ck(cudaMemcpy(host_paths.data() + old, d_paths, np * sizeof(visrt_path), cudaMemcpyDeviceToHost),
                       "D2H paths");
            total_seq += seqs;
            leg_tests += static_cast<int64_t>(tests);
            return true;
        };
        int batch = static_cast<int>(std::min<int64_t>(nsnap, 4096));
        for (int s0 = 0; s0 < nsnap;) {
            const int ns = static_cast<int>(std::min<int64_t>(batch, nsnap - s0));
            if (!run_batch(s0, ns)) {
                if (ns == 1) throw visrt::UsageError("one snapshot exceeds the frontier capacity");
                batch = std::max(1, ns / 2);
                // discard partial node counts of the failed batch
                std::vector<unsigned long long> zero(ns, 0);
                ck(cudaMemcpy(d_nodes + s0, zero.data(), ns * 8, cudaMemcpyHostToDevice), "reset");
                continue;
            }
            s0 += ns;
        }
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        std::vector<unsigned long long> nodes(std::max<int64_t>(nsnap, 1));
        ck(cudaMemcpy(nodes.data(), d_nodes, nodes.size() * 8, cudaMemcpyDeviceToHost), "D2H nodes");
        // group by snapshot, order by face sequence (deterministic output)
        std::sort(host_paths.begin(), host_paths.end(), [](const visrt_path& x, const visrt_path& y) {
            if (x.snap != y.snap) return x.snap < y.snap;
            if (x.nrefl != y.nrefl) return x.nrefl < y.nrefl;
            if (!std::equal(x.faces, x.faces + x.nrefl, y.faces))
                return std::lexicographical_compare(x.faces, x.faces + x.nrefl, y.faces, y.faces + y.nrefl);
            return x.edge < y.edge;
        });
        tr->nsnap = nsnap;
        tr->paths = std::move(host_paths);
        tr->path_off.assign(nsnap + 1, 0);
        for (const auto& p : tr->paths) tr->path_off[p.snap + 1]++;
        for (int64_t k = 0; k < nsnap; ++k) tr->path_off[k + 1] += tr->path_off[k];
        tr->nodes.assign(nsnap, 0);
        total_seq = 0;   // resolve_sequence calls: (nodes + LOS) x (1 + diffraction attempt)
        for (int64_t k = 0; k < nsnap; ++k) {
            tr->nodes[k] = static_cast<int64_t>(nodes[k]);
            total_nodes += tr->nodes[k];
            total_seq += (tr->nodes[k] + 1) * ((!snap_edge.empty() && snap_edge[k] >= 0) ? 2 : 1);
        }
        tr->snap_edge = snap_edge;
        if (stats) {
            stats->nodes = total_nodes;
            stats->sequences = total_seq;
            stats->paths = static_cast<int64_t>(tr->paths.size());
            stats->leg_tests = leg_tests;
            stats->ms = ms;
        }
    });
}

extern "C" int64_t visrt_trace_results(const visrt_tracer* tr, int64_t* path_off, visrt_path* paths, int64_t cap,
                                       int64_t* nodes) {
    if (!tr) return -1;
    if (path_off) std::copy(tr->path_off.begin(), tr->path_off.end(), path_off);
    if (paths) std::copy_n(tr->paths.begin(), std::min<int64_t>(cap, tr->paths.size()), paths);
    if (nodes) std::copy(tr->nodes.begin(), tr->nodes.end(), nodes);
    return static_cast<int64_t>(tr->paths.size());
}

extern "C" int64_t visrt_trace_snapshot_edges(const visrt_tracer* tr, int32_t* snap_edge) {
    if (!tr) return -1;
    if (snap_edge)
        for (int64_t k = 0; k < tr->nsnap; ++k) snap_edge[k] = tr->snap_edge.empty() ? -1 : tr->snap_edge[k];
    return tr->nsnap;
}

// resolve_keys (src/raytracer.cpp:554-570): re-solve fixed interaction
// sequences at new endpoints — the dynamic-run inner loop — as ONE batched
// pass: every (sample, key) is a keyed node of the unfold kernel (forward
// images, backward unfolding, Fermat point for a diffraction key) and its legs
// are swept by the leg kernel; results land in per-(sample, key) slots.
extern "C" int visrt_resolve_keys(visrt_scene* sc, int64_t nsamp, const double* tx, const double* rx, int flags,
                                  const int64_t* key_off, const visrt_seqkey* keys, int32_t nedges,
                                  const double* edge_ab, uint8_t* ok, visrt_path* paths, visrt_stats* stats,
                                  void* stream) {
    return visrt::capi_guard([&] {
        visrt::ScopedDevice dev(sc);
        if (nsamp < 0 || (nsamp > 0 && (!tx || !rx || !key_off))) throw visrt::UsageError("null argument");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const visrt::DevScene& ds = visrt::scene_dev(sc);
        const int device = visrt::scene_device(sc);
        const int rx_fixed = (flags & VISRT_TRACE_RX_FIXED) ? 1 : 0;
        const int64_t nk = nsamp > 0 ? key_off[nsamp] : 0;
        std::vector<visrt::TreeNode> nodes(static_cast<size_t>(nk));
        for (int64_t k = 0; k < nsamp; ++k) {
            for (int64_t q = key_off[k]; q < key_off[k + 1]; ++q) {
                const visrt_seqkey& K = keys[q];
                if (K.nrefl < 0 || K.nrefl > 4) throw visrt::UsageError("keys hold 0..4 reflections");
                for (int i = 0; i < K.nrefl; ++i)
                    if (K.faces[i] < 0 || K.faces[i] >= ds.n) throw visrt::UsageError("bad face index");
                if (K.edge < -1 || K.edge >= nedges) throw visrt::UsageError("bad edge index");
                visrt::TreeNode& nd = nodes[static_cast<size_t>(q)];
                nd = visrt::TreeNode{};
                nd.snap = static_cast<int32_t>(k);
                nd.depth = K.nrefl;
                nd.f0 = K.nrefl > 0 ? K.faces[0] : -1;
                nd.f1 = K.nrefl > 1 ? K.faces[1] : -1;
                nd.f2 = K.nrefl > 2 ? K.faces[2] : -1;
                nd.f3 = K.nrefl > 3 ? K.faces[3] : -1;
                nd.rank = K.edge;
            }
        }
        std::vector<void*> tmp;
        visrt::FreeGuard guard{tmp};
        auto up = [&](const void* src, size_t bytes) {
            void* d = visrt::dalloc<char>(std::max<size_t>(bytes, 16), tmp);
            if (bytes) ck(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, st), "H2D");
            return d;
        };
        double* d_tx = static_cast<double*>(up(tx, nsamp * 24));
        double* d_rx = static_cast<double*>(up(rx, (rx_fixed ? 1 : nsamp) * 24));
        visrt::TreeNode* d_nodes = static_cast<visrt::TreeNode*>(up(nodes.data(), nodes.size() * sizeof(visrt::TreeNode)));
        double* d_edges = static_cast<double*>(up(edge_ab, std::max(nedges, 0) * 48));
        uint8_t* d_ok = visrt::dalloc<uint8_t>(std::max<int64_t>(nk, 1), tmp);
        visrt_path* d_paths = visrt::dalloc<visrt_path>(std::max<int64_t>(nk, 1), tmp);
        const long long cand_cap = std::min<long long>(std::max<int64_t>(nk, 1), 1ll << 22);
        visrt::Cand* d_cand = visrt::dalloc<visrt::Cand>(cand_cap, tmp);
        unsigned long long* d_ctr = visrt::dalloc<unsigned long long>(4, tmp);   // ncand, cursor, tests
        ck(cudaMemsetAsync(d_ok, 0, std::max<int64_t>(nk, 1), st), "memset");
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
        visrt::TreeArgs a{};
        a.s = ds;
        a.tx = d_tx;
        a.rx = d_rx;
        a.rx_fixed = rx_fixed;
        a.edge_ab = d_edges;
        a.keyed = 1;
        a.cand = d_cand;
        a.cand_cap = cand_cap;
        a.ncand = d_ctr;
        a.counter = d_ctr + 1;
        unsigned long long tests = 0;
        const int ub = visrt::grid_of(reinterpret_cast<const void*>(ds.maxv <= 4 ? visrt::k_tree_unfold<4>
                                                                                  : visrt::k_tree_unfold<8>),
                                      256, 0, device);
        for (long long b0 = 0; b0 < nk; b0 += cand_cap) {
            const long long nb = std::min<long long>(cand_cap, nk - b0);
            a.in = d_nodes + b0;
            a.nin = nb;
            a.slot_ok = d_ok + b0;
            a.slot_paths = d_paths + b0;
            ck(cudaMemsetAsync(d_ctr, 0, 32, st), "memset");
            if (ds.maxv <= 4) visrt::k_tree_unfold<4><<<ub, 256, 0, st>>>(a);
            else visrt::k_tree_unfold<8><<<ub, 256, 0, st>>>(a);
            ck(cudaGetLastError(), "k_tree_unfold");
            if (ds.maxv <= 4) visrt::launch_legs_t<4>(a, device, st);
            else visrt::launch_legs_t<8>(a, device, st);
            unsigned long long t2 = 0;
            ck(cudaMemcpyAsync(&t2, d_ctr + 2, 8, cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaStreamSynchronize(st), "sync");
            tests += t2;
        }
        cudaEventRecord(e1, st);
        if (nk > 0) {
            ck(cudaMemcpyAsync(ok, d_ok, nk, cudaMemcpyDeviceToHost, st), "D2H");
            if (paths) ck(cudaMemcpyAsync(paths, d_paths, nk * sizeof(visrt_path), cudaMemcpyDeviceToHost, st), "D2H");
        }
        ck(cudaStreamSynchronize(st), "sync");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        int64_t found = 0;
        for (int64_t q = 0; q < nk; ++q) found += ok[q] != 0;
        if (stats) {
            *stats = visrt_stats{};
            stats->pairs = nk;
            stats->admitted = found;
            stats->tests_exec = static_cast<int64_t>(tests);
            stats->ms = ms;
        }
    });
}
