// Device-side scene state and the exact FP64 predicate shared by the kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "visrt_internal.h"

namespace visrt {

struct DevScene {
    int32_t n = 0;
    int32_t maxv = 0;
    int32_t words = 0;             // uint64 words per bit-matrix row
    const double* rec = nullptr;   // occluder records (layout by maxv: 4 or 8)
    int32_t rec_stride = 0;        // doubles per record
    const double* samples = nullptr;
    const double* pts = nullptr;   // padded rings [n][8][3]
    const double* normal = nullptr;
    const double* pn = nullptr;    // [n][6] first vertex + normal (image-tree plane tests)
    const double* seg = nullptr;   // [n][3][6]
    const double* aabb = nullptr;  // [n][6]
    const int32_t* nv = nullptr;
    const int32_t* ns = nullptr;
    const int32_t* orient = nullptr;
    const int32_t* seg_ok = nullptr;
    const float* box = nullptr;    // [n][8] fp32 culling boxes (centre rel. origin, dilated half)
    double ox = 0, oy = 0, oz = 0; // box origin
    // two-level culling hierarchy (Morton order, sweep.h)
    const float* sbox = nullptr;   // [n][8] member boxes, Morton order
    const float* tbox = nullptr;   // [ntiles][8] tile union boxes
    const double* srec = nullptr;  // occluder records, Morton order
    const int32_t* perm = nullptr; // Morton position -> face index
    const int32_t* inv = nullptr;  // face index -> Morton position
    const float* gbox = nullptr;   // [ngroups][8] group union boxes (kGroup faces)
    const float* cbox = nullptr;   // [nchunks][8] chunk union boxes (64 tiles)
    const float* tframe = nullptr; // [ntiles][8] quantisation frame of each tile (sweep.h qsat)
    const uint32_t* qbox = nullptr;// [n even][2] 8-bit member boxes in their tile's frame
    int32_t ntiles = 0, nchunks = 0, ngroups = 0;
};

// A sightline in the fp32 culling frame: midpoint (relative to the scene
// origin), half extent and its absolute value.
struct SegF {
    float mx, my, mz, ex, ey, ez, ax, ay, az;
};

__device__ __forceinline__ SegF make_segf(const DevScene& s, double ax, double ay, double az, double bx,
                                          double by, double bz) {
    SegF g;
    g.mx = static_cast<float>(0.5 * (ax + bx) - s.ox);
    g.my = static_cast<float>(0.5 * (ay + by) - s.oy);
    g.mz = static_cast<float>(0.5 * (az + bz) - s.oz);
    g.ex = static_cast<float>(0.5 * (bx - ax));
    g.ey = static_cast<float>(0.5 * (by - ay));
    g.ez = static_cast<float>(0.5 * (bz - az));
    g.ax = fabsf(g.ex);
    g.ay = fabsf(g.ey);
    g.az = fabsf(g.ez);
    return g;
}

// Conservative segment-vs-box separating-axis test in fp32 (3 box axes + 3
// edge-cross axes). false => the segment cannot meet the face (the box is
// dilated by box_margin(), which bounds every fp32 rounding here), so the
// exact FP64 predicate is skipped; true => run the exact predicate.
__device__ __forceinline__ bool sat_maybe(const float* __restrict__ B, const SegF& g) {
    const float dx = g.mx - B[0], dy = g.my - B[1], dz = g.mz - B[2];
    const float hx = B[4], hy = B[5], hz = B[6];
    bool ok = fabsf(dx) <= hx + g.ax;
    ok &= fabsf(dy) <= hy + g.ay;
    ok &= fabsf(dz) <= hz + g.az;
    ok &= fabsf(__fmaf_rn(dy, g.ez, -dz * g.ey)) <= __fmaf_rn(hy, g.az, hz * g.ay);
    ok &= fabsf(__fmaf_rn(dz, g.ex, -dx * g.ez)) <= __fmaf_rn(hx, g.az, hz * g.ax);
    ok &= fabsf(__fmaf_rn(dx, g.ey, -dy * g.ex)) <= __fmaf_rn(hx, g.ay, hy * g.ax);
    return ok;
}

struct PairArgs {
    DevScene s;
    long long npairs;
    const int32_t* ci;               // candidate list (nullptr: all i<j)
    const int32_t* cj;
    uint8_t* cbit;                   // per-candidate not-Occluded bit (optional)
    unsigned long long* bits;        // N x words, symmetric
    unsigned long long* counter;     // [0] work cursor, [1] tests executed
    int8_t* kind;                    // detail: per pair 0/1/2
    uint32_t* blk_mask;              // detail: per pair ceil(N/32) words
    int32_t blk_words;
    int32_t flat;                    // K2w: 1 = non-resident sweep without the group level (A/B knob)
    int32_t chunk;                   // K2w: consecutive pairs per warp grab
    int32_t tiled;                   // K2w: 1 = grabs are tr x tc tiles of the pair matrix (all pairs)
    int32_t tr, tc;                  // K2w: tile shape (reference faces x aim faces), set by the launcher
    int32_t serp;                    // K2w: 1 = tiles are walked boustrophedon (consecutive pairs always share a face)
    int32_t tmorton;                 // K2w: 1 = tiles cut the pair matrix in Morton positions (spatial neighbours), not face indices
    int32_t stride;                  // K2w profiling aid: decide every stride-th pair only (VISRT_K2_STRIDE, default 1)
    int32_t nocull;                  // K2w: 1 = no fp32 culling, every occluder tested exactly (VISRT_NOCULL)
    // row block [row0, row1) of the i<j triangle (visrt_pair_visibility_rows; row1 = 0: every row).
    // The host starts the work cursor at the block's first pair / tile: all-pairs walks
    // count absolute pair indices in [pbegin, npairs), tiled walks tiles below tile_end.
    int32_t row0, row1;
    long long pbegin, tile_end;
};

// ---------------------------------------------------------------------------
// Exact FP64 arithmetic: explicit round-to-nearest intrinsics are never
// contracted into FMAs, so every product/sum rounds exactly like the
// reference's separate x86-64 SSE2 mul/add.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
// dot(p - a, v) = ((dx*vx + dy*vy) + dz*vz), include/rt/geom.hpp:29
__device__ __forceinline__ double dot_rel(double px, double py, double pz, double ax, double ay,
                                          double az, double vx, double vy, double vz) {
    return dadd(dadd(dmul(dsub(px, ax), vx), dmul(dsub(py, ay), vy)), dmul(dsub(pz, az), vz));
}

// segment_face_intersection (src/geom.cpp:169-180) + ConvexPolygon::contains
// (src/geom.cpp:155-167) on one occluder record R (see RecLayout).
#ifdef VISRT_SEG_STATS
// development aid: where the exact predicate decides (total, |d| <= eps, same
// side, off-plane, first edge, later edge, hit) — per translation unit
__device__ unsigned long long g_seg_stats[8];
#define SEG_STAT(k) atomicAdd(&g_seg_stats[k], 1ull)
#else
#define SEG_STAT(k) ((void)0)
#endif
#ifndef VISRT_SEG_V2
#define VISRT_SEG_V2 1   // 1: occluder records read as double2 words (LDG.E.128)
#endif
// The predicate on a record whose plane words (P, n: V[0..2]) the caller holds
// already — a warp-uniform occluder tested on many sightlines loads them once.
template <int MAXV>
__device__ __forceinline__ bool seg_hits_pn(const double2* __restrict__ V, double2 v0, double2 v1, double2 v2,
                                            double ax, double ay, double az, double bx, double by, double bz) {
    const double Px = v0.x, Py = v0.y, Pz = v1.x;
    const double nx = v1.y, ny = v2.x, nz = v2.y;
    const double da = dot_rel(ax, ay, az, Px, Py, Pz, nx, ny, nz);
    const double db = dot_rel(bx, by, bz, Px, Py, Pz, nx, ny, nz);
    if (fabs(da) <= kEps || fabs(db) <= kEps) return SEG_STAT(1), false;
    if (dmul(da, db) > 0.0) return SEG_STAT(2), false;
    const double t = __ddiv_rn(da, dsub(da, db));
    const double px = dadd(ax, dmul(dsub(bx, ax), t));
    const double py = dadd(ay, dmul(dsub(by, ay), t));
    const double pz = dadd(az, dmul(dsub(bz, az), t));
    if (fabs(dot_rel(px, py, pz, Px, Py, Pz, nx, ny, nz)) > kEps) return SEG_STAT(3), false;
    const double2 v3 = V[3], v4 = V[4];
    if (dot_rel(px, py, pz, Px, Py, Pz, v3.x, v3.y, v4.x) < -kEps) return SEG_STAT(4), false;
    double e0 = v4.y;
#pragma unroll
    for (int k = 1; k < MAXV; ++k) {
        const double2 w0 = V[3 * k + 2], w1 = V[3 * k + 3], w2 = V[3 * k + 4];
        if (dot_rel(px, py, pz, e0, w0.x, w0.y, w1.x, w1.y, w2.x) < -kEps) return SEG_STAT(5), false;
        e0 = w2.y;
    }
    SEG_STAT(6);
    return true;
}
template <int MAXV>
__device__ __forceinline__ bool seg_hits(const double* __restrict__ R, double ax, double ay,
                                         double az, double bx, double by, double bz) {
    SEG_STAT(0);
#if VISRT_SEG_V2
    // the record as 16-B words (records are 16-B multiples on a 256-B aligned
    // base): 14 LDG.E.128 instead of 27 LDG.E.64 for a quad; an edge's six
    // doubles start on an odd double, so its first one rides in the previous
    // stage's last word
    const double2* __restrict__ V = reinterpret_cast<const double2*>(R);
    const double2 v0 = V[0], v1 = V[1], v2 = V[2];
    return seg_hits_pn<MAXV>(V, v0, v1, v2, ax, ay, az, bx, by, bz);
#else
    const double Px = R[0], Py = R[1], Pz = R[2];
    const double nx = R[3], ny = R[4], nz = R[5];
    const double da = dot_rel(ax, ay, az, Px, Py, Pz, nx, ny, nz);
    const double db = dot_rel(bx, by, bz, Px, Py, Pz, nx, ny, nz);
    if (fabs(da) <= kEps || fabs(db) <= kEps) return SEG_STAT(1), false;
    if (dmul(da, db) > 0.0) return SEG_STAT(2), false;
    const double t = __ddiv_rn(da, dsub(da, db));
    const double px = dadd(ax, dmul(dsub(bx, ax), t));
    const double py = dadd(ay, dmul(dsub(by, ay), t));
    const double pz = dadd(az, dmul(dsub(bz, az), t));
    if (fabs(dot_rel(px, py, pz, Px, Py, Pz, nx, ny, nz)) > kEps) return SEG_STAT(3), false;
    if (dot_rel(px, py, pz, Px, Py, Pz, R[6], R[7], R[8]) < -kEps) return SEG_STAT(4), false;
#pragma unroll
    for (int k = 1; k < MAXV; ++k) {
        const double* E = R + 9 + (k - 1) * 6;
        if (dot_rel(px, py, pz, E[0], E[1], E[2], E[3], E[4], E[5]) < -kEps) return SEG_STAT(5), false;
    }
    SEG_STAT(6);
    return true;
#endif
}

// Unordered pair index p (i < j, row-major upper triangle) -> (i, j).
__device__ __forceinline__ void pair_from_index(long long p, int n, int& i, int& j) {
    const double b = 2.0 * n - 1.0;
    long long ii = static_cast<long long>((b - sqrt(b * b - 8.0 * static_cast<double>(p))) * 0.5);
    if (ii < 0) ii = 0;
    auto off = [n](long long r) { return r * (2LL * n - r - 1) / 2; };
    while (ii + 1 < n && off(ii + 1) <= p) ++ii;
    while (ii > 0 && off(ii) > p) --ii;
    i = static_cast<int>(ii);
    j = static_cast<int>(p - off(ii) + ii + 1);
}

// ---------------------------------------------------------------------------
// TMA bulk copy (cp.async.bulk, SASS UBLKCP) + mbarrier helpers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

}  // namespace visrt
