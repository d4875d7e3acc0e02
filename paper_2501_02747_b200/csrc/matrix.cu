// (1) Inter-visibility matrix kernels for sm_100a.
//
//   K1 k-prefilter   first_order_pair's gate (src/vismatrix.cpp:597-604:
//                    non-oblique, mutually_front 160-169, required_planes
//                    171-181) over all i<j, ordered prefix-sum compaction
//                    (cub::DeviceSelect) into a candidate list.
//   K2 k_pair_bits   occlusion_judgment's Occluded verdict (253-302) with
//                    early exit: one lane = one pair state machine walking its
//                    sightlines; the block sweeps occluder tiles cyclically out
//                    of shared memory (TMA bulk copies, double-buffered), every
//                    lane testing the same occluder (smem broadcast) against its
//                    own sightline. A sightline stops at its first hit; a pair
//                    stops at its first clear (or degenerate) sightline.
//   K2d k_pair_detail Visible / Partial / Occluded + blocker sets (no early exit).
//
// All geometry is the reference's FP64 predicate with explicit _rn intrinsics
// (device.h), so every decision is bit-identical to the CPU oracle.
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

static int persistent_grid(const void* fn, size_t smem, int device) {
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kThreads, smem);
    if (per < 1) per = 1;
    return sms * per;
}

template <class K>
static cudaError_t launch_persistent(K fn, size_t smem, const PairArgs& a, int device, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const int grid = persistent_grid(reinterpret_cast<const void*>(fn), smem, device);
    fn<<<grid, kThreads, smem, st>>>(a);
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

static size_t sweep_smem(const DevScene& s, bool resident) { return sweep_smem_bytes(s.n, s.ntiles, resident); }

template <int MAXV>
static cudaError_t launch_bits_t(const PairArgs& a, int device, cudaStream_t st) {
    const bool res = use_resident(a.s.n);
    const size_t smem = sweep_smem(a.s, res);
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

// Ordered compaction of the prefiltered pairs; returns the device count in *d_count.
cudaError_t launch_prefilter(const DevScene& s, long long npairs, long long* d_sel, long long* d_count,
                             void*& temp, size_t& temp_bytes, cudaStream_t st) {
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
