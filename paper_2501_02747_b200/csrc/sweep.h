// Culled any-hit occluder sweep shared by the matrix (K2), region (K4) and
// tree (K6) kernels. See matrix.cu for the design notes.
#pragma once

#include "device.h"

namespace visrt {

constexpr int kTile = 64;       // occluders per virtual tile (one 64-bit survivor mask)
constexpr int kThreads = 256;   // 8 warps
constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------------------
// Occluder sweep. Every lane walks the occluders cyclically in "virtual
// tiles" of kTile; per virtual tile it first runs the fp32 culling test on all
// kTile boxes (uniform index -> shared-memory broadcast), collecting a
// survivor mask, then runs the exact FP64 predicate on the survivors only
// (records read through L1/L2). Two box sources:
//   RESIDENT: all N culling boxes staged once in shared memory (one TMA bulk
//             copy); warps then run free, with no block barriers;
//   STREAM:   scenes too large for that stream kStreamTile-box tiles through
//             a double-buffered TMA ring with one block barrier per tile.
// ---------------------------------------------------------------------------
constexpr int kStreamTile = 256;          // boxes per streamed tile (4 virtual tiles)
constexpr int kResidentMaxBoxes = 6144;   // 192 KB of fp32 boxes

struct BoxStream {
    float* sbox;        // RESIDENT: [n][8]; STREAM: 2 x [kStreamTile][8]
    uint64_t* bar;
    const float* box;
    int n, ntiles, t0;

    __device__ int tile_of(int it) const { return (t0 + it) % ntiles; }
    __device__ void issue(int it) const {
        const int t = tile_of(it);
        const int cnt = min(kStreamTile, n - t * kStreamTile);
        const uint32_t bytes = static_cast<uint32_t>(cnt) * 32u;
        mbar_expect_tx(&bar[it & 1], bytes);
        bulk_g2s(sbox + (it & 1) * kStreamTile * 8, box + static_cast<size_t>(t) * kStreamTile * 8, bytes,
                 &bar[it & 1]);
    }
    __device__ void wait(int it) const { mbar_wait(&bar[it & 1], (it >> 1) & 1); }
    __device__ const float* tile(int it) const { return sbox + (it & 1) * kStreamTile * 8; }
};

template <bool RESIDENT>
__device__ __forceinline__ void sweep_init(BoxStream& bs) {
    if (threadIdx.x == 0) {
        mbar_init(&bs.bar[0], 1);
        mbar_init(&bs.bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (RESIDENT) {
            // one bulk copy per 64 KB chunk (the size operand is 32-bit, chunks keep it small)
            const uint32_t total = static_cast<uint32_t>(bs.n) * 32u;
            mbar_expect_tx(&bs.bar[0], total);
            for (uint32_t off = 0; off < total; off += 65536u) {
                const uint32_t b = min(65536u, total - off);
                bulk_g2s(reinterpret_cast<char*>(bs.sbox) + off, reinterpret_cast<const char*>(bs.box) + off, b,
                         &bs.bar[0]);
            }
        } else {
            bs.issue(0);
            bs.issue(1);
        }
    }
    if (RESIDENT) bs.wait(0);
}

// Survivor mask of one virtual tile (boxes B[0..cnt)), own faces excluded.
__device__ __forceinline__ unsigned long long tile_survivors(const float* __restrict__ B, int cnt, int base,
                                                            const SegF& g, int pi, int pj) {
    unsigned long long mask = 0;
#pragma unroll 4
    for (int kk = 0; kk < cnt; ++kk)
        if (sat_maybe(B + kk * 8, g)) mask |= 1ull << kk;
    if (pi >= base && pi < base + cnt) mask &= ~(1ull << (pi - base));
    if (pj >= base && pj < base + cnt) mask &= ~(1ull << (pj - base));
    return mask;
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

// Drives `vtile(boxes, base, cnt)` (one virtual tile for the whole warp) and
// `refill()` until the warp (RESIDENT) or the block (STREAM) runs dry.
template <bool RESIDENT, class VTile, class Busy, class Refill>
__device__ __forceinline__ void sweep_loop(BoxStream& bs, VTile&& vtile, Busy&& busy, Refill&& refill) {
    const int n = bs.n;
    const int nvt = (n + kTile - 1) / kTile;
    if (RESIDENT) {
        const int warp = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
        int vt = warp % nvt;
        for (;;) {
            const int base = vt * kTile;
            vtile(bs.sbox + static_cast<size_t>(base) * 8, base, min(kTile, n - base));
            refill();
            if (!__any_sync(kFull, busy())) break;
            if (++vt == nvt) vt = 0;
        }
    } else {
        for (int it = 0;; ++it) {
            bs.wait(it);
            const int tb = bs.tile_of(it) * kStreamTile;
            const int tcnt = min(kStreamTile, n - tb);
            const float* T = bs.tile(it);
            for (int v = 0; v < tcnt; v += kTile) {
                vtile(T + v * 8, tb + v, min(kTile, tcnt - v));
                refill();
            }
            const int alive = __syncthreads_or(busy());
            if (!alive) {
                bs.wait(it + 1);   // drain the in-flight tile before the CTA retires
                break;
            }
            if (threadIdx.x == 0) bs.issue(it + 2);
        }
    }
}

}  // namespace visrt
