// (3) Unfiltered image tree: image_tree(scene, source, max_depth)
// (src/raytracer.cpp:458-486, include/rt/raytracer.hpp:51-61).
//
// The reference recurses depth-first: for every face f != last (in face
// order) whose plane has the current image strictly in front
// (signed_distance > kEps), it appends the node (f, mirror_point(image, f),
// parent, depth) and recurses into it. Here the tree is grown level by level
// on the GPU — a warp per parent node walks all faces 32 at a time; a count
// pass, an exclusive scan and a fill pass (ballot prefix sums) write each
// parent's children contiguously in face order — and the host then assigns
// the depth-first (pre-order) positions from the subtree sizes, which gives
// exactly the reference's node vector.
#include <algorithm>
#include <vector>

#include <cub/cub.cuh>

#include "capi_internal.h"
#include "sweep.h"
#include "tables.h"

namespace visrt {
namespace {

struct ImgNode {
    int32_t face, parent;    // parent: index in the previous level (-1 at depth 1)
    double x, y, z;          // image
};

__device__ __forceinline__ double sdist(const DevScene& s, int f, double x, double y, double z) {
    const double* P = s.pts + static_cast<size_t>(f) * VISRT_MAX_VERTS * 3;
    const double* N = s.normal + 3 * static_cast<size_t>(f);
    return dot_rel(x, y, z, P[0], P[1], P[2], N[0], N[1], N[2]);
}

// FILL = false: count children per parent; true: write them at off[p].
template <bool FILL>
__global__ void __launch_bounds__(256) k_image_level(DevScene s, const ImgNode* in, long long nin, double sx,
                                                     double sy, double sz, unsigned long long* count,
                                                     const unsigned long long* off, ImgNode* out) {
    const int lane = threadIdx.x & 31;
    const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    const long long nparents = in ? nin : 1;
    for (long long p = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5; p < nparents;
         p += nwarps) {
        const double ix = in ? in[p].x : sx, iy = in ? in[p].y : sy, iz = in ? in[p].z : sz;
        const int last = in ? in[p].face : -1;
        unsigned long long w = FILL ? off[p] : 0ull;
        for (int base = 0; base < s.n; base += 32) {
            const int f = base + lane;
            const bool ok = f < s.n && f != last && sdist(s, f, ix, iy, iz) > kEps;
            const unsigned m = __ballot_sync(kFull, ok);
            if (FILL && ok) {
                ImgNode c;
                c.face = f;
                c.parent = in ? static_cast<int32_t>(p) : -1;
                // mirror_point (src/geom.cpp:122-124): p - n * (2 * signed_distance(p))
                const double* N = s.normal + 3 * static_cast<size_t>(f);
                const double d2 = dmul(2.0, sdist(s, f, ix, iy, iz));
                c.x = dsub(ix, dmul(N[0], d2));
                c.y = dsub(iy, dmul(N[1], d2));
                c.z = dsub(iz, dmul(N[2], d2));
                out[w + __popc(m & ((1u << lane) - 1u))] = c;
            }
            w += __popc(m);
        }
        if (!FILL && lane == 0) count[p] = w;
    }
}

}  // namespace
}  // namespace visrt

extern "C" int visrt_image_tree(visrt_scene* sc, const double* src, int32_t max_depth, int32_t* face,
                                int32_t* parent, int32_t* depth, double* image, int64_t cap, int64_t* nnodes,
                                visrt_stats* stats, void* stream) {
    using namespace visrt;
    return capi_guard([&] {
        ScopedDevice dev(sc);
        if (!src || !nnodes) throw UsageError("null argument");
        const DevScene& ds = scene_dev(sc);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        constexpr long long kMaxNodes = 1ll << 27;
        std::vector<std::vector<ImgNode>> levels;
        std::vector<void*> keep;
        FreeGuard guard{keep};
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float ms_total = 0.f;
        ImgNode* d_in = nullptr;
        long long nin = 0, total = 0;
        for (int d = 0; d < max_depth; ++d) {
            const long long np = d == 0 ? 1 : nin;
            if (np == 0) break;
            std::vector<void*> tmp;
            FreeGuard g2{tmp};
            unsigned long long* d_cnt = dalloc<unsigned long long>(static_cast<size_t>(np) + 1, tmp);
            unsigned long long* d_off = dalloc<unsigned long long>(static_cast<size_t>(np) + 1, tmp);
            ck(cudaMemsetAsync(d_cnt, 0, (np + 1) * 8, st), "memset");
            const int grid = static_cast<int>(std::min<long long>((np + 7) / 8, 148 * 16));
            cudaEventRecord(e0, st);
            k_image_level<false><<<grid, 256, 0, st>>>(ds, d_in, nin, src[0], src[1], src[2], d_cnt, nullptr, nullptr);
            ck(cudaGetLastError(), "k_image_level");
            size_t tb = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, tb, d_cnt, d_off, np + 1, st);
            void* d_tb = dalloc<char>(tb, tmp);
            ck(cub::DeviceScan::ExclusiveSum(d_tb, tb, d_cnt, d_off, np + 1, st), "scan");
            unsigned long long nout = 0;
            ck(cudaMemcpyAsync(&nout, d_off + np, 8, cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaStreamSynchronize(st), "sync");
            if (total + static_cast<long long>(nout) > kMaxNodes)
                throw UsageError("image tree exceeds 2^27 nodes; lower max_depth");
            ImgNode* d_out = dalloc<ImgNode>(static_cast<size_t>(nout), keep);
            k_image_level<true><<<grid, 256, 0, st>>>(ds, d_in, nin, src[0], src[1], src[2], nullptr, d_off, d_out);
            ck(cudaGetLastError(), "k_image_level");
            cudaEventRecord(e1, st);
            levels.emplace_back(static_cast<size_t>(nout));
            if (nout) ck(cudaMemcpyAsync(levels.back().data(), d_out, nout * sizeof(ImgNode), cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaStreamSynchronize(st), "sync");
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            ms_total += ms;
            d_in = d_out;
            nin = static_cast<long long>(nout);
            total += nin;
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        // depth-first positions: subtree sizes bottom-up, then pre-order
        const int L = static_cast<int>(levels.size());
        std::vector<std::vector<long long>> size(L), pos(L);
        for (int d = L - 1; d >= 0; --d) {
            size[d].assign(levels[d].size(), 1);
            if (d + 1 < L)
                for (size_t c = 0; c < levels[d + 1].size(); ++c) size[d][levels[d + 1][c].parent] += size[d + 1][c];
        }
        for (int d = 0; d < L; ++d) {
            pos[d].resize(levels[d].size());
            long long next_root = 0;
            std::vector<long long> cursor;   // next free position under each parent
            if (d > 0) {
                cursor.resize(levels[d - 1].size());
                for (size_t p = 0; p < cursor.size(); ++p) cursor[p] = pos[d - 1][p] + 1;
            }
            for (size_t k = 0; k < levels[d].size(); ++k) {
                if (d == 0) {
                    pos[d][k] = next_root;
                    next_root += size[d][k];
                } else {
                    long long& c = cursor[levels[d][k].parent];
                    pos[d][k] = c;
                    c += size[d][k];
                }
            }
        }
        *nnodes = total;
        if (face || parent || depth || image) {
            if (cap < total) throw UsageError("output capacity below the node count");
            for (int d = 0; d < L; ++d)
                for (size_t k = 0; k < levels[d].size(); ++k) {
                    const long long q = pos[d][k];
                    const ImgNode& nd = levels[d][k];
                    if (face) face[q] = nd.face;
                    if (parent) parent[q] = d == 0 ? -1 : static_cast<int32_t>(pos[d - 1][nd.parent]);
                    if (depth) depth[q] = d + 1;
                    if (image) {
                        image[3 * q] = nd.x;
                        image[3 * q + 1] = nd.y;
                        image[3 * q + 2] = nd.z;
                    }
                }
        }
        if (stats) {
            *stats = visrt_stats{};
            stats->pairs = total;
            stats->tests_exec = 0;
            stats->ms = ms_total;
        }
    });
}

// closest_diffraction_edge (src/vistable.cpp:529-561) for a batch of
// receivers: the host computes every closest point with the reference's
// arithmetic, ONE batched GPU sweep decides every receiver->closest-point
// sightline, and the reference's sequential selection (distance with kEps
// slack, ties to the lowest edge id) runs on the host over those answers —
// the sweep result of an edge the loop skips is simply not read.
namespace visrt {
void closest_edges(const visrt_scene* sc, int64_t nrx, const double* rx_xyz, int32_t nedges, const double* edge_ab,
                   const int32_t* edge_rank, int32_t* out_edge, float* ms_out, int64_t* tests_out, cudaStream_t st) {
    const DevScene& ds = scene_dev(sc);
    if (nedges > 0 && (!edge_ab || !edge_rank)) throw UsageError("null edge arrays");
    const long long nseg = nrx * static_cast<long long>(nedges);
    std::vector<double> A(3 * static_cast<size_t>(nseg)), B(3 * static_cast<size_t>(nseg)), D(static_cast<size_t>(nseg));
    for (int64_t r = 0; r < nrx; ++r) {
        const double* p = rx_xyz + 3 * r;
        for (int32_t e = 0; e < nedges; ++e) {
            const double* a = edge_ab + 6 * static_cast<size_t>(e);
            const double* b = a + 3;
            // closest_point_on_segment (src/vistable.cpp:529-535)
            const double dx = b[0] - a[0], dy = b[1] - a[1], dz = b[2] - a[2];
            const double len2 = dx * dx + dy * dy + dz * dz;
            double c[3];
            if (len2 <= kEps * kEps) {
                c[0] = a[0]; c[1] = a[1]; c[2] = a[2];
            } else {
                const double t = std::clamp(((p[0] - a[0]) * dx + (p[1] - a[1]) * dy + (p[2] - a[2]) * dz) / len2,
                                            0.0, 1.0);
                c[0] = a[0] + dx * t; c[1] = a[1] + dy * t; c[2] = a[2] + dz * t;
            }
            const size_t q = static_cast<size_t>(r) * nedges + e;
            const double ex = p[0] - c[0], ey = p[1] - c[1], ez = p[2] - c[2];
            D[q] = std::sqrt(ex * ex + ey * ey + ez * ez);   // distance(receiver, cp)
            for (int k = 0; k < 3; ++k) {
                A[3 * q + k] = p[k];
                B[3 * q + k] = c[k];
            }
        }
    }
    std::vector<uint8_t> clear(static_cast<size_t>(nseg), 0);
    float ms = 0.f;
    int64_t tests = 0;
    if (nseg > 0) {
        std::vector<void*> tmp;
        FreeGuard guard{tmp};
        double* dA = dalloc<double>(A.size(), tmp);
        double* dB = dalloc<double>(B.size(), tmp);
        uint8_t* dC = dalloc<uint8_t>(clear.size(), tmp);
        unsigned long long* d_ctr = dalloc<unsigned long long>(2, tmp);
        ck(cudaMemcpyAsync(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice, st), "H2D");
        ck(cudaMemcpyAsync(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice, st), "H2D");
        ck(cudaMemsetAsync(d_ctr, 0, 16, st), "memset");
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
        ck(launch_segments_clear(ds, nseg, dA, dB, dC, d_ctr, scene_device(sc), st), "k_segments_clear");
        cudaEventRecord(e1, st);
        unsigned long long ctr[2];
        ck(cudaMemcpyAsync(clear.data(), dC, clear.size(), cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaMemcpyAsync(ctr, d_ctr, 16, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "sync");
        cudaEventElapsedTime(&ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        tests = static_cast<int64_t>(ctr[1]);
    }
    // the reference's sequential selection (src/vistable.cpp:548-558)
    for (int64_t r = 0; r < nrx; ++r) {
        int best = -1;
        double best_dist = 0.0;
        for (int32_t e = 0; e < nedges; ++e) {
            const size_t q = static_cast<size_t>(r) * nedges + e;
            const double d = D[q];
            if (best >= 0 && d > best_dist + kEps) continue;
            if (!clear[q]) continue;
            if (best < 0 || d < best_dist - kEps ||
                (std::abs(d - best_dist) <= kEps && edge_rank[e] < edge_rank[best])) {
                best = e;
                best_dist = d;
            }
        }
        out_edge[r] = best;
    }
    if (ms_out) *ms_out = ms;
    if (tests_out) *tests_out = tests;
}
}  // namespace visrt

extern "C" int visrt_closest_edges(visrt_scene* sc, int64_t nrx, const double* rx_xyz, int32_t nedges,
                                   const double* edge_ab, const int32_t* edge_rank, int32_t* out_edge,
                                   visrt_stats* stats, void* stream) {
    using namespace visrt;
    return capi_guard([&] {
        ScopedDevice dev(sc);
        float ms = 0.f;
        int64_t tests = 0;
        closest_edges(sc, nrx, rx_xyz, nedges, edge_ab, edge_rank, out_edge, &ms, &tests,
                      static_cast<cudaStream_t>(stream));
        if (stats) {
            *stats = visrt_stats{};
            stats->pairs = nrx * static_cast<int64_t>(nedges);
            stats->tests_exec = tests;
            stats->ms = ms;
        }
    });
}
